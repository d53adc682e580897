"""Optimizer-state remap and a short training run against the reference.

* RmsPropState.remap across a 3-round recursive calibrate: merged parents take
  the mean of their children's second moments (round by round), split
  children copy their parent's -- compared leaf by leaf in canonical order,
  bit-exactly (optim.py:89-104).
* train(): same data, config and seed as a reference train() run; leaf counts
  per epoch must match exactly, epoch losses within 1e-3 relative (the CUDA
  gradients are fp32 sums in atomic order, the reference's fp64 serial).
"""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_rmsprop_remap_matches_reference():
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.octree import from_pool_arrays
    from paper_2307_15333_b200.optim import RmsPropState
    from paper_2307_15333_b200.signals import SignalBuffer
    z = np.load(os.path.join(GOLDEN, "optim_remap.npz"))
    tree = from_pool_arrays(z, device="cuda")
    state = RmsPropState(tree)
    state.v_sigma.copy_(torch.from_numpy(z["v_sigma"]))
    state.v_sh.copy_(torch.from_numpy(z["v_sh"]))
    buf = SignalBuffer(tree)
    buf.accumulator.copy_(torch.from_numpy(z["acc"]))
    rep = calibrate(tree, buf, CalibrationConfig(tau=float(z["tau"]), gamma=float(z["gamma"]),
                                                 recursive=True), events=False)
    assert (rep.recursion_rounds, rep.merges_applied, rep.splits_applied) == (
        int(z["rounds"]), int(z["merges"]), int(z["splits"]))
    state.remap(rep)
    leaf = z["canon_is_leaf"]
    node = tree.topology().node.cpu().numpy()
    np.testing.assert_array_equal(node < 0, leaf)
    np.testing.assert_array_equal(state.v_sigma.cpu().numpy()[leaf], z["canon_v_sigma"][leaf])
    np.testing.assert_array_equal(state.v_sh.cpu().numpy()[leaf], z["canon_v_sh"][leaf])


class _Bundle:
    def __init__(self, origins, dirs, targets):
        self.origins, self.dirs, self.targets, self.heldout = origins, dirs, targets, []


def test_short_training_run_matches_reference():
    from paper_2307_15333_b200.octree import LeafPayload, build_dense
    from paper_2307_15333_b200.optim import TrainConfig, train
    from paper_2307_15333_b200.scene_io import load_tree_bytes
    z = np.load(os.path.join(GOLDEN, "train_small.npz"))
    trainee = build_dense(2, (0.0, 0.0, 0.0), 1.0, 1, LeafPayload(0.3, [0.0, 0.0, 0.0]),
                          max_depth=5, device="cuda")
    cfg = TrainConfig(epochs=6, interval=2, tau=0.5, gamma=0.1, batch_size=500, seed=3)
    _, hist = train(trainee, _Bundle(z["origins"], z["dirs"], z["targets"]), cfg)
    np.testing.assert_array_equal([h["leaf_count"] for h in hist], z["leaf_count"])
    np.testing.assert_allclose([h["loss"] for h in hist], z["loss"], rtol=1e-3)
    ref = load_tree_bytes(z["final_dot1"].tobytes(), device="cuda")
    np.testing.assert_array_equal(trainee.topology().node.cpu().numpy(),
                                  ref.topology().node.cpu().numpy())
    np.testing.assert_allclose(trainee.sigma.cpu().numpy(), ref.sigma.cpu().numpy(),
                               atol=1e-3, rtol=1e-3)


def _batch_setup(seed=11, B=16, n=1 << 15):
    from helpers import irregular_tree, ray_batch
    tree = irregular_tree(seed, B, depth=3, splits=80, merges=6, resplits=20, max_depth=6, device="cuda")
    o, d = ray_batch(seed + 1, 3 * n)
    t = np.random.default_rng(seed + 2).uniform(0, 1, (o.shape[0], 3))
    o, d, t = (torch.from_numpy(x).cuda() for x in (o, d, t))
    idx = torch.randperm(o.shape[0], generator=torch.Generator().manual_seed(seed))[:n].cuda()
    return tree, o, d, t, idx


def test_train_step_equals_unfused_step():
    """optim.train_step (in-place batch, signal into the accumulator,
    gradients consumed by the optimizer) == render_and_backprop on the
    gathered batch + rmsprop_step + SignalBuffer.accumulate."""
    from paper_2307_15333_b200.octree import from_canonical_tensors
    from paper_2307_15333_b200.optim import RmsPropState, StepWorkspace, rmsprop_step, train_step
    from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop
    from paper_2307_15333_b200.signals import SignalBuffer
    tree, o, d, t, idx = _batch_setup()
    topo = tree.topology()

    def clone():
        return from_canonical_tensors(tree.center, tree.half_extent, tree.basis_count, tree.max_depth,
                                      topo.node.clone(), tree._sigma.clone(), tree._sh_store.clone(),
                                      topo.level_offsets) if topo.pool_id is None else None

    if topo.pool_id is not None:  # make the tree canonical first
        from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
        tree = load_tree_bytes(tree_bytes(tree), device="cuda")
        topo = tree.topology()
    a, b = clone(), clone()
    sa, sb = RmsPropState(a), RmsPropState(b)
    ba, bb = SignalBuffer(a), SignalBuffer(b)
    ws = BackpropWorkspace.for_tree(a)
    sws = StepWorkspace(b, bb)
    for k in range(2):
        sl = idx[k * 8192:(k + 1) * 8192]
        loss_a, g, sig = render_and_backprop(a, o[sl], d[sl], t[sl], 0.5, workspace=ws)
        rmsprop_step(a, g, sa)
        ba.accumulate(sig, sl.numel())
        loss_b = train_step(b, o, d, t, sb, bb, sws, 0.5, ray_index=sl)
        assert float(loss_b) == pytest.approx(float(loss_a), rel=1e-6)  # step 2: fp32-atomic noise
    torch.testing.assert_close(b.sigma, a.sigma, atol=1e-5, rtol=1e-4)
    torch.testing.assert_close(b.sh, a.sh, atol=1e-5, rtol=1e-4)
    torch.testing.assert_close(sb.v_sh, sa.v_sh, atol=1e-9, rtol=1e-3)
    # step 2 runs on payloads that already differ by fp32-atomic noise
    torch.testing.assert_close(bb.accumulator, ba.accumulator, atol=1e-9, rtol=1e-4)
    assert bb.epoch_rays == ba.epoch_rays
    assert not bool(sws.ws.dsigma.any()) and not bool(sws.ws.dsh_store.any())


@pytest.mark.parametrize("basis", [1, 4, 9, 16])
def test_train_epoch_resident_planned_equals_plain(basis):
    """train_epoch over a ResidentRays pool with a coherence rank and cost
    column (plans prepared on a side stream, no sort) == train_epoch over the
    plain dataset (per-batch key sort): same batches from the same rng, so
    the epoch loss and the trained payload agree to fp32-atomic noise; the
    cost column is rewritten by the backward.  Every SH degree."""
    from paper_2307_15333_b200.octree import from_canonical_tensors
    from paper_2307_15333_b200.optim import ResidentRays, RmsPropState, TrainConfig, train_epoch
    from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
    from paper_2307_15333_b200.signals import SignalBuffer
    tree, o, d, t, _ = _batch_setup(seed=21, B=basis, n=1 << 15)
    tree = load_tree_bytes(tree_bytes(tree), device="cuda")
    topo = tree.topology()

    def clone():
        return from_canonical_tensors(tree.center, tree.half_extent, tree.basis_count, tree.max_depth,
                                      topo.node.clone(), tree._sigma.clone(), tree._sh_store.clone(),
                                      topo.level_offsets)

    data = _Bundle(o.cpu().numpy(), d.cpu().numpy(), t.cpu().numpy())
    cfg = TrainConfig(batch_size=20000, background=0.5)
    out = []
    for planned in (False, True):
        tr = clone()
        st, buf = RmsPropState(tr), SignalBuffer(tr)
        src = ResidentRays(tr, data, cfg.batch_size, plan=True) if planned else data
        if planned:
            assert src.rank is not None and src.costs is not None
            src.costs.zero_()  # every ray's entry is rewritten by the backward that trains it
        loss = train_epoch(tr, src, st, buf, cfg, np.random.default_rng(5))
        if planned:
            from paper_2307_15333_b200.render import ray_costs
            assert torch.equal(src.costs > 0, ray_costs(tr, src.origins, src.dirs) > 0)
        out.append((loss, tr, st, buf))
    (l0, a, sa, ba), (l1, b, sb, bb) = out
    assert l1 == pytest.approx(l0, rel=1e-5)
    torch.testing.assert_close(b.sigma, a.sigma, atol=1e-5, rtol=1e-4)
    torch.testing.assert_close(b.sh, a.sh, atol=1e-5, rtol=1e-4)
    torch.testing.assert_close(bb.accumulator, ba.accumulator, atol=1e-9, rtol=1e-4)
    assert bb.epoch_rays == ba.epoch_rays == o.shape[0]


def test_train_planned_matches_unplanned_across_refines():
    """train() with batches large enough for the ranked plan (ResidentRays:
    rays resident in key order, cost column, plans beside the update) over
    epochs with calibrations in between == the same epochs through the plain
    per-batch path: leaf counts equal every epoch, losses within fp32-atomic
    noise, the final topology identical."""
    from paper_2307_15333_b200.calibrate import calibrate
    from paper_2307_15333_b200.optim import ResidentRays, RmsPropState, TrainConfig, train, train_epoch
    from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
    from paper_2307_15333_b200.signals import SignalBuffer
    tree, o, d, t, _ = _batch_setup(seed=51, n=1 << 15)
    blob = tree_bytes(tree)
    data = _Bundle(o.cpu().numpy(), d.cpu().numpy(), t.cpu().numpy())
    cfg = TrainConfig(epochs=4, interval=2, tau=0.05, gamma=0.05, batch_size=20000, seed=9, background=0.5)
    a = load_tree_bytes(blob, device="cuda")
    _, hist = train(a, data, cfg)
    # the same schedule, unplanned batches
    b = load_tree_bytes(blob, device="cuda")
    state = RmsPropState(b, cfg.beta, cfg.eps, cfg.lr_sigma, cfg.lr_sh)
    buf = SignalBuffer(b, cfg.signal)
    rng = np.random.default_rng(cfg.seed)
    losses, leaves = [], []
    for epoch in range(1, cfg.epochs + 1):
        pool = ResidentRays(b, data, cfg.batch_size, cfg.early_stop_eps, plan=False)
        losses.append(train_epoch(b, pool, state, buf, cfg, rng))
        if epoch % cfg.interval == 0:
            rep = calibrate(b, buf, cfg.calibration(), events=False)
            state.remap(rep, reset=cfg.reset_state_on_calibration)
        leaves.append(b.leaf_count)
    assert [h["leaf_count"] for h in hist] == leaves
    np.testing.assert_allclose([h["loss"] for h in hist], losses, rtol=1e-5)
    np.testing.assert_array_equal(a.topology().node.cpu().numpy(), b.topology().node.cpu().numpy())


def test_train_epoch_device_shuffle_covers_every_ray_once():
    """TrainConfig(device_shuffle=True) draws the epoch permutation on the GPU:
    with the learning rates at zero (the payload fixed) an epoch still sees
    every ray exactly once -- the epoch's signal and mean loss equal the
    numpy-permutation epoch's (batch order does not matter then)."""
    from paper_2307_15333_b200.optim import ResidentRays, RmsPropState, TrainConfig, train_epoch
    from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
    from paper_2307_15333_b200.signals import SignalBuffer
    tree, o, d, t, _ = _batch_setup(seed=71, n=1 << 15)
    blob = tree_bytes(tree)
    data = _Bundle(o.cpu().numpy(), d.cpu().numpy(), t.cpu().numpy())
    out = []
    for dev_shuffle in (False, True):
        tr = load_tree_bytes(blob, device="cuda")
        cfg = TrainConfig(batch_size=20000, background=0.5, lr_sigma=0.0, lr_sh=0.0, device_shuffle=dev_shuffle)
        st, buf = RmsPropState(tr, lr_sigma=0.0, lr_sh=0.0), SignalBuffer(tr)
        pool = ResidentRays(tr, data, cfg.batch_size)
        loss = train_epoch(tr, pool, st, buf, cfg, np.random.default_rng(3))
        assert buf.epoch_rays == pool.n
        out.append((loss, buf.accumulator.clone()))
    assert out[1][0] == pytest.approx(out[0][0], rel=1e-9)
    torch.testing.assert_close(out[1][1], out[0][1], rtol=1e-10, atol=1e-12)


def test_rmsprop_sparse_equals_dense():
    """dot_rmsprop_step_sparse (touched rows listed first) == the dense
    update bit for bit on the same gradients: payload, state and the
    consumed (zeroed) gradients."""
    from paper_2307_15333_b200.octree import from_canonical_tensors
    from paper_2307_15333_b200.optim import RmsPropState, rmsprop_step
    from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop
    from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
    tree, o, d, t, idx = _batch_setup(seed=81, n=1 << 12)
    tree = load_tree_bytes(tree_bytes(tree), device="cuda")
    topo = tree.topology()
    ws = BackpropWorkspace.for_tree(tree)
    _, g0, _ = render_and_backprop(tree, o, d, t, 0.5, workspace=ws, ray_index=idx[: 1 << 11])
    torch.cuda.synchronize()
    assert 0 < int(ws.touched.sum()) < tree.capacity  # a sparse step
    outs = []
    for sparse in (False, True):
        tr = from_canonical_tensors(tree.center, tree.half_extent, tree.basis_count, tree.max_depth,
                                    topo.node.clone(), tree._sigma.clone(), tree._sh_store.clone(), topo.level_offsets)
        st = RmsPropState(tr)
        st.v_sh.copy_(torch.linspace(0.0, 1e-6, st.v_sh.numel(), dtype=torch.float64, device="cuda")
                      .reshape(st.v_sh.shape))
        w2 = BackpropWorkspace.for_tree(tr)
        w2.dsigma.copy_(ws.dsigma)
        w2.dsh_store.copy_(ws.dsh_store)
        w2.touched.copy_(ws.touched)
        from paper_2307_15333_b200.render import GradBuffer
        g = GradBuffer(w2.dsigma, w2.dsh_store[:, :3 * tr.basis_count], w2.touched, tr.generation, w2.dsh_store)
        rmsprop_step(tr, g, st, consume=True, sparse=sparse)
        torch.cuda.synchronize()
        outs.append((tr.sigma.clone(), tr.sh.clone(), st.v_sigma.clone(), st.v_sh.clone(), w2.dsigma.clone(),
                     w2.dsh_store.clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


class _HeldoutBundle(_Bundle):
    def __init__(self, origins, dirs, targets, heldout):
        super().__init__(origins, dirs, targets)
        self.heldout = heldout


def test_heldout_psnr_matches_reference():
    """train() with held-out views (optim.py:157-195) against a reference run
    (tests/golden/train_heldout.npz): leaf counts per epoch exact, losses
    within 1e-3, the per-epoch held-out PSNR within 0.02 dB (the trained
    payloads differ by fp32-atomic rounding), and the reference's own final
    tree scored by our heldout_psnr within 1e-3 dB of its score."""
    from paper_2307_15333_b200.octree import LeafPayload, build_dense
    from paper_2307_15333_b200.optim import TrainConfig, heldout_psnr, train
    from paper_2307_15333_b200.scene_io import Camera, load_tree_bytes
    z = np.load(os.path.join(GOLDEN, "train_heldout.npz"))
    cams = [Camera(int(w), int(h), float(f), p) for w, h, f, p in
            zip(z["cam_w"], z["cam_h"], z["cam_f"], z["cam_pose"])]
    bundle = _HeldoutBundle(z["origins"], z["dirs"], z["targets"], list(zip(cams, z["heldout_images"])))
    trainee = build_dense(2, (0.0, 0.0, 0.0), 1.0, 4, LeafPayload(0.3, [0.0] * 12), max_depth=5, device="cuda")
    cfg = TrainConfig(epochs=4, interval=2, tau=0.3, gamma=0.1, batch_size=600, seed=5)
    _, hist = train(trainee, bundle, cfg)
    np.testing.assert_array_equal([h["leaf_count"] for h in hist], z["leaf_count"])
    np.testing.assert_allclose([h["loss"] for h in hist], z["loss"], rtol=1e-3)
    got = np.array([h["psnr"] for h in hist])
    assert np.all(np.isfinite(got))
    np.testing.assert_allclose(got, z["psnr"], atol=0.02)
    ref_tree = load_tree_bytes(z["final_dot1"].tobytes(), device="cuda")
    assert heldout_psnr(ref_tree, bundle, 1.0) == pytest.approx(float(z["final_psnr"]), abs=1e-3)
