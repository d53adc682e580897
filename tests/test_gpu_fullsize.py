"""Parity at BASELINE.json's full sizes, through the production paths, against
the pinned oracle (tests/test_oracle_golden.py):

* configs[1]: one 2^20-ray random training batch of the 100-view pool
  (ray_index + coherence plan + learned warp schedule, and the bench's
  ranked-pool plan with cost regrouping): loss, dsigma, dSH (scale-aware
  1e-4 / 1e-3), touched set equal, signal to f64-atomic rounding; the
  deterministic path's signal bit-equal to the reference's.
* configs[2]: one 800x800 view through render_rays on Camera.rays()
  (segments bit-exact, rgb / T_final / weight sum / depth within 1e-4 /
  1e-3) and through render_views (in-kernel rays).
* configs[3]: one 2^21-ray batch of the depth-10 configs[3] scene.
* configs[4]: the 16M-leaf refine -- topology and payload bit-exact
  against the oracle's vectorised restatement of calibrate (prune, LIFO
  splits, canonical BFS order).
Plus the size-independent properties (weight conservation, determinism,
tree validity) the oracle cannot reach cheaply.
"""

import numpy as np
import pytest
import torch

from helpers import assert_grads_close

pytestmark = pytest.mark.gpu

ATOL, RTOL = 1e-4, 1e-3


@pytest.fixture(scope="module")
def scene():
    from paper_2307_15333_b200 import scenes
    return scenes.config2_scene(device="cuda")


@pytest.fixture(scope="module")
def pool(scene):
    import bench
    return bench.build_training_pool(scene, torch.device("cuda"))


def _view_rays(scene, seed=4, i=0):
    import bench
    from paper_2307_15333_b200 import scenes
    focal, poses = scenes.hemisphere_cameras(8, 800, 800, 4.03, seed=seed)
    return bench.view_rays_torch(focal, poses[i], torch.device("cuda"))


def _batch_vs_oracle(oracle, tree, o, d, t, idx):
    """Production backward (ray_index into the resident pool, coherence plan,
    learned schedule warmed by two earlier batches) vs the oracle on the
    gathered host batch; deterministic path's signal bit-exact."""
    from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop
    n = int(idx.numel())
    for k in range(2):  # populate the learned warp-schedule table first
        render_and_backprop(tree, o, d, t, 1.0, ray_index=idx.roll(1000 * (k + 1)))
    ws = BackpropWorkspace.for_tree(tree)
    loss, g, sig = render_and_backprop(tree, o, d, t, 1.0, ray_index=idx, workspace=ws)
    oh, dh, th = (x[idx].cpu().numpy() for x in (o, d, t))
    tree._host()
    r_loss, r_g, r_sig = oracle.render_and_backprop(tree, oh, dh, th, 1.0)
    assert float(loss) == pytest.approx(r_loss, rel=RTOL, abs=ATOL)
    touched = torch.nonzero(g.touched_mask).reshape(-1).cpu().numpy()
    np.testing.assert_array_equal(touched, r_g.touched)
    assert_grads_close(g.dsigma.cpu().numpy()[touched], r_g.dsigma[touched], what="dsigma")
    assert_grads_close(g.dsh.cpu().numpy()[touched], r_g.dsh[touched], what="dsh")
    np.testing.assert_allclose(sig.cpu().numpy(), r_sig, rtol=1e-12, atol=1e-15)
    # the bench's training path: the pool ranked by its 62-bit keys, the
    # batch planned by the cooperative kernel (key order regrouped by cost in
    # 128-ray windows, warps launched longest first)
    from paper_2307_15333_b200.render import plan_batch, pool_rank, ray_costs
    pr = pool_rank(tree, o, d)
    plan = plan_batch(tree, o, d, idx, rank=pr, costs=ray_costs(tree, o, d))
    assert plan.warp_order is not None and torch.equal(torch.sort(plan.idx).values, torch.sort(idx).values)
    ws2 = BackpropWorkspace.for_tree(tree)
    loss2, g2, sig2 = render_and_backprop(tree, o, d, t, 1.0, ray_index=idx, workspace=ws2, plan=plan)
    del pr, plan
    assert float(loss2) == pytest.approx(r_loss, rel=RTOL, abs=ATOL)
    np.testing.assert_array_equal(torch.nonzero(g2.touched_mask).reshape(-1).cpu().numpy(), r_g.touched)
    assert_grads_close(g2.dsigma.cpu().numpy()[touched], r_g.dsigma[touched], what="dsigma (ranked plan)")
    assert_grads_close(g2.dsh.cpu().numpy()[touched], r_g.dsh[touched], what="dsh (ranked plan)")
    np.testing.assert_allclose(sig2.cpu().numpy(), r_sig, rtol=1e-12, atol=1e-15)
    # the deterministic reduction: the reference's serial order, bit for bit
    ws.zero_()
    _, gd, sd = render_and_backprop(tree, o, d, t, 1.0, ray_index=idx, workspace=ws, deterministic=True)
    np.testing.assert_array_equal(sd.cpu().numpy(), r_sig)
    assert torch.equal(gd.touched_mask.cpu(), torch.from_numpy((np.bincount(r_g.touched, minlength=tree.capacity) > 0)
                                                                 .astype(np.uint8)))
    return n


def test_config2_batch_vs_oracle(oracle, scene, pool):
    """configs[1]: a full 2^20-ray training batch against the reference's algorithm."""
    o, d, t = pool
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    idx = torch.randperm(o.shape[0], generator=g, device="cuda")[: 1 << 20]
    assert _batch_vs_oracle(oracle, scene, o, d, t, idx) == 1 << 20


def test_config3_view_vs_oracle(oracle, scene):
    """configs[2]: one 800x800 view, exact rays and in-kernel rays."""
    from paper_2307_15333_b200 import scenes
    from paper_2307_15333_b200.render import render_rays, render_views, segment_batch
    from paper_2307_15333_b200.scene_io import Camera
    focal, poses = scenes.hemisphere_cameras(200, 800, 800, 4.03, seed=4)
    cam = Camera(800, 800, focal, poses[17])
    o, d = cam.rays()
    scene._host()
    want_seg = oracle.segment_batch(scene, o, d)
    for a, b in zip(segment_batch(scene, o, d), want_seg):
        np.testing.assert_array_equal(a, b)
    r_rgb, r_tf, r_ws = oracle.render_rays(scene, o, d, 1.0, 1e-4, return_aux=True)
    r_depth = oracle.render_depth(scene, o, d, 1e-4)
    rgb, tf, ws, depth = render_rays(scene, o, d, 1.0, 1e-4, return_aux=True, return_depth=True)
    np.testing.assert_allclose(rgb, r_rgb, atol=ATOL, rtol=RTOL)
    np.testing.assert_allclose(tf, r_tf, atol=ATOL, rtol=RTOL)
    np.testing.assert_allclose(ws, r_ws, atol=ATOL, rtol=RTOL)
    np.testing.assert_allclose(depth, r_depth, atol=ATOL, rtol=RTOL)
    img, tfv, depv = render_views(scene, [cam], 1.0, 1e-4, return_aux=True)
    np.testing.assert_allclose(img[0].reshape(-1, 3).cpu().numpy(), r_rgb, atol=ATOL, rtol=RTOL)
    np.testing.assert_allclose(tfv[0].reshape(-1).cpu().numpy(), r_tf, atol=ATOL, rtol=RTOL)
    np.testing.assert_allclose(depv[0].reshape(-1).cpu().numpy(), r_depth, atol=ATOL, rtol=RTOL)


def test_config4_batch_vs_oracle(oracle):
    """configs[3]: one 2^21-ray batch of the depth-10 scene (8.5M leaves,
    1920x1080 ring views) against the reference's algorithm."""
    import bench
    wl = bench.workloads()["c4"]
    tree = wl.scene(torch.device("cuda"))
    o, d, t = bench.build_training_pool(tree, torch.device("cuda"), wl)
    g = torch.Generator(device="cuda")
    g.manual_seed(4)
    idx = torch.randperm(o.shape[0], generator=g, device="cuda")[: 1 << 21]
    assert _batch_vs_oracle(oracle, tree, o, d, t, idx) == 1 << 21
    del o, d, t, tree
    torch.cuda.empty_cache()


def _canonical_expect(pool):
    order, new_index = pool.level_order()
    leaf = pool._leaf[order] == 1
    node = np.where(leaf, ~np.arange(order.size), new_index[pool._child[order, 0]]).astype(np.int32)
    return order, leaf, node


def test_config5_refine_bit_exact(oracle):
    """configs[4]: the 16M-leaf refine (log-normal(-6, 2) signals, tau 0.01,
    gamma 0.1): node table, leaf sigma and every SH coefficient of the
    refined canonical tree equal the oracle's, bit for bit."""
    import bench
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.signals import SignalBuffer
    tree = bench.config5_tree(torch.device("cuda"))
    topo = tree.topology()
    node0 = topo.node
    leaf0 = node0 < 0
    g = torch.Generator(device="cuda")
    g.manual_seed(55)
    acc = torch.zeros(node0.shape[0], dtype=torch.float64, device="cuda")
    acc[leaf0] = torch.exp(-6.0 + 2.0 * torch.randn(int(leaf0.sum()), generator=g, device="cuda",
                                                    dtype=torch.float64))
    pool = oracle.PoolTree.from_canonical_words(tree.center, tree.half_extent, 16, tree.max_depth,
                                               node0.cpu().numpy(), tree.sigma.cpu().numpy(),
                                               tree.sh.cpu().numpy())
    acc_h = acc.cpu().numpy()
    buf = SignalBuffer(tree)
    buf.accumulator.copy_(acc)
    rep = calibrate(tree, buf, CalibrationConfig(tau=0.01, gamma=0.10))
    ref = oracle.calibrate(pool, acc_h, 0.01, 0.10, fast=True)
    assert rep.leaves_before > 15_000_000
    assert (rep.merges_applied, rep.splits_applied, rep.leaves_after) == (
        ref.merges_applied, ref.splits_applied, ref.leaves_after)
    order, leaf, node = _canonical_expect(pool)
    got_node = tree.topology().node.cpu().numpy()
    np.testing.assert_array_equal(got_node, node)
    got_sig = tree.sigma.cpu().numpy()
    np.testing.assert_array_equal(got_sig[leaf], pool.sigma[order[leaf]])
    rows = np.nonzero(leaf)[0]
    for lo in range(0, rows.size, 1 << 22):  # 48 floats per row: compare in slabs
        r = rows[lo:lo + (1 << 22)]
        np.testing.assert_array_equal(tree.sh[torch.from_numpy(r).cuda()].cpu().numpy(), pool.sh[order[r]])


def test_config2_view_weight_conservation(scene):
    """sum_i T_i Q_i + T_final = 1 for every pixel of an 800x800 view (eps 0
    and 1e-4), and T_final in [0, 1]."""
    from paper_2307_15333_b200.render import render_rays
    o, d = _view_rays(scene)
    for eps in (0.0, 1e-4):
        rgb, tf, ws = render_rays(scene, o, d, 1.0, eps, return_aux=True)
        assert float((ws - 1.0).abs().max()) < 1e-5
        assert float(tf.min()) >= 0.0 and float(tf.max()) <= 1.0
        assert torch.isfinite(rgb).all()


def test_config2_full_batch_deterministic_and_atomic_agree(scene, pool):
    """A 2^20-ray training batch: the deterministic path is bit-identical run
    to run; the default (atomic, learned-schedule) path agrees with it within
    the float tolerance and has the identical touched set."""
    from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop
    o, d, t = pool
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    idx = torch.randperm(o.shape[0], generator=g, device="cuda")[: 1 << 20]
    outs = []
    for _ in range(2):
        ws = BackpropWorkspace.for_tree(scene)
        loss, gr, sig = render_and_backprop(scene, o, d, t, 1.0, ray_index=idx, workspace=ws,
                                            deterministic=True)
        outs.append((float(loss), gr.dsigma.clone(), gr.dsh.clone(), sig.clone(), gr.touched_mask.clone()))
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1:], outs[1][1:]):
        assert torch.equal(a, b)
    for _ in range(3):  # warm the schedule table, then compare
        ws = BackpropWorkspace.for_tree(scene)
        loss, gr, sig = render_and_backprop(scene, o, d, t, 1.0, ray_index=idx, workspace=ws)
    assert float(loss) == pytest.approx(outs[0][0], rel=1e-9)
    touched = gr.touched_mask.bool()
    assert_grads_close(gr.dsigma[touched].cpu().numpy(), outs[0][1][touched].cpu().numpy(), what="dsigma")
    assert_grads_close(gr.dsh[touched].cpu().numpy(), outs[0][2][touched].cpu().numpy(), what="dsh")
    torch.testing.assert_close(sig, outs[0][3], atol=1e-9, rtol=1e-9)
    assert torch.equal(gr.touched_mask, outs[0][4])


def test_config5_refine_structure():
    """configs[4] refine (16M leaves): the result is a valid canonical octree
    with L = 7I + 1 and the counts the plan predicted; refining twice more
    keeps it valid."""
    import bench
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.signals import SignalBuffer
    tree = bench.config5_tree(torch.device("cuda"))
    n0, l0 = tree.topology().n_nodes, tree.leaf_count
    buf = SignalBuffer(tree)
    g = torch.Generator(device="cuda")
    g.manual_seed(55)
    node = tree.topology().node
    leaf = node < 0
    acc = torch.zeros(node.shape[0], dtype=torch.float64, device="cuda")
    acc[leaf] = torch.exp(-6.0 + 2.0 * torch.randn(int(leaf.sum()), generator=g, device="cuda",
                                                  dtype=torch.float64))
    buf.accumulator.copy_(acc)
    rep = calibrate(tree, buf, CalibrationConfig(tau=0.01, gamma=0.10), events=False)
    assert rep.leaves_before == l0
    assert tree.leaf_count == l0 - 7 * rep.merges_applied + 7 * rep.splits_applied
    assert tree.topology().n_nodes == n0 - 8 * rep.merges_applied + 8 * rep.splits_applied
    w = tree.topology().node
    internal = w[w >= 0]
    assert int((w < 0).sum()) == 7 * int(internal.numel()) + 1
    assert int(internal.max()) + 8 <= w.shape[0] and int(internal.min()) >= 1
    # every non-root node is the child of exactly one internal node
    kids = (internal[:, None] + torch.arange(8, device="cuda")).reshape(-1)
    assert int(kids.numel()) == w.shape[0] - 1
    assert torch.equal(torch.sort(kids).values, torch.arange(1, w.shape[0], device="cuda", dtype=kids.dtype))
    # leaves carry their own pool row (canonical: pool id == BFS index)
    lid = torch.nonzero(w < 0).reshape(-1)
    assert torch.equal((~w[lid]).to(torch.int64), lid)
