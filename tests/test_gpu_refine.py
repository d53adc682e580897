"""GPU parity of the DOT refine pass (prune / sample / canonical rebuild).

Bar: selections (prune parents, sample leaves) equal as sets of pool ids, and
the refined tree's canonical .dot1 bytes identical (sha256) to the
reference's ``save_tree`` of its own calibrated tree -- topology, merged
fp64-mean payloads, split copies and BFS order all at once.
"""

import glob
import hashlib
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CALIB_CASES = sorted(glob.glob(os.path.join(GOLDEN, "calib_*.npz")))


def _setup(z):
    from paper_2307_15333_b200.octree import from_pool_arrays
    from paper_2307_15333_b200.signals import SignalBuffer, SignalTarget
    tree = from_pool_arrays(z, device="cuda")
    tgt = SignalTarget.DENSITY_SIGMA if str(z["target"]) == "sigma" else SignalTarget.RAY_WEIGHT_Q
    buf = SignalBuffer(tree, tgt)
    buf.accumulator.copy_(torch.from_numpy(z["acc"]))
    buf.epoch_rays = 1
    thr = float(z["threshold"])
    return tree, buf, (None if np.isnan(thr) else thr)


@pytest.fixture(params=CALIB_CASES, ids=lambda p: os.path.basename(p)[6:-4])
def case(request):
    return np.load(request.param)


def test_select_prune(case):
    from paper_2307_15333_b200.calibrate import select_prune
    tree, buf, _ = _setup(case)
    np.testing.assert_array_equal(select_prune(tree, buf, float(case["tau"])), case["sel_prune"])


def test_select_sample(case):
    from paper_2307_15333_b200.calibrate import select_sample
    tree, buf, thr = _setup(case)
    got = select_sample(tree, buf, float(case["gamma"]), thr)
    np.testing.assert_array_equal(got, case["sel_sample_pre"])


def test_calibrate_bytes_identical(case, oracle):
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.scene_io import tree_bytes
    tree, buf, thr = _setup(case)
    cfg = CalibrationConfig(tau=float(case["tau"]), gamma=float(case["gamma"]),
                            recursive=bool(case["recursive"]), sample_threshold=thr,
                            check_invariants=True)
    rep = calibrate(tree, buf, cfg)
    assert rep.merges_applied == int(case["merges_applied"])
    assert rep.splits_applied == int(case["splits_applied"])
    assert rep.recursion_rounds == int(case["recursion_rounds"])
    assert rep.leaves_before == int(case["leaves_before"])
    assert rep.leaves_after == int(case["leaves_after"]) == tree.leaf_count
    assert hashlib.sha256(tree_bytes(tree)).hexdigest() == str(case["after_dot1_sha256"])
    # events (built lazily from the device remap): merges in the reference's
    # (round, id) order with the reference's parent and kid pool ids; splits
    # in its order; split kids are canonical ids of the refined tree, i.e. the
    # reference's kid pool ids through the BFS renumbering of its own result
    merges = [(n, k) for kind, n, k in rep.events if kind == "merge"]
    np.testing.assert_array_equal([m[0] for m in merges], case["merge_parents"])
    if merges:
        np.testing.assert_array_equal([m[1] for m in merges], case["child"][case["merge_parents"]])
    splits = [(n, k) for kind, n, k in rep.events if kind == "split"]
    np.testing.assert_array_equal([n for n, _ in splits], case["split_leaves"])
    if splits:
        after = {k[6:]: case[k] for k in case.files if k.startswith("after_")}
        after["free"] = case["after_free"]
        _, new_index = oracle.PoolTree.from_arrays(after).level_order()
        np.testing.assert_array_equal([k for _, k in splits], new_index[case["split_kids"]])
    assert buf.is_fresh() and buf.epoch_rays == 0 and not bool(buf.accumulator.any())


def test_config1_calibrate_with_reference_signal():
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
    from paper_2307_15333_b200.signals import SignalBuffer
    z = np.load(os.path.join(GOLDEN, "config1.npz"))
    tree = load_tree_bytes(z["scene_dot1"].tobytes(), device="cuda")
    buf = SignalBuffer(tree)
    buf.accumulate(z["signal"], z["origins"].shape[0])
    rep = calibrate(tree, buf, CalibrationConfig(tau=0.01, gamma=0.05))
    assert rep.merges_applied == int(z["calib_merges"])
    assert rep.splits_applied == int(z["calib_splits"])
    assert hashlib.sha256(tree_bytes(tree)).hexdigest() == str(z["calib_sha256"])


def test_config1_calibrate_with_own_signal():
    """End to end on device: our backward's signal drives our refine.  The
    selection may only differ from the reference where a signal sits within
    1e-9 relative of tau or of the k-th value (fp32 vs fp64 accumulation)."""
    from paper_2307_15333_b200.calibrate import select_prune, select_sample
    from paper_2307_15333_b200.render import render_and_backprop
    from paper_2307_15333_b200.scene_io import load_tree_bytes
    from paper_2307_15333_b200.signals import SignalBuffer
    z = np.load(os.path.join(GOLDEN, "config1.npz"))
    tree = load_tree_bytes(z["scene_dot1"].tobytes(), device="cuda")
    _, _, sig = render_and_backprop(tree, z["origins"], z["dirs"], z["targets"], 1.0)
    ref = z["signal"]
    near = np.abs(sig - ref) > 1e-12 * np.maximum(np.abs(ref), 1.0)
    buf = SignalBuffer(tree)
    buf.accumulate(sig, 1)
    rbuf = SignalBuffer(tree)
    rbuf.accumulate(ref, 1)
    a, b = select_prune(tree, buf, 0.01), select_prune(tree, rbuf, 0.01)
    assert len(np.setxor1d(a, b)) <= 8 * near.sum()
    a, b = select_sample(tree, buf, 0.05), select_sample(tree, rbuf, 0.05)
    assert len(np.setxor1d(a, b)) <= 2 * near.sum() + 2


@pytest.mark.parametrize("seed,recursive,gamma", [(1, False, 0.1), (2, True, 0.05), (3, False, 0.0)])
def test_large_lognormal_vs_oracle(oracle, seed, recursive, gamma):
    """Config-5-shaped (log-normal(-6, 2) signals, tau 0.01) on a 260k-leaf tree."""
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.octree import build_dense
    from paper_2307_15333_b200.signals import SignalBuffer
    rng = np.random.default_rng(seed)
    tree = build_dense(6, (0.0, 0.0, 0.0), 1.0, 4, seed, max_depth=7, device="cuda")
    leaves = tree.leaf_ids()
    acc = np.zeros(tree.capacity)
    acc[leaves] = rng.lognormal(-6.0, 2.0, leaves.size)
    acc[leaves[::97]] = acc[leaves[5]]  # ties at arbitrary values
    pool = oracle.PoolTree.from_arrays({
        "root_center": tree.center, "half_extent": tree.half_extent, "basis_count": 4,
        "max_depth": 7, "child": tree._child, "parent": tree._parent, "depth": tree._depth,
        "leaf": tree._leaf, "alive": tree._alive, "center": tree._center,
        "sigma": tree.sigma.cpu().numpy(), "sh": tree.sh.cpu().numpy(), "free": []})
    want = oracle.calibrate(pool, acc, 0.01, gamma, recursive)
    buf = SignalBuffer(tree)
    buf.accumulate(acc, 1)
    rep = calibrate(tree, buf, CalibrationConfig(tau=0.01, gamma=gamma, recursive=recursive),
                    events=False)
    assert (rep.merges_applied, rep.splits_applied, rep.recursion_rounds) == \
        (want.merges_applied, want.splits_applied, want.recursion_rounds)
    c = pool.canonical()
    from paper_2307_15333_b200.scene_io import canonical_arrays
    node, leaf, sigma, sh = canonical_arrays(tree)
    np.testing.assert_array_equal(leaf, c["is_leaf"] == 1)
    np.testing.assert_array_equal(np.where(leaf, -1, node), np.where(c["is_leaf"] == 1, -1, c["kids"][:, 0]))
    np.testing.assert_array_equal(sigma, c["sigma"])
    np.testing.assert_array_equal(sh, c["sh"])


def test_refine_render_neutral_split():
    """Sampling copies payloads exactly: renders are unchanged (test_calibrate.py:255-267)."""
    from paper_2307_15333_b200.calibrate import sample
    from paper_2307_15333_b200.render import render_and_backprop, render_rays
    from paper_2307_15333_b200.signals import SignalBuffer
    from helpers import irregular_tree, ray_batch
    tree = irregular_tree(371, 4, depth=2, splits=5, max_depth=4, device="cuda")
    o, d = ray_batch(372, 300)
    buf = SignalBuffer(tree)
    _, _, sig = render_and_backprop(tree, o, d, np.zeros((300, 3)), 0.0)
    buf.accumulate(sig, 300)
    o2, d2 = ray_batch(373, 80)
    before = render_rays(tree, o2, d2, 0.6, early_stop_eps=0.0)
    rep = sample(tree, buf, 0.3)
    assert rep.splits_applied > 0
    assert rep.leaves_after == rep.leaves_before + 7 * rep.splits_applied
    after = render_rays(tree, o2, d2, 0.6, early_stop_eps=0.0)
    np.testing.assert_allclose(after, before, atol=1e-6)
    tree.validate()


def test_rmsprop_row_chunks_equal_full_update():
    """rows=(lo, hi) updates (used to overlap the gradient all-reduce) compose
    to exactly the full update."""
    from paper_2307_15333_b200.optim import RmsPropState, rmsprop_step
    from paper_2307_15333_b200.parallel import chunk_bounds
    from paper_2307_15333_b200.render import render_and_backprop
    from helpers import irregular_tree, ray_batch
    o, d = ray_batch(12, 4000)
    tg = np.random.default_rng(13).uniform(0, 1, (4000, 3))
    trees = [irregular_tree(11, 16, depth=3, splits=20, max_depth=5, device="cuda") for _ in range(2)]
    _, g, _ = render_and_backprop(trees[0], o, d, tg, 1.0)  # one gradient for both updates
    g.generation = trees[1].generation
    outs = []
    for j, tree in enumerate(trees):
        st = RmsPropState(tree)
        if j == 0:
            rmsprop_step(tree, g, st)
        else:
            for lo, hi in chunk_bounds(tree.capacity, 5):
                rmsprop_step(tree, g, st, rows=(lo, hi))
        outs.append((tree.sigma.cpu(), tree.sh.cpu(), st.v_sigma.cpu(), st.v_sh.cpu()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_rmsprop_bit_exact_vs_oracle(oracle):
    from paper_2307_15333_b200.optim import RmsPropState, rmsprop_step
    from paper_2307_15333_b200.render import GradBuffer
    from helpers import irregular_tree
    rng = np.random.default_rng(5)
    tree = irregular_tree(55, 9, depth=2, splits=4, max_depth=4, device="cuda")
    cap, nsh = tree.capacity, 27
    st = RmsPropState(tree)
    v0s = rng.uniform(0, 1e-3, cap)
    v0h = rng.uniform(0, 1e-3, (cap, nsh))
    st.v_sigma.copy_(torch.from_numpy(v0s))
    st.v_sh.copy_(torch.from_numpy(v0h))
    gs = rng.normal(0, 1e-2, cap).astype(np.float32)
    gh = rng.normal(0, 1e-2, (cap, nsh)).astype(np.float32)
    mask = np.zeros(cap, np.uint8)
    mask[tree.leaf_ids()[::2]] = 1
    sig0 = tree.sigma.cpu().numpy().copy()
    sh0 = tree.sh.cpu().numpy().copy()
    rmsprop_step(tree, GradBuffer(gs.astype(np.float64), gh.astype(np.float64), mask, tree.generation), st)
    vs, vh = v0s.copy(), v0h.copy()
    oracle.rmsprop_step(sig0, sh0, vs, vh, gs.astype(np.float64), gh.astype(np.float64),
                        np.nonzero(mask)[0])
    np.testing.assert_array_equal(tree.sigma.cpu().numpy(), sig0)
    np.testing.assert_array_equal(tree.sh.cpu().numpy(), sh0)
    np.testing.assert_array_equal(st.v_sigma.cpu().numpy(), vs)
    np.testing.assert_array_equal(st.v_sh.cpu().numpy(), vh)


def test_config1_end_to_end_deterministic_refine_bytes_identical():
    """Our deterministic backward's signal (bit-identical to the reference's)
    drives our refine: the refined tree is byte-identical to the reference's
    calibrate output on the same scene and rays (configs[0] end to end)."""
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.render import render_and_backprop
    from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
    from paper_2307_15333_b200.signals import SignalBuffer
    z = np.load(os.path.join(GOLDEN, "config1.npz"))
    tree = load_tree_bytes(z["scene_dot1"].tobytes(), device="cuda")
    _, _, sig = render_and_backprop(tree, z["origins"], z["dirs"], z["targets"], 1.0,
                                    deterministic=True)
    buf = SignalBuffer(tree)
    buf.accumulate(sig, z["origins"].shape[0])
    rep = calibrate(tree, buf, CalibrationConfig(tau=0.01, gamma=0.05))
    assert rep.merges_applied == int(z["calib_merges"])
    assert rep.splits_applied == int(z["calib_splits"])
    assert hashlib.sha256(tree_bytes(tree)).hexdigest() == str(z["calib_sha256"])


def test_rmsprop_zero_gradient_rows_bit_exact(oracle):
    """Touched rows whose gradients are exactly zero (leaves touched only past
    the early-termination cut) take the kernel's shortcut paths; v must still
    decay and theta stay put, bit for bit like the reference update."""
    from paper_2307_15333_b200.optim import RmsPropState, rmsprop_step
    from paper_2307_15333_b200.render import GradBuffer
    from helpers import irregular_tree
    rng = np.random.default_rng(8)
    tree = irregular_tree(56, 16, depth=2, splits=4, max_depth=4, device="cuda")
    cap, nsh = tree.capacity, 48
    st = RmsPropState(tree)
    v0s = rng.uniform(0, 1e-3, cap)
    v0h = rng.uniform(0, 1e-3, (cap, nsh))
    st.v_sigma.copy_(torch.from_numpy(v0s))
    st.v_sh.copy_(torch.from_numpy(v0h))
    gs = rng.normal(0, 1e-2, cap).astype(np.float32)
    gh = rng.normal(0, 1e-2, (cap, nsh)).astype(np.float32)
    rows = np.arange(cap)
    gs[rows % 3 == 0] = 0.0
    gh[rows % 3 == 0] = 0.0                   # whole rows zero
    gh[rows % 3 == 1, 4:8] = 0.0              # single zero quads
    gh[rows % 5 == 0, 12] = -0.0
    mask = np.zeros(cap, np.uint8)
    mask[tree.leaf_ids()] = 1
    sig0 = tree.sigma.cpu().numpy().copy()
    sh0 = tree.sh.cpu().numpy().copy()
    rmsprop_step(tree, GradBuffer(gs.astype(np.float64), gh.astype(np.float64), mask, tree.generation), st)
    vs, vh = v0s.copy(), v0h.copy()
    oracle.rmsprop_step(sig0, sh0, vs, vh, gs.astype(np.float64), gh.astype(np.float64), np.nonzero(mask)[0])
    np.testing.assert_array_equal(tree.sigma.cpu().numpy(), sig0)
    np.testing.assert_array_equal(tree.sh.cpu().numpy(), sh0)
    np.testing.assert_array_equal(st.v_sigma.cpu().numpy(), vs)
    np.testing.assert_array_equal(st.v_sh.cpu().numpy(), vh)


@pytest.mark.parametrize("B", [16, 1])
def test_rmsprop_f32_state_within_tolerance(oracle, B):
    """The opt-in f32 second-moment update (state_dtype=float32) against the
    reference's f64 update (oracle): payloads and state within 1e-6 relative,
    zero-gradient rows still decay v only, untouched rows untouched."""
    from paper_2307_15333_b200.optim import RmsPropState, rmsprop_step
    from paper_2307_15333_b200.render import GradBuffer
    from helpers import irregular_tree
    rng = np.random.default_rng(9 + B)
    tree = irregular_tree(57, B, depth=2, splits=4, max_depth=4, device="cuda")
    cap, nsh = tree.capacity, 3 * B
    st = RmsPropState(tree, state_dtype=torch.float32)
    v0s = rng.uniform(0, 1e-3, cap).astype(np.float32)
    v0h = rng.uniform(0, 1e-3, (cap, nsh)).astype(np.float32)
    st.v_sigma.copy_(torch.from_numpy(v0s))
    st.v_sh.copy_(torch.from_numpy(v0h))
    gs = rng.normal(0, 1e-2, cap).astype(np.float32)
    gh = rng.normal(0, 1e-2, (cap, nsh)).astype(np.float32)
    gs[::3] = 0.0
    gh[::3] = 0.0
    mask = (rng.uniform(size=cap) < 0.7).astype(np.uint8)
    sig0 = tree.sigma.cpu().numpy().copy()
    sh0 = tree.sh.cpu().numpy().copy()
    for _ in range(2):
        rmsprop_step(tree, GradBuffer(gs, gh, mask, tree.generation), st)
    vs, vh = v0s.astype(np.float64), v0h.astype(np.float64)
    es, eh = sig0.copy(), sh0.copy()
    for _ in range(2):
        oracle.rmsprop_step(es, eh, vs, vh, gs.astype(np.float64), gh.astype(np.float64), np.nonzero(mask)[0])
    np.testing.assert_allclose(tree.sigma.cpu().numpy(), es, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(tree.sh.cpu().numpy(), eh, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(st.v_sigma.cpu().numpy(), vs, rtol=1e-6, atol=0)
    np.testing.assert_allclose(st.v_sh.cpu().numpy(), vh, rtol=1e-6, atol=0)
    untouched = mask == 0
    np.testing.assert_array_equal(st.v_sh.cpu().numpy()[untouched], v0h[untouched])
    np.testing.assert_array_equal(tree.sh.cpu().numpy()[untouched], sh0[untouched])
