"""Pin the CPU oracle to the reference: every golden fixture (outputs of
octrf itself, tests/golden/make_golden.py) must be reproduced -- bit-exactly
for segments, rgb, gradients, signal, selections and refined pools."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN

RENDER = sorted(glob.glob(os.path.join(GOLDEN, "render_*.npz")))
CALIB = sorted(glob.glob(os.path.join(GOLDEN, "calib_*.npz")))


@pytest.mark.parametrize("path", RENDER, ids=lambda p: os.path.basename(p)[7:-4])
def test_oracle_render_golden(oracle, path):
    z = np.load(path)
    t = oracle.PoolTree.from_arrays(z)
    tn, tf = float(z["t_near"]), float(z["t_far"])
    off, leaf, tt, dl = oracle.segment_batch(t, z["origins"], z["dirs"], tn, tf)
    np.testing.assert_array_equal(off, z["seg_offsets"])
    np.testing.assert_array_equal(leaf, z["seg_leaf"])
    np.testing.assert_array_equal(tt, z["seg_t"])
    np.testing.assert_array_equal(dl, z["seg_delta"])
    for tag, eps in (("eps", 1e-4), ("noeps", 0.0)):
        rgb, tfin, wsum = oracle.render_rays(t, z["origins"], z["dirs"], z["bg"], eps, tn, tf,
                                             return_aux=True)
        np.testing.assert_array_equal(rgb, z[f"rgb_{tag}"])
        np.testing.assert_array_equal(tfin, z[f"tfin_{tag}"])
        np.testing.assert_array_equal(wsum, z[f"wsum_{tag}"])
        loss, g, sig = oracle.render_and_backprop(t, z["origins"], z["dirs"], z["targets"], z["bg"],
                                                  eps, tn, tf)
        assert loss == float(z[f"loss_{tag}"])
        np.testing.assert_array_equal(g.dsigma, z[f"dsigma_{tag}"])
        np.testing.assert_array_equal(g.dsh, z[f"dsh_{tag}"])
        np.testing.assert_array_equal(g.touched, z[f"touched_{tag}"])
        np.testing.assert_array_equal(sig, z[f"signal_{tag}"])


@pytest.mark.parametrize("path", CALIB, ids=lambda p: os.path.basename(p)[6:-4])
def test_oracle_calibrate_golden(oracle, path):
    z = np.load(path)
    t = oracle.PoolTree.from_arrays(z)
    thr = float(z["threshold"])
    thr = None if np.isnan(thr) else thr
    use_sigma = str(z["target"]) == "sigma"
    np.testing.assert_array_equal(oracle.select_prune(t, z["acc"], float(z["tau"]), use_sigma),
                                  z["sel_prune"])
    np.testing.assert_array_equal(
        oracle.select_sample(t, z["acc"], float(z["gamma"]), thr, use_sigma), z["sel_sample_pre"])
    r = oracle.calibrate(t, z["acc"], float(z["tau"]), float(z["gamma"]), bool(z["recursive"]),
                         thr, use_sigma)
    assert (r.merges_applied, r.splits_applied, r.recursion_rounds, r.leaves_after) == (
        int(z["merges_applied"]), int(z["splits_applied"]), int(z["recursion_rounds"]),
        int(z["leaves_after"]))
    for k in ("child", "parent", "depth", "leaf", "alive", "center"):
        np.testing.assert_array_equal(getattr(t, "_" + k), z["after_" + k])
    np.testing.assert_array_equal(t.sigma, z["after_sigma"])
    np.testing.assert_array_equal(t.sh, z["after_sh"])
    np.testing.assert_array_equal(np.asarray(t._free), z["after_free"])
    splits = [n for kind, n, _ in r.events if kind == "split"]
    np.testing.assert_array_equal(splits, z["split_leaves"])


def test_oracle_config1_golden(oracle):
    from paper_2307_15333_b200.scene_io import load_tree_bytes
    z = np.load(os.path.join(GOLDEN, "config1.npz"))
    tree = load_tree_bytes(z["scene_dot1"].tobytes(), device="cpu")
    off, leaf, t, d = oracle.segment_batch(tree, z["origins"], z["dirs"])
    np.testing.assert_array_equal(off, z["seg_offsets"])
    np.testing.assert_array_equal(leaf, z["seg_leaf"])
    np.testing.assert_array_equal(t, z["seg_t"])
    np.testing.assert_array_equal(d, z["seg_delta"])
    rgb = oracle.render_rays(tree, z["origins"], z["dirs"], 1.0)
    np.testing.assert_array_equal(rgb, z["rgb"])
    loss, g, sig = oracle.render_and_backprop(tree, z["origins"], z["dirs"], z["targets"], 1.0)
    assert loss == float(z["loss"])
    np.testing.assert_array_equal(g.touched, z["touched"])
    np.testing.assert_array_equal(g.dsigma[g.touched], z["dsigma_touched"])
    np.testing.assert_array_equal(sig, z["signal"])


def test_oracle_remap_golden(oracle):
    """RmsPropState.remap restatement vs the reference across 3 prune rounds."""
    z = np.load(os.path.join(GOLDEN, "optim_remap.npz"))
    t = oracle.PoolTree.from_arrays(z)
    r = oracle.calibrate(t, z["acc"], float(z["tau"]), float(z["gamma"]), True)
    assert r.recursion_rounds == int(z["rounds"])
    vs, vh = oracle.rmsprop_remap(z["v_sigma"].copy(), z["v_sh"].copy(), r.events, t.capacity)
    c = t.canonical()
    leaf = z["canon_is_leaf"]
    np.testing.assert_array_equal(c["is_leaf"] == 1, leaf)
    np.testing.assert_array_equal(vs[c["order"]][leaf], z["canon_v_sigma"][leaf])
    np.testing.assert_array_equal(vh[c["order"]][leaf], z["canon_v_sh"][leaf])


@pytest.mark.parametrize("path", CALIB, ids=lambda p: os.path.basename(p)[6:-4])
def test_oracle_fast_calibrate_golden(oracle, path):
    """The vectorised oracle (used at configs[4]'s 16M leaves) leaves the
    reference's exact pool behind: slots, free list, payload, split ids."""
    z = np.load(path)
    t = oracle.PoolTree.from_arrays(z)
    thr = float(z["threshold"])
    thr = None if np.isnan(thr) else thr
    r = oracle.calibrate(t, z["acc"], float(z["tau"]), float(z["gamma"]), bool(z["recursive"]),
                         thr, str(z["target"]) == "sigma", fast=True)
    assert (r.merges_applied, r.splits_applied, r.recursion_rounds, r.leaves_after) == (
        int(z["merges_applied"]), int(z["splits_applied"]), int(z["recursion_rounds"]),
        int(z["leaves_after"]))
    for k in ("child", "parent", "depth", "leaf", "alive", "center"):
        np.testing.assert_array_equal(getattr(t, "_" + k), z["after_" + k])
    np.testing.assert_array_equal(t.sigma, z["after_sigma"])
    np.testing.assert_array_equal(t.sh, z["after_sh"])
    np.testing.assert_array_equal(np.asarray(t._free), z["after_free"])
    np.testing.assert_array_equal(r.sample_selection, z["split_leaves"])
    np.testing.assert_array_equal(r.split_kids, z["split_kids"])
    if r.merge_rounds:
        np.testing.assert_array_equal(np.concatenate([p for p, _ in r.merge_rounds]), z["merge_parents"])


def test_oracle_fast_load_equals_sequential(oracle):
    """from_canonical_words == from_canonical (load_tree's BFS split loop),
    and a fast calibrate that grows the pool == the sequential one."""
    rng = np.random.default_rng(5)
    t = oracle.PoolTree((0.1, -0.2, 0.3), 1.5, 4, 5, 8)
    t.sigma[0] = 1.0
    for _ in range(60):
        leaves = t.leaf_ids()
        ok = leaves[t._depth[leaves] < 4]
        kids = t.split_leaf(int(rng.choice(ok)))
        t.sigma[kids] = rng.uniform(0, 3, 8)
        t.sh[kids] = rng.normal(0, 1, (8, 12))
    c = t.canonical()
    node = np.where(c["is_leaf"] == 1, ~np.arange(c["is_leaf"].size), c["kids"][:, 0])
    args = ((0.1, -0.2, 0.3), 1.5, 4, 5)
    a = oracle.PoolTree.from_canonical(*args, c["kids"], c["is_leaf"], c["sigma"], c["sh"])
    b = oracle.PoolTree.from_canonical_words(*args, node, c["sigma"], c["sh"])
    for k in ("_child", "_parent", "_depth", "_leaf", "_alive", "_center", "sigma", "sh"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k))
    assert a._free == b._free and a.leaf_count == b.leaf_count
    acc = np.where(a._leaf == 1, rng.lognormal(-2, 2, a.capacity), 0.0)
    ra = oracle.calibrate(a, acc, 0.05, 0.5)
    rb = oracle.calibrate(b, acc, 0.05, 0.5, fast=True)
    assert b.capacity > a.capacity // 2 and (ra.splits_applied, ra.merges_applied) == (rb.splits_applied, rb.merges_applied)
    for k in ("_child", "_parent", "_depth", "_leaf", "_alive", "_center", "sigma", "sh"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k))
    assert a._free == b._free


@pytest.mark.parametrize("path", RENDER, ids=lambda p: os.path.basename(p)[7:-4])
def test_oracle_weights_definition(oracle, path):
    """oracle_weights (depth, per-leaf sum / max of T_i Q_i -- extras with no
    reference counterpart) restated in Python over the reference's segment
    lists, and tied to the reference's own outputs: summed over leaves the
    weight sum equals sum_rays (weight sum - T_final) of render_rays."""
    import math
    z = np.load(path)
    t = oracle.PoolTree.from_arrays(z)
    tn, tf = float(z["t_near"]), float(z["t_far"])
    for tag, eps in (("eps", 1e-4), ("noeps", 0.0)):
        depth, wsum, wmax = oracle.render_weights(t, z["origins"], z["dirs"], eps, tn, tf)
        off, leaf, st, sd = z["seg_offsets"], z["seg_leaf"], z["seg_t"], z["seg_delta"]
        want_d = np.zeros(off.size - 1)
        want_s = np.zeros(t.capacity)
        want_m = np.zeros(t.capacity)
        for r in range(off.size - 1):
            trans = 1.0
            for s in range(off[r], off[r + 1]):
                a = math.exp(-float(t.sigma[leaf[s]]) * sd[s])
                w = trans * (1.0 - a)
                want_d[r] += w * (st[s] + 0.5 * sd[s])
                want_s[leaf[s]] += w
                want_m[leaf[s]] = max(want_m[leaf[s]], w)
                trans *= a
                if eps > 0.0 and trans < eps:
                    break
        np.testing.assert_allclose(depth, want_d, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(wsum, want_s, rtol=1e-12, atol=1e-15)
        np.testing.assert_array_equal(wmax, want_m)
        ref = (z[f"wsum_{tag}"] - z[f"tfin_{tag}"]).sum()
        assert wsum.sum() == pytest.approx(ref, rel=1e-12, abs=1e-12)
