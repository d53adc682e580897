"""Size-independent properties of the CUDA render / backward path, mirroring
the reference's own property tests: weight conservation
(tests/test_render.py:184-190), render-neutral subdivision and merging
(test_render.py:192-213), and finite-difference gradients
(tests/test_acceptance.py:147-186, test_gradients.py:45-84)."""

import numpy as np
import pytest
import torch

from helpers import irregular_tree, ray_batch

pytestmark = pytest.mark.gpu


def test_weight_conservation():
    """sum_i T_i Q_i + T_final == 1 with no early termination."""
    from paper_2307_15333_b200.render import render_rays
    tree = irregular_tree(41, 1, depth=2, splits=10, max_depth=4, sigma_range=(0.0, 20.0), device="cuda")
    o, d = ray_batch(42, 200)
    _rgb, _tfin, wsum = render_rays(tree, o, d, 0.0, early_stop_eps=0.0, return_aux=True)
    np.testing.assert_allclose(wsum, 1.0, atol=1e-5)


def test_subdivision_is_render_neutral():
    """Splitting a leaf copies its payload to 8 children: same image."""
    from paper_2307_15333_b200.render import render_rays
    tree = irregular_tree(51, 4, depth=2, splits=6, max_depth=4, device="cuda")
    o, d = ray_batch(52, 300)
    before = render_rays(tree, o, d, 0.2, early_stop_eps=0.0)
    rng = np.random.default_rng(53)
    for _ in range(5):
        leaves = tree.leaf_ids()
        ok = leaves[tree._depth[leaves] < tree.max_depth]
        tree.split_leaf(int(rng.choice(ok)))
    after = render_rays(tree, o, d, 0.2, early_stop_eps=0.0)
    np.testing.assert_allclose(after, before, atol=1e-6)


def test_merging_constant_region_is_render_neutral():
    from paper_2307_15333_b200.octree import LeafPayload, build_dense
    from paper_2307_15333_b200.render import render_rays
    tree = build_dense(2, (0.0, 0.0, 0.0), 1.0, 1, LeafPayload(0.7, [0.4, -0.1, 0.2]), device="cuda")
    o, d = ray_batch(54, 60)
    before = render_rays(tree, o, d, 1.0, early_stop_eps=0.0)
    for child in tree.children(0):
        tree.merge_children(int(child))
    tree.merge_children(0)
    assert tree.stats().leaf_count == 1
    after = render_rays(tree, o, d, 1.0, early_stop_eps=0.0)
    np.testing.assert_allclose(after, before, atol=1e-6)


def _loss(tree, o, d, tgt, bg):
    from paper_2307_15333_b200.render import render_and_backprop
    loss, _g, _s = render_and_backprop(tree, o, d, tgt, bg, early_stop_eps=0.0)
    return float(loss)


@pytest.mark.parametrize("B", [1, 4])
def test_finite_difference_gradients(B):
    """Analytic dL/dsigma and dL/dSH of the fused backward vs central
    differences of the fused forward's loss, on the leaves with the largest
    gradients (sigma and SH are f32 on the device: the step actually taken
    is read back, not assumed)."""
    from paper_2307_15333_b200.render import render_and_backprop
    tree = irregular_tree(61 + B, B, depth=2, splits=8, max_depth=4, sigma_range=(0.2, 4.0), device="cuda")
    o, d = ray_batch(62, 256, miss_fraction=0.0)
    tgt = np.random.default_rng(63).uniform(0.0, 1.0, (256, 3))
    bg = 0.3
    _loss0, g, _sig = render_and_backprop(tree, o, d, tgt, bg, early_stop_eps=0.0)
    ds, dsh = np.asarray(g.dsigma), np.asarray(g.dsh)
    order = np.argsort(-np.abs(ds))[:6]
    for leaf in order:
        leaf = int(leaf)
        old = float(tree.sigma[leaf])
        h = 1e-2 * max(1.0, abs(old))
        tree.sigma[leaf] = old + h
        hp = float(tree.sigma[leaf]) - old
        lp = _loss(tree, o, d, tgt, bg)
        tree.sigma[leaf] = old - h
        hm = old - float(tree.sigma[leaf])
        lm = _loss(tree, o, d, tgt, bg)
        tree.sigma[leaf] = old
        fd = (lp - lm) / (hp + hm)
        assert fd == pytest.approx(ds[leaf], rel=2e-2, abs=1e-3 * np.abs(ds).max())
    flat = np.abs(dsh[:, : 3 * B])
    rows, cols = np.unravel_index(np.argsort(-flat, axis=None)[:6], flat.shape)
    for leaf, k in zip(rows.tolist(), cols.tolist()):
        old = float(tree.sh[leaf, k])
        h = 1e-2
        tree.sh[leaf, k] = old + h
        hp = float(tree.sh[leaf, k]) - old
        lp = _loss(tree, o, d, tgt, bg)
        tree.sh[leaf, k] = old - h
        hm = old - float(tree.sh[leaf, k])
        lm = _loss(tree, o, d, tgt, bg)
        tree.sh[leaf, k] = old
        fd = (lp - lm) / (hp + hm)
        assert fd == pytest.approx(dsh[leaf, k], rel=2e-2, abs=1e-3 * flat.max())
    torch.cuda.synchronize()


def _clip(o, d, c, h):
    """Slab clip of a ray against the root cube (independent restatement)."""
    t0, t1 = 0.0, np.inf
    for a in range(3):
        if d[a] == 0.0:
            if not (c[a] - h <= o[a] < c[a] + h):
                return None
            continue
        ta, tb = (c[a] - h - o[a]) / d[a], (c[a] + h - o[a]) / d[a]
        t0, t1 = max(t0, min(ta, tb)), min(t1, max(ta, tb))
    return (t0, t1) if t1 > t0 else None


@pytest.mark.parametrize("seed,center,half", [(11, (0.0, 0.0, 0.0), 1.0), (21, (0.3, -0.2, 0.05), 1.7)])
def test_segments_contiguous_cover_chord_and_lie_in_their_leaf(seed, center, half):
    """segment_batch on the device: t_{s+1} == t_s + delta_s bit for bit, the
    segments cover the clipped chord, and points inside each segment locate
    (host point location) to the segment's leaf."""
    from paper_2307_15333_b200.render import segment_batch
    tree = irregular_tree(seed, 1, depth=2, splits=12, max_depth=4, center=center, half=half, device="cuda")
    o, d = ray_batch(seed + 1, 128, center=center, half=half, miss_fraction=0.1)
    offsets, leaf, t, delta = segment_batch(tree, o, d)
    for r in range(len(o)):
        lo, hi = int(offsets[r]), int(offsets[r + 1])
        span = _clip(o[r], d[r], np.asarray(center), half)
        if lo == hi:
            assert span is None or span[1] - span[0] < 1e-9
            continue
        tt, dd = t[lo:hi], delta[lo:hi]
        np.testing.assert_array_equal(tt[1:], tt[:-1] + dd[:-1])
        assert (dd > 0).all()
        assert tt[0] == pytest.approx(span[0], abs=1e-12)
        assert tt[-1] + dd[-1] == pytest.approx(span[1], abs=1e-12)
        for s in range(lo, hi):
            for frac in (0.25, 0.5, 0.75):
                p = o[r] + (t[s] + frac * delta[s]) * d[r]
                assert tree.locate(p)[0] == leaf[s]
