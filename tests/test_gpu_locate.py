"""The locate table (dot_locate_build) is an exact restatement of the root
descent (_kernels.py:56-68) for dyadic roots: with it, traversal must return
the same segments bit for bit as the fp64 descent and as the reference's
algorithm (C oracle), including rays that run exactly along cell faces,
start inside cells, or graze edges, and for every table level."""

import numpy as np
import pytest

from helpers import assert_grads_close  # noqa: E402

pytestmark = pytest.mark.gpu


def _with_level(tree, monkeypatch, level):
    monkeypatch.setenv("DOT_LOCATE_LEVEL", str(level))
    topo = tree.topology()
    topo.locate, topo.locate_level = None, -1
    tree.tree_view()
    return topo.locate_level


def _face_rays(center, half, n, seed, depth):
    """Axis-parallel and diagonal rays lying exactly on cell faces / edges."""
    rng = np.random.default_rng(seed)
    c = np.asarray(center, dtype=np.float64)
    cell = 2.0 * half / 2 ** depth
    o, d = [], []
    for _ in range(n):
        a = rng.integers(3)
        p = c + (rng.integers(-2 ** depth // 2, 2 ** depth // 2 + 1, 3) * cell)
        p[a] = c[a] - 3.0 * half  # start outside along axis a
        v = np.zeros(3)
        v[a] = 1.0
        if rng.uniform() < 0.3:  # diagonal in the face plane
            b = (a + 1 + rng.integers(2)) % 3
            v[b] = rng.choice([-1.0, 1.0])
            p[b] = c[b] - v[b] * 3.0 * half
        if rng.uniform() < 0.2:  # start inside, on a face
            p[a] = c[a] + rng.integers(-2 ** depth // 2, 2 ** depth // 2) * cell
        o.append(p)
        d.append(v / np.linalg.norm(v))
    return np.array(o), np.array(d)


@pytest.mark.parametrize("center,half", [((0.0, 0.0, 0.0), 1.0), ((0.5, -0.25, 0.125), 0.5),
                                         ((1.0, 1.0, -2.0), 2.0), ((3.0, 0.0, 0.0), 0.25)])
def test_locate_matches_fp64_descent_and_oracle(oracle, monkeypatch, center, half):
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200 import _lib
    from paper_2307_15333_b200.render import render_and_backprop, render_rays, segment_batch
    tree = irregular_tree(31, 4, depth=2, splits=60, merges=6, resplits=30, max_depth=7,
                          center=center, half=half, device="cuda")
    v, _ = tree.tree_view()
    assert _lib.load().dot_locate_supported(_lib.ctypes.byref(v)) == 1
    o1, d1 = ray_batch(5, 3000, center=center, half=half)
    o2, d2 = _face_rays(center, half, 1500, 6, 7)
    o, d = np.concatenate([o1, o2]), np.concatenate([d1, d2])
    tg = np.random.default_rng(2).uniform(0, 1, (o.shape[0], 3))
    assert _with_level(tree, monkeypatch, 0) == 0
    base = segment_batch(tree, o, d)
    rgb0 = render_rays(tree, o, d, 0.5)
    ref = oracle.segment_batch(tree, o, d)
    for a, b in zip(base, ref):
        np.testing.assert_array_equal(a, b)
    for level in (1, 2, 3, 5, 7, 9):
        got_level = _with_level(tree, monkeypatch, level)
        assert got_level == min(level, len(tree.topology().level_offsets) - 2)
        got = segment_batch(tree, o, d)
        for a, b in zip(got, base):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(render_rays(tree, o, d, 0.5), rgb0)
    loss, g, sig = render_and_backprop(tree, o, d, tg, 0.5)
    r_loss, r_g, r_sig = oracle.render_and_backprop(tree, o, d, tg, 0.5)
    np.testing.assert_array_equal(g.touched, r_g.touched)
    assert_grads_close(g.dsh, r_g.dsh, what="dsh")


def test_non_dyadic_root_ignores_table(monkeypatch):
    from helpers import irregular_tree
    from paper_2307_15333_b200 import _lib
    tree = irregular_tree(3, 1, depth=2, splits=5, center=(0.1, 0.0, 0.0), half=1.0, device="cuda")
    assert _with_level(tree, monkeypatch, 6) == 0
    v, _ = tree.tree_view()
    assert _lib.load().dot_locate_supported(_lib.ctypes.byref(v)) == 0
    assert v.locate is None
