"""Seeded scene / ray builders for the tests (our own API, no reference)."""

import numpy as np


def irregular_tree(seed, basis_count=1, depth=2, splits=6, merges=2, resplits=2, max_depth=4,
                   center=(0.0, 0.0, 0.0), half=1.0, sigma_range=(0.05, 5.0), device=None):
    """Dense build, random splits, merges (freeing slots), then splits that
    reuse those slots LIFO -- a non-canonical pool like the reference's."""
    from paper_2307_15333_b200.octree import build_dense
    rng = np.random.default_rng(seed)
    nsh = 3 * basis_count

    def init(c):
        return rng.uniform(*sigma_range, len(c)), rng.normal(0.0, 1.0, (len(c), nsh))

    tree = build_dense(depth, center, half, basis_count, init, max_depth=max_depth, device=device)

    def split_some(k):
        import torch
        for _ in range(k):
            leaves = tree.leaf_ids()
            ok = leaves[tree._depth[leaves] < max_depth]
            if ok.size == 0:
                return
            kids = tree.split_leaf(int(rng.choice(ok)))
            tk = torch.from_numpy(kids).to(tree.device)
            tree.sigma[tk] = torch.from_numpy(rng.uniform(*sigma_range, 8).astype(np.float32)).to(tree.device)
            tree.sh[tk] = torch.from_numpy(rng.normal(0.0, 1.0, (8, nsh)).astype(np.float32)).to(tree.device)

    split_some(splits)
    for _ in range(merges):
        ints = tree.internal_ids()
        ok = [int(n) for n in ints if tree._leaf[tree._child[n]].all()]
        if not ok:
            break
        tree.merge_children(int(rng.choice(ok)))
    split_some(resplits)
    return tree


def ray_batch(seed, n, center=(0.0, 0.0, 0.0), half=1.0, miss_fraction=0.1):
    rng = np.random.default_rng(seed)
    c = np.asarray(center, dtype=np.float64)
    u = rng.normal(0.0, 1.0, (n, 3))
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    origins = c + u * (3.0 * half)
    dirs = c + rng.uniform(-0.9, 0.9, (n, 3)) * half - origins
    k = int(n * miss_fraction)
    if k:
        dirs[:k] = rng.normal(0.0, 1.0, (k, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return origins, dirs


def assert_grads_close(got, want, rtol=1e-3, atol_frac=1e-4, what="gradient"):
    """Gradient parity at the north star's 1e-4 abs / 1e-3 rel, with the
    absolute floor scaled to the gradient's own magnitude (leaf gradients
    are ~1e-6 at 2/n scaling, far below a fixed 1e-4): elementwise
    |got - want| <= atol_frac * max|want| + rtol * |want|, plus a relative L2
    error below rtol.  A zeroed or 1 %-scaled gradient fails both."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (got.shape, want.shape)
    scale = float(np.abs(want).max()) if want.size else 0.0
    if scale == 0.0:
        assert not np.any(got), f"{what}: reference is zero, got nonzero"
        return
    np.testing.assert_allclose(got, want, rtol=rtol, atol=atol_frac * scale, err_msg=what)
    rel = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    assert rel < rtol, f"{what}: relative L2 error {rel:.3e} >= {rtol}"
