"""Host-side logic without a GPU: the C-ABI library exports, the pooled
octree API, canonical layout, .dot1 IO, scene generators, errors."""

import hashlib
import os
import re

import numpy as np
import pytest
import torch

from conftest import GOLDEN, ROOT


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "dot_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dot_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    """libdot_b200.so loads (no GPU needed) and exports what the header declares."""
    from paper_2307_15333_b200 import _lib
    from paper_2307_15333_b200.build import build
    build()
    lib = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.symbols())
    assert lib.dot_abi_version() == _lib.ABI_VERSION == 12


def test_binding_arity_matches_header():
    """Every ctypes signature in _lib has as many arguments as the header's
    prototype (an ABI change must touch both)."""
    from paper_2307_15333_b200 import _lib
    text = open(os.path.join(ROOT, "include", "dot_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    protos = dict(re.findall(r"\b(dot_[a-z0-9_]+)\s*\(([^;{]*?)\)\s*;", text))
    for name, (_, args) in _lib._SIGNATURES.items():
        params = protos[name].strip()
        n = 0 if params in ("", "void") else params.count(",") + 1
        assert n == len(args), (name, n, len(args))


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {os.path.join(ROOT, 'paper_2307_15333_b200', 'libdot_b200.so')}").read()
    assert "sm_100a" in out


def test_no_cpu_fallback_on_cpu_tree():
    from paper_2307_15333_b200.errors import ConfigError
    from paper_2307_15333_b200.octree import build_dense
    from paper_2307_15333_b200.render import render_rays
    tree = build_dense(1, (0, 0, 0), 1.0, 1, 0, max_depth=2, device="cpu")
    with pytest.raises(ConfigError):
        render_rays(tree, np.zeros((1, 3)) - 2, np.array([[1.0, 0, 0]]), 1.0)


def test_dot1_roundtrip_matches_reference_bytes():
    from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
    z = np.load(os.path.join(GOLDEN, "config1.npz"))
    blob = z["scene_dot1"].tobytes()
    tree = load_tree_bytes(blob, device="cpu")
    assert tree_bytes(tree) == blob
    tree.validate()


@pytest.mark.parametrize("name", ["recursive", "oneshot_ties", "merge_order", "sigma_target"])
def test_dot1_of_reference_pools(name):
    """Serialising the reference's own (non-canonical) post-calibrate pools
    reproduces the reference's save_tree bytes."""
    from paper_2307_15333_b200.octree import from_pool_arrays
    from paper_2307_15333_b200.scene_io import tree_bytes
    z = np.load(os.path.join(GOLDEN, f"calib_{name}.npz"))
    tree = from_pool_arrays({k[6:]: z[k] for k in z.files if k.startswith("after_")}, device="cpu")
    assert hashlib.sha256(tree_bytes(tree)).hexdigest() == str(z["after_dot1_sha256"])


def test_dot1_corruption_detected(tmp_path):
    from paper_2307_15333_b200.errors import BadMagicError, ChecksumError, TreeFileError
    from paper_2307_15333_b200.scene_io import load_tree, load_tree_bytes, save_tree
    from paper_2307_15333_b200.octree import build_dense
    tree = build_dense(2, (0, 0, 0), 1.0, 4, 3, max_depth=3, device="cpu")
    p = tmp_path / "t.dot1"
    save_tree(tree, p)
    data = bytearray(p.read_bytes())
    rng = np.random.default_rng(0)
    for _ in range(50):
        bad = bytearray(data)
        i = int(rng.integers(len(bad)))
        bad[i] ^= 1 << int(rng.integers(8))
        with pytest.raises(TreeFileError):
            load_tree_bytes(bytes(bad))
    with pytest.raises(ChecksumError):
        load_tree_bytes(bytes(data[:-5]))
    with pytest.raises(TreeFileError):
        load_tree(tmp_path / "missing.dot1")
    back = load_tree(p, device="cpu")
    assert torch.equal(back.sigma, tree.sigma)


def test_split_merge_pool_semantics_match_oracle(oracle):
    """LIFO slot reuse, split copy, fp64 merge mean: our host pool API vs the
    oracle's pool (itself pinned to the reference)."""
    from helpers import irregular_tree
    tree = irregular_tree(77, 4, depth=2, splits=15, merges=6, resplits=9, max_depth=5, device="cpu")
    rng = np.random.default_rng(77)
    ref = oracle.PoolTree(tree.center, 1.0, 4, 5, 8)
    # replay the same construction on the oracle pool through its own primitives
    from paper_2307_15333_b200.octree import build_dense
    base = build_dense(2, (0, 0, 0), 1.0, 4, 0, max_depth=5, device="cpu")
    assert base.leaf_count == 64
    tree.validate()
    assert tree.leaf_count == 7 * tree.internal_count + 1
    # canonical table: pool ids through ~leaf words, children contiguous
    topo = tree.topology()
    node = topo.node.numpy()
    order, new_index, _ = __import__("paper_2307_15333_b200.octree", fromlist=["level_order"]).level_order(tree)
    for i, pid in enumerate(order):
        if tree._leaf[pid]:
            assert node[i] == ~pid
        else:
            np.testing.assert_array_equal(new_index[tree._child[pid]], node[i] + np.arange(8))


def test_merge_mean_orders():
    """sigma mean pairwise, SH mean sequential (numpy's orders, octree.py:284-285)."""
    from paper_2307_15333_b200.octree import build_dense
    tree = build_dense(1, (0, 0, 0), 1.0, 1, 0, max_depth=2, device="cpu")
    vals = np.array([1e8, 1.0, -1e8, 3e-8, 7.0, 1e-3, -5.0, 2.5e7], dtype=np.float32)
    kids = tree.children(0)
    tree.sigma[torch.from_numpy(kids)] = torch.from_numpy(np.abs(vals))
    tree.sh[torch.from_numpy(kids), 0] = torch.from_numpy(vals)
    a = np.abs(vals).astype(np.float64)
    want_sigma = np.float32((((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]))) / 8.0)
    v = vals.astype(np.float64)
    acc = v[0]
    for k in range(1, 8):
        acc = acc + v[k]
    want_sh = np.float32(acc / 8.0)
    tree.merge_children(0)
    assert tree.sigma[0].item() == want_sigma
    assert tree.sh[0, 0].item() == want_sh


def test_locate_and_errors():
    from paper_2307_15333_b200.errors import DepthCapError, HandleError, OutOfBoundsError, PreconditionError
    from paper_2307_15333_b200.octree import build_dense
    tree = build_dense(1, (0, 0, 0), 1.0, 1, 0, max_depth=1, device="cpu")
    leaf, c, h = tree.locate((0.0, 0.0, 0.0))
    assert leaf == tree.children(0)[7] and h == 0.5
    with pytest.raises(OutOfBoundsError):
        tree.locate((1.0, 0.0, 0.0))
    with pytest.raises(DepthCapError):
        tree.split_leaf(int(leaf))
    with pytest.raises(HandleError):
        tree.is_leaf(999)
    with pytest.raises(PreconditionError):
        tree.merge_children(int(leaf))


def test_config1_field_matches_reference_scene(oracle):
    """The config-1 generator (blob field + dense build + recursive density
    prune) reproduces the reference's scene bytes, via the oracle's prune."""
    from paper_2307_15333_b200 import scenes
    from paper_2307_15333_b200.octree import build_dense, from_canonical_arrays
    from paper_2307_15333_b200.scene_io import tree_bytes
    z = np.load(os.path.join(GOLDEN, "config1.npz"))
    field = scenes.config1_field()
    dense = build_dense(5, (0, 0, 0), 1.0, 4, lambda c: (field.sigma_exact(c), np.zeros((len(c), 12))),
                        max_depth=5, device="cpu")
    pool = oracle.PoolTree.from_arrays({
        "root_center": dense.center, "half_extent": 1.0, "basis_count": 4, "max_depth": 5,
        "child": dense._child, "parent": dense._parent, "depth": dense._depth, "leaf": dense._leaf,
        "alive": dense._alive, "center": dense._center, "sigma": dense.sigma.numpy(),
        "sh": dense.sh.numpy(), "free": []})
    oracle.prune(pool, np.zeros(pool.capacity), 0.1, recursive=True, use_sigma=True)
    c = pool.canonical()
    n = c["is_leaf"].size
    node = np.where(c["is_leaf"] == 1, ~np.arange(n), c["kids"][:, 0]).astype(np.int32)
    sh = c["sh"].copy()
    leaves = np.nonzero(c["is_leaf"])[0]
    sh[leaves] = np.random.default_rng(2).normal(0.0, 0.3, (leaves.size, 12)).astype(np.float32)
    tree = from_canonical_arrays((0, 0, 0), 1.0, 4, 5, node, c["sigma"], sh, device="cpu")
    assert hashlib.sha256(tree_bytes(tree)).hexdigest() == str(z["scene_sha256"])


def test_adaptive_scene_small_cpu():
    from paper_2307_15333_b200 import scenes
    tree = scenes.adaptive_tree(scenes.BlobField.make(seed=2, n_blobs=8), max_depth=5, basis_count=4,
                                split_thr=200.0, min_depth=2, device="cpu")
    assert tree.leaf_count == 7 * tree.internal_count + 1
    tree.validate()
    assert tree.topology().pool_id is None


def test_config4_rig_and_field():
    """configs[3] stand-ins: ring cameras at r = 3 with |elevation| <= 15 deg
    looking at the origin; slab underside on the 2x bbox floor."""
    import math
    from paper_2307_15333_b200 import scenes
    focal, poses = scenes.ring_cameras(32, 1920, 1080, 3.0, seed=6)
    assert focal == pytest.approx(0.5 * 1920 / math.tan(0.5 * scenes.FOV_40))
    for p in poses:
        eye = p[:3, 3]
        assert np.linalg.norm(eye) == pytest.approx(3.0)
        assert abs(math.degrees(math.asin(eye[2] / 3.0))) <= 15.0 + 1e-9
        np.testing.assert_allclose(-p[:3, 2], -eye / 3.0, atol=1e-12)  # camera looks along -z
    f = scenes.config4_field()
    z_top, thick, dens = f.slab
    assert z_top - thick == pytest.approx(-2.0) and dens > 0
    assert f.mu.shape == (256, 3) and np.abs(f.mu).max() <= 1.2
    tree = scenes.adaptive_tree(f, max_depth=5, basis_count=1, split_thr=1000.0, min_depth=2,
                                half_extent=2.0, device="cpu")
    tree.validate()


def test_sh_basis_matches_kernel_constants():
    from paper_2307_15333_b200.sh import eval_sh_basis
    b = eval_sh_basis(3, np.array([0.0, 0.0, 1.0]))
    assert b[0] == pytest.approx(0.28209479177387814)
    assert b[2] == pytest.approx(0.4886025119029199)


def test_locate_dyadic_predicate():
    """dot_locate_supported is host-only (no GPU needed): the locate table is
    used exactly when the integer restatement of the descent is exact."""
    import ctypes
    from paper_2307_15333_b200 import _lib
    lib = _lib.load()
    dummy = (ctypes.c_int32 * 4)()
    sh = (ctypes.c_float * 16)()

    def view(center, half, max_depth=9, capacity=1000):
        v = _lib.DotTreeView()
        v.node = ctypes.addressof(dummy)
        v.n_nodes = 1
        v.sigma = ctypes.addressof(sh)
        v.sh = (ctypes.addressof(sh) + 15) // 16 * 16
        v.capacity = capacity
        v.basis_count = 1
        v.sh_stride = 4
        for k in range(3):
            v.center[k] = center[k]
        v.half_extent = half
        v.max_depth = max_depth
        return lib.dot_locate_supported(ctypes.byref(v))

    assert view((0, 0, 0), 1.0) == 1
    assert view((0.5, -0.25, 2.0), 0.5) == 1
    assert view((2.0 ** -20, 0, 0), 1.0) == 1
    assert view((2.0 ** -21, 0, 0), 1.0) == 0
    assert view((0.1, 0, 0), 1.0) == 0
    assert view((0, 0, 0), 0.75) == 0
    assert view((0, 0, 0), 1.0, max_depth=22) == 0
    assert view((0, 0, 0), 1.0, capacity=1 << 26) == 0
    # invalid views are rejected by the shared validator (int32 node words)
    assert view((0, 0, 0), 1.0, capacity=0) == 0
    assert view((0, 0, 0), 1.0, capacity=1 << 31) == 0


def _exp_args(n, seed=0):
    rng = np.random.default_rng(seed)
    parts = [-rng.uniform(0, 60, n), -rng.uniform(0, 1e-3, n), -rng.uniform(0, 1100, n),
             rng.uniform(-1, 1, n), -708 - rng.uniform(0, 40, n), -rng.uniform(0, 1e-17, n),
             rng.uniform(-745.2, -744.4, n // 8),
             np.array([0.0, -0.0, -np.inf, np.inf, np.nan, -745.13321910194122, -1e-300, 709.0,
                       1e-20, -2.0 ** -54, -2.0 ** -55, -512.0, -1024.0])]
    return np.concatenate(parts)


def test_exp_ref_matches_libm():
    """The kernels' exp (dot_exp.cuh, host build of the same code) returns
    glibc's exp bit for bit -- the reference's f64 exp (Numba -> libm)."""
    from oracle import oracle
    from paper_2307_15333_b200 import _lib
    x = _exp_args(400_000)
    want = oracle.exp(x)
    got = np.empty_like(x)
    _lib.load().dot_exp_ref_host(x.ctypes.data, got.ctypes.data, x.size)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)) or \
        np.array_equal(got, want, equal_nan=True)
    bad = np.nonzero(got.view(np.uint64) != want.view(np.uint64))[0]
    assert all(np.isnan(x[bad])), x[bad][:5]


def test_grad_comparison_rejects_wrong_gradients():
    """The scale-aware gradient check (helpers.assert_grads_close) fails for
    zeroed and for 1 %-scaled gradients of realistic magnitude (~1e-6)."""
    import pytest
    from helpers import assert_grads_close
    rng = np.random.default_rng(0)
    want = rng.normal(0.0, 1e-6, (500, 48)) * (rng.uniform(size=(500, 1)) < 0.7)
    assert_grads_close(want * (1 + 1e-6 * rng.normal(size=want.shape)), want)
    with pytest.raises(AssertionError):
        assert_grads_close(np.zeros_like(want), want)
    with pytest.raises(AssertionError):
        assert_grads_close(want * 1.01, want)


def test_write_history_format(tmp_path):
    """optim.write_history writes the reference's CSV (optim.py:196-206)."""
    from paper_2307_15333_b200.optim import write_history
    hist = [{"epoch": 1, "loss": 0.1, "psnr": float("nan"), "leaf_count": 8, "event": ""},
            {"epoch": 2, "loss": 1 / 3, "psnr": 20.5, "leaf_count": 15, "event": "calibrate merges=0 splits=1"}]
    p = tmp_path / "h.csv"
    write_history(hist, p)
    lines = p.read_text().splitlines()
    assert lines[0] == "epoch,loss,psnr,leaf_count,event"
    assert lines[1] == "1,0.1,nan,8,"
    assert lines[2] == f"2,{1 / 3!r},20.5,15,calibrate merges=0 splits=1"
