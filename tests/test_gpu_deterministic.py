"""Deterministic backward (render_and_backprop(deterministic=True) ->
dot_render_bwd_sorted): per-leaf sums in the reference's serial ray-major
order (scatter_kernel, _kernels.py:327-346), bit-identical from run to run,
and the same values as the reference within the float tolerance."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN

from helpers import assert_grads_close  # noqa: E402

pytestmark = pytest.mark.gpu

ATOL, RTOL = 1e-4, 1e-3
RENDER_CASES = sorted(glob.glob(os.path.join(GOLDEN, "render_*.npz")))


@pytest.mark.parametrize("path", RENDER_CASES, ids=lambda p: os.path.basename(p)[7:-4])
@pytest.mark.parametrize("tag,eps", [("eps", 1e-4), ("noeps", 0.0)])
def test_golden_deterministic(path, tag, eps):
    from paper_2307_15333_b200.octree import from_pool_arrays
    from paper_2307_15333_b200.render import render_and_backprop
    z = np.load(path)
    tree = from_pool_arrays(z, device="cuda")
    loss, g, sig = render_and_backprop(tree, z["origins"], z["dirs"], z["targets"], z["bg"], eps,
                                       float(z["t_near"]), float(z["t_far"]), deterministic=True)
    assert loss == pytest.approx(float(z[f"loss_{tag}"]), rel=RTOL, abs=ATOL)
    assert_grads_close(g.dsigma, z[f"dsigma_{tag}"], what="dsigma")
    assert_grads_close(g.dsh, z[f"dsh_{tag}"], what="dsh")
    np.testing.assert_array_equal(g.touched, z[f"touched_{tag}"])
    # same traversal (bit-exact), same exp (exp_ref == glibc), same order:
    # the signal is the reference's to the last bit
    np.testing.assert_array_equal(sig, z[f"signal_{tag}"])


def test_config1_signal_order(oracle):
    """Config 1 (coherence-sorted internally): the deterministic signal uses
    the reference's summation order and exp, so it matches the reference's
    signal to the last bit."""
    from paper_2307_15333_b200.render import render_and_backprop
    from paper_2307_15333_b200.scene_io import load_tree_bytes
    z = np.load(os.path.join(GOLDEN, "config1.npz"))
    tree = load_tree_bytes(z["scene_dot1"].tobytes(), device="cuda")
    _, g, sig = render_and_backprop(tree, z["origins"], z["dirs"], z["targets"], 1.0,
                                    deterministic=True)
    np.testing.assert_array_equal(sig, z["signal"])
    np.testing.assert_array_equal(g.touched, z["touched"])


def test_bit_identical_across_runs_and_vs_atomic():
    import torch
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop
    tree = irregular_tree(77, 16, depth=3, splits=200, merges=10, resplits=50, max_depth=6,
                          device="cuda")
    o, d = ray_batch(78, 1 << 16)
    tg = np.random.default_rng(79).uniform(0, 1, (o.shape[0], 3))
    o, d, tg = (torch.from_numpy(x).cuda() for x in (o, d, tg))
    outs = []
    for _ in range(3):
        ws = BackpropWorkspace.for_tree(tree)
        loss, g, sig = render_and_backprop(tree, o, d, tg, 0.5, workspace=ws, deterministic=True)
        outs.append((loss.item(), g.dsigma.clone(), g.dsh.clone(), sig.clone(), g.touched_mask.clone()))
    for other in outs[1:]:
        assert other[0] == outs[0][0]
        for a, b in zip(other[1:], outs[0][1:]):
            assert torch.equal(a, b)
    ws = BackpropWorkspace.for_tree(tree)
    loss, g, sig = render_and_backprop(tree, o, d, tg, 0.5, workspace=ws)
    assert loss.item() == pytest.approx(outs[0][0], rel=1e-12)
    torch.testing.assert_close(g.dsigma, outs[0][1], atol=1e-5, rtol=1e-4)
    torch.testing.assert_close(g.dsh, outs[0][2], atol=1e-5, rtol=1e-4)
    torch.testing.assert_close(sig, outs[0][3], atol=1e-12, rtol=1e-12)
    assert torch.equal(g.touched_mask, outs[0][4])


def test_accumulate_and_empty():
    import torch
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop
    tree = irregular_tree(5, 4, depth=2, splits=20, device="cuda")
    o, d = ray_batch(6, 4000)
    tg = np.random.default_rng(7).uniform(0, 1, (o.shape[0], 3))
    ws = BackpropWorkspace.for_tree(tree)
    render_and_backprop(tree, o[:2000], d[:2000], tg[:2000], 0.5, workspace=ws, grad_scale=1 / 2000,
                        deterministic=True)
    _, g, sig = render_and_backprop(tree, o[2000:], d[2000:], tg[2000:], 0.5, workspace=ws,
                                    grad_scale=1 / 2000, accumulate=True, deterministic=True)
    _, g2, sig2 = render_and_backprop(tree, o, d, tg, 0.5, deterministic=True)
    np.testing.assert_allclose(g.dsigma, g2.dsigma, atol=1e-6, rtol=1e-5)
    np.testing.assert_allclose(g.dsh, g2.dsh, atol=1e-6, rtol=1e-5)
    np.testing.assert_allclose(sig, sig2, atol=1e-12, rtol=1e-12)
    loss, g, sig = render_and_backprop(tree, o[:0], d[:0], tg[:0], 0.5, deterministic=True)
    assert loss == 0.0 and not g.touched_mask.any()


def test_sorted_rejects_bad_ray_index():
    import ctypes
    import torch
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200 import _lib
    from paper_2307_15333_b200.errors import InputError
    from paper_2307_15333_b200.render import BackpropWorkspace
    tree = irregular_tree(9, 1, depth=2, device="cuda")
    o, d = ray_batch(1, 100)
    o, d = torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()
    t = torch.zeros_like(o)
    ws = BackpropWorkspace.for_tree(tree)
    bad = torch.arange(100, device="cuda")
    bad[7] = 3  # repeated index
    view, _ = tree.tree_view()
    bg = np.ones(3)
    with pytest.raises(InputError):
        _lib.call("dot_render_bwd_sorted", ctypes.byref(view), _lib.ptr(o), _lib.ptr(d), _lib.ptr(t),
                  _lib.ptr(bad), None, None, 100, bg.ctypes.data_as(ctypes.c_void_p), 1e-4, 0.0, float("inf"), 0.02,
                  _lib.ptr(ws.dsigma), _lib.ptr(ws.dsh_store), tree.sh_stride, _lib.ptr(ws.signal),
                  _lib.ptr(ws.touched), _lib.ptr(ws.loss), _lib.stream_ptr())
