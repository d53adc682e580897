"""Training-signal paths beyond the fused backward (GPU):

* ``render.signal_pass`` (dot_signal_fwd):
  the signal of ``render_and_backprop`` without gradients -- equal to the
  reference's per-leaf sum Q (golden fixtures, oracle) and to the backward's
  own signal; touched marks equal the reference's.
* North-star extras (no reference counterpart, defined by
  oracle/dot_oracle.c oracle_weights): per-leaf sum and max of the
  compositing weight T_i Q_i, from signal_pass and from the backward.  The
  max is exact (same exp, same transmittance products); sums are f64
  atomics (order differs).
* Out-of-range ray indices are rejected (loss NaN / InputError).
"""

import glob
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

RENDER_CASES = sorted(glob.glob(os.path.join(GOLDEN, "render_*.npz")))


@pytest.mark.parametrize("path", RENDER_CASES, ids=lambda p: os.path.basename(p)[7:-4])
@pytest.mark.parametrize("tag,eps", [("eps", 1e-4), ("noeps", 0.0)])
def test_signal_pass_matches_reference(path, tag, eps):
    from paper_2307_15333_b200.octree import from_pool_arrays
    from paper_2307_15333_b200.render import signal_pass
    z = np.load(path)
    tree = from_pool_arrays(z, device="cuda")
    tn, tf = float(z["t_near"]), float(z["t_far"])
    sig = signal_pass(tree, z["origins"], z["dirs"], eps, tn, tf)
    np.testing.assert_allclose(sig, z[f"signal_{tag}"], rtol=1e-12, atol=1e-15)
    touched = torch.zeros(tree.capacity, dtype=torch.uint8, device="cuda")
    o, d = (torch.from_numpy(z[k]).cuda() for k in ("origins", "dirs"))
    signal_pass(tree, o, d, eps, tn, tf, touched=touched)
    np.testing.assert_array_equal(torch.nonzero(touched).reshape(-1).cpu().numpy(), z[f"touched_{tag}"])


def test_weight_extras_vs_oracle(oracle):
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.render import render_and_backprop, signal_pass
    from paper_2307_15333_b200.signals import SignalBuffer
    tree = irregular_tree(31, 9, depth=3, splits=40, merges=6, resplits=10, max_depth=6, device="cuda")
    o, d = ray_batch(32, 40000)
    tg = np.random.default_rng(33).uniform(0, 1, (o.shape[0], 3))
    _, want_s, want_m = oracle.render_weights(tree, o, d, 1e-4)
    _, r_g, r_sig = oracle.render_and_backprop(tree, o, d, tg, 1.0)
    cap = tree.capacity
    ws, wm = (torch.zeros(cap, dtype=torch.float64, device="cuda") for _ in range(2))
    od, dd, td = (torch.from_numpy(x).cuda() for x in (o, d, tg))
    buf = SignalBuffer(tree)
    signal_pass(tree, od, dd, 1e-4, buffer=buf, weight_sum=ws, weight_max=wm)
    assert buf.epoch_rays == o.shape[0]
    np.testing.assert_allclose(buf.accumulator.cpu().numpy(), r_sig, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(ws.cpu().numpy(), want_s, rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(wm.cpu().numpy(), want_m)
    # the same extras from the fused backward
    ws2, wm2 = (torch.zeros(cap, dtype=torch.float64, device="cuda") for _ in range(2))
    _, g, sig = render_and_backprop(tree, od, dd, td, 1.0, weight_sum=ws2, weight_max=wm2)
    np.testing.assert_allclose(ws2.cpu().numpy(), want_s, rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(wm2.cpu().numpy(), want_m)
    np.testing.assert_allclose(sig.cpu().numpy(), r_sig, rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(torch.nonzero(g.touched_mask).reshape(-1).cpu().numpy(), r_g.touched)


def test_out_of_range_ray_index_is_rejected():
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.errors import InputError
    from paper_2307_15333_b200.render import render_and_backprop, signal_pass
    tree = irregular_tree(41, 4, depth=2, splits=5, max_depth=4, device="cuda")
    o, d = ray_batch(42, 1000)
    t = np.full((1000, 3), 0.5)
    idx = np.arange(0, 2000, 2)  # half of them past the 1000 rays
    od, dd, td = (torch.from_numpy(x).cuda() for x in (o, d, t))
    loss, _, _ = render_and_backprop(tree, od, dd, td, 1.0, ray_index=torch.from_numpy(idx).cuda())
    assert torch.isnan(loss)
    ok = torch.from_numpy(idx[idx < 1000]).cuda()
    loss, _, _ = render_and_backprop(tree, od, dd, td, 1.0, ray_index=ok)
    assert torch.isfinite(loss)
    with pytest.raises(InputError):
        signal_pass(tree, o, d, ray_index=idx)
    torch.cuda.synchronize()  # the context survived the rejected indices


def test_numpy_gradients_are_lazy_and_optimizer_stays_on_device():
    """With numpy inputs the GradBuffer converts to float64 numpy only when
    read; rmsprop_step consumes the device tensors directly (same update)."""
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.optim import RmsPropState, rmsprop_step
    from paper_2307_15333_b200.render import render_and_backprop
    tree = irregular_tree(51, 4, depth=2, splits=8, max_depth=4, device="cuda")
    o, d = ray_batch(52, 5000)
    t = np.random.default_rng(53).uniform(0, 1, (5000, 3))
    _, g, _ = render_and_backprop(tree, o, d, t, 1.0)
    assert not g._np  # nothing converted yet
    before = tree.sigma.clone()
    st = RmsPropState(tree)
    rmsprop_step(tree, g, st)
    assert not g._np
    assert isinstance(g.dsigma, np.ndarray) and g.dsigma.dtype == np.float64
    assert g.dsh.shape == (tree.capacity, 12) and isinstance(g.touched, np.ndarray)
    assert not torch.equal(before, tree.sigma)


def test_diagnostic_flags_rejected_by_product_library():
    """Timing-diagnostic flag bits exist only in experiment builds: the
    product library rejects everything but bit 15 (per-lane REDs)."""
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.errors import InputError
    from paper_2307_15333_b200.render import render_and_backprop
    tree = irregular_tree(71, 4, depth=2, splits=4, max_depth=4, device="cuda")
    o, d = ray_batch(72, 500)
    t = np.full((500, 3), 0.5)
    for bad in (1, 8192, 16384):
        with pytest.raises(InputError):
            render_and_backprop(tree, o, d, t, 1.0, kernel_flags=bad)
    l1, g1, _ = render_and_backprop(tree, o, d, t, 1.0)
    l2, g2, _ = render_and_backprop(tree, o, d, t, 1.0, kernel_flags=32768)
    assert l2 == pytest.approx(l1, rel=1e-9)
    np.testing.assert_array_equal(g1.touched, g2.touched)


def test_ray_costs_and_cost_ordered_launch():
    """dot_ray_costs gives exactly the per-ray cost the backward reports
    (composited + post-cut / 2); dot_sched_order_costs is a permutation of
    the warps with non-increasing warp (chunk) cost, a short last chunk last;
    a plan built from costs gives the same results and refreshes the costs."""
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200 import _lib
    from paper_2307_15333_b200.render import BackpropWorkspace, plan_batch, ray_costs, render_and_backprop
    tree = irregular_tree(81, 9, depth=3, splits=60, merges=4, max_depth=6, device="cuda")
    o, d = ray_batch(82, 70001)
    t = np.random.default_rng(83).uniform(0, 1, (o.shape[0], 3))
    o, d, t = (torch.from_numpy(x).cuda() for x in (o, d, t))
    costs = ray_costs(tree, o, d)
    assert int(costs.max()) > 3
    idx = torch.randperm(o.shape[0], generator=torch.Generator().manual_seed(2))[:50000].cuda()
    fresh = torch.zeros_like(costs)
    p = plan_batch(tree, o, d, idx, costs=fresh)  # all-zero costs: any order, then refreshed
    ws = BackpropWorkspace.for_tree(tree)
    l1, g1, s1 = render_and_backprop(tree, o, d, t, 0.5, ray_index=idx, workspace=ws, plan=p)
    torch.cuda.synchronize()
    assert torch.equal(fresh[idx], costs[idx])  # the backward's counts == dot_ray_costs
    assert not bool(fresh[torch.ones(o.shape[0], dtype=torch.bool, device="cuda").index_fill_(0, idx, False)].any())
    ws2 = BackpropWorkspace.for_tree(tree)
    l2, g2, s2 = render_and_backprop(tree, o, d, t, 0.5, ray_index=idx, workspace=ws2,
                                     plan=plan_batch(tree, o, d, idx, costs=costs))
    assert float(l2) == pytest.approx(float(l1), rel=1e-9)
    torch.testing.assert_close(g2.dsh, g1.dsh, atol=1e-7, rtol=1e-4)
    assert torch.equal(g2.touched_mask, g1.touched_mask)
    torch.testing.assert_close(s2, s1, rtol=1e-12, atol=1e-15)
    # the order itself
    n = 70001
    slot = costs[:n].contiguous()
    nw = (n + 31) // 32
    for chunk in (1, 16):
        order = torch.empty(nw, dtype=torch.int32, device="cuda")
        _lib.call("dot_sched_order_costs", _lib.ptr(slot), n, None, n, chunk, _lib.ptr(order), _lib.stream_ptr())
        od = order.cpu().numpy()
        assert np.array_equal(np.sort(od), np.arange(nw))
        pad = np.zeros(nw * 32, dtype=np.int64)
        pad[:n] = slot.cpu().numpy()
        wc = np.minimum(pad.reshape(nw, 32).max(1), 1023)
        nfull = nw // chunk
        cc = wc[: nfull * chunk].reshape(nfull, chunk).max(1)
        firsts = od[: nfull * chunk: chunk] // chunk
        assert np.all(np.diff(cc[firsts]) <= 0)
        if nw % chunk:
            assert np.array_equal(od[nfull * chunk:], np.arange(nfull * chunk, nw))


def test_signal_pass_with_ranked_plan():
    """signal_pass(plan=) with a ranked, cost-regrouped plan (its warp order
    materialised into the ray order when the batch is whole warps) gives the
    signal of the unplanned pass (f64 atomics: 1e-12) and the same touched
    set, for whole-warp and ragged batches."""
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.render import plan_batch, pool_rank, ray_costs, signal_pass
    tree = irregular_tree(91, 16, depth=3, splits=40, merges=4, max_depth=6, device="cuda")
    o, d = ray_batch(92, 50_000)
    o, d = torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()
    pr = pool_rank(tree, o, d)
    costs = ray_costs(tree, o, d)
    for m in (30_016, 30_011):
        idx = torch.randperm(50_000, generator=torch.Generator().manual_seed(4))[:m].cuda()
        plan = plan_batch(tree, o, d, idx, rank=pr, costs=costs)
        assert plan.warp_order is not None
        t1 = torch.zeros(tree.capacity, dtype=torch.uint8, device="cuda")
        t2 = torch.zeros_like(t1)
        s1 = signal_pass(tree, o, d, ray_index=idx, plan=plan, touched=t1)
        s2 = signal_pass(tree, o, d, ray_index=idx, coherent=False, touched=t2)
        torch.testing.assert_close(s1, s2, rtol=1e-12, atol=1e-15)
        assert torch.equal(t1, t2)
