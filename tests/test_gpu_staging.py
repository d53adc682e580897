"""Host-fed training through RayBatchStager + LossReader.

The staged loop (H2D of batch k+1 on a side stream while batch k computes,
loss read one step late) must give the same per-step losses and the same
trained leaves as the plain loop that hands render_and_backprop pinned host
tensors directly: both run the same kernels on the same rays; only the copy
schedule differs.  Losses agree to fp32-atomic noise (the leaf gradients are
float sums in atomic order), touched sets exactly.
"""

import numpy as np
import pytest
import torch

from helpers import irregular_tree, ray_batch

pytestmark = pytest.mark.gpu


def _batches(n_batches, n):
    out = []
    for k in range(n_batches):
        o, d = ray_batch(100 + k, n)
        t = np.random.default_rng(200 + k).uniform(0.0, 1.0, (n, 3))
        out.append(tuple(torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (o, d, t)))
    return out


def _train(staged: bool, batches):
    from paper_2307_15333_b200.optim import RmsPropState, rmsprop_step
    from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop
    from paper_2307_15333_b200.staging import LossReader, RayBatchStager
    tree = irregular_tree(5, basis_count=4, device="cuda")
    state = RmsPropState(tree)
    ws = BackpropWorkspace.for_tree(tree)
    touched = []
    if staged:
        stager, reader = RayBatchStager("cuda", depth=2), LossReader()
        stager.stage(*batches[0])
        for k in range(len(batches)):
            o, d, t = stager.take()
            assert o.is_cuda and o.shape == batches[k][0].shape
            if k + 1 < len(batches):
                stager.stage(*batches[k + 1])
            loss, grads, _ = render_and_backprop(tree, o, d, t, 0.5, workspace=ws)
            touched.append(ws.touched.clone())
            rmsprop_step(tree, grads, state)
            stager.release()
            reader.push(loss)
        reader.flush()
        losses = reader.values
    else:
        losses = []
        for o, d, t in batches:
            loss, grads, _ = render_and_backprop(tree, o, d, t, 0.5, workspace=ws)
            touched.append(ws.touched.clone().cuda())
            rmsprop_step(tree, grads, state)
            losses.append(float(loss.item()))
    torch.cuda.synchronize()
    return losses, touched, tree.sigma.clone(), tree.sh.clone()


def test_staged_loop_matches_direct_host_calls():
    batches = _batches(5, 3000)
    la, ta, sa, sha = _train(False, batches)
    lb, tb, sb, shb = _train(True, batches)
    assert len(lb) == len(la) == 5
    np.testing.assert_allclose(lb, la, rtol=1e-5, atol=1e-9)
    for x, y in zip(ta, tb):
        assert torch.equal(x.cpu(), y.cpu())
    np.testing.assert_allclose(sb.cpu().numpy(), sa.cpu().numpy(), rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(shb.cpu().numpy(), sha.cpu().numpy(), rtol=1e-4, atol=1e-5)


def test_stager_rejects_misuse():
    from paper_2307_15333_b200.errors import InputError
    from paper_2307_15333_b200.staging import RayBatchStager
    b = _batches(3, 64)
    st = RayBatchStager("cuda", depth=2)
    with pytest.raises(InputError):
        st.take()
    st.stage(*b[0])
    st.stage(*b[1])
    with pytest.raises(InputError):  # both slots in flight
        st.stage(*b[2])
    with pytest.raises(InputError):
        st.release()
    with pytest.raises(InputError):
        RayBatchStager("cuda").stage(b[0][0], b[0][1], b[0][2][:10])
    with pytest.raises(InputError):
        RayBatchStager("cuda", depth=1)


def test_stager_plans_match_in_stream_plans():
    """RayBatchStager(plan_tree=...) sorts each staged batch on the copy
    stream; the plan equals plan_batch on the same rays and the step it
    drives equals the step that sorts internally."""
    import numpy as np
    import torch
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.render import BackpropWorkspace, plan_batch, render_and_backprop
    from paper_2307_15333_b200.staging import RayBatchStager
    tree = irregular_tree(41, 4, depth=3, splits=30, max_depth=6, device="cuda")
    o, d = ray_batch(42, 40000)
    t = np.random.default_rng(43).uniform(0, 1, o.shape)
    st = RayBatchStager("cuda", max_rays=40000, plan_tree=tree)
    st.stage(torch.from_numpy(o), torch.from_numpy(d), torch.from_numpy(t))
    od, dd, td, plan = st.take_with_plan()
    ref = plan_batch(tree, od, dd)
    assert torch.equal(plan.idx, ref.idx) and torch.equal(plan.sorted_keys, ref.sorted_keys)
    ws1, ws2 = BackpropWorkspace.for_tree(tree), BackpropWorkspace.for_tree(tree)
    l1, g1, s1 = render_and_backprop(tree, od, dd, td, 0.5, workspace=ws1, plan=plan)
    l2, g2, s2 = render_and_backprop(tree, od, dd, td, 0.5, workspace=ws2)
    st.release()
    assert float(l1) == pytest.approx(float(l2), rel=1e-12)  # f64 atomic order
    torch.testing.assert_close(g1.dsh, g2.dsh, atol=1e-7, rtol=1e-5)
    assert torch.equal(g1.touched_mask, g2.touched_mask)


def test_stager_ranked_plans_with_ids():
    """RayBatchStager(plan_rank=) with batches staged with their dataset ids
    and costs: batches of varying size (a smaller last one), the plan
    launched behind the backward (plan_next as train_step's after_backward)
    or lazily by take_with_plan; each plan is a permutation of the batch's
    slots regrouped in key order, and training equals the unplanned staged
    loop to fp32-atomic noise."""
    from paper_2307_15333_b200.optim import RmsPropState, StepWorkspace, train_step
    from paper_2307_15333_b200.render import pool_rank, ray_costs
    from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
    from paper_2307_15333_b200.signals import SignalBuffer
    from paper_2307_15333_b200.staging import LossReader, RayBatchStager
    base = irregular_tree(61, 16, depth=3, splits=40, merges=4, max_depth=6, device="cuda")
    blob = tree_bytes(base)
    n_pool = 60000
    o, d = ray_batch(62, n_pool)
    t = np.random.default_rng(63).uniform(0, 1, (n_pool, 3))
    od, dd = torch.from_numpy(o).cuda(), torch.from_numpy(d).cuda()
    ref_tree = load_tree_bytes(blob, device="cuda")
    pr = pool_rank(ref_tree, od, dd)
    costs = ray_costs(ref_tree, od, dd).cpu()
    perm = np.random.default_rng(64).permutation(n_pool)
    sizes = [20000, 20000, 16000, 4000]
    batches, at = [], 0
    for m in sizes:
        ids = perm[at:at + m]
        at += m
        batches.append(tuple(torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (o[ids], d[ids], t[ids]))
                       + (costs[torch.from_numpy(ids)].contiguous().pin_memory(),
                          torch.from_numpy(ids.astype(np.int64)).pin_memory()))

    def run(ranked: bool):
        tree = load_tree_bytes(blob, device="cuda")
        st, buf = RmsPropState(tree), SignalBuffer(tree)
        sws = StepWorkspace(tree, buf)
        stager = RayBatchStager("cuda", max_rays=max(sizes), plan_tree=tree if ranked else None,
                                plan_rank=pr if ranked else None)
        reader = LossReader()
        stager.stage(*batches[0])
        for k in range(len(batches)):
            ob, db, tb, plan = stager.take_with_plan()
            if ranked:
                m = sizes[k]
                assert torch.equal(torch.sort(plan.idx).values, torch.arange(m, device="cuda"))
            if k + 1 < len(batches):
                stager.stage(*batches[k + 1])
            hook = stager.plan_next if (ranked and k % 2 == 0) else None  # odd steps: the lazy launch
            loss = train_step(tree, ob, db, tb, st, buf, sws, 0.5, plan=plan, after_backward=hook)
            stager.release()
            reader.push(loss)
        reader.flush()
        torch.cuda.synchronize()
        return reader.values, tree

    la, ta = run(False)
    lb, tb = run(True)
    np.testing.assert_allclose(lb, la, rtol=1e-5, atol=1e-9)
    torch.testing.assert_close(tb.sigma, ta.sigma, atol=1e-5, rtol=1e-4)
    torch.testing.assert_close(tb.sh, ta.sh, atol=1e-5, rtol=1e-4)
