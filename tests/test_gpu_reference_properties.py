"""The reference's own property tests, restated for the
CUDA path: batch duplication and order invariance of loss / gradients /
signal (test_gradients.py:97-110, test_signals.py:73-80), occlusion
discrimination of the Q signal (test_signals.py:102-117), the refine fixed
point and recursion monotonicity (test_calibrate.py:135-156), untouched
leaves never moving under the optimizer (test_optim.py:70-84)."""

import numpy as np
import pytest
import torch

from helpers import assert_grads_close

pytestmark = pytest.mark.gpu


def _scene(seed=91, B=4):
    from helpers import irregular_tree, ray_batch
    tree = irregular_tree(seed, B, depth=3, splits=30, merges=4, max_depth=5, device="cuda")
    o, d = ray_batch(seed + 1, 6000)
    t = np.random.default_rng(seed + 2).uniform(0, 1, (o.shape[0], 3))
    return tree, o, d, t


def test_duplicated_batch_same_loss_and_gradients_double_signal():
    from paper_2307_15333_b200.render import render_and_backprop
    tree, o, d, t = _scene()
    l1, g1, s1 = render_and_backprop(tree, o, d, t, 1.0)
    l2, g2, s2 = render_and_backprop(tree, np.concatenate([o, o]), np.concatenate([d, d]),
                                     np.concatenate([t, t]), 1.0)
    assert l2 == pytest.approx(l1, rel=1e-12)
    assert_grads_close(g2.dsigma, g1.dsigma, what="dsigma")
    assert_grads_close(g2.dsh, g1.dsh, what="dsh")
    np.testing.assert_array_equal(g2.touched, g1.touched)
    np.testing.assert_allclose(s2, 2.0 * s1, rtol=1e-12, atol=1e-15)


def test_batch_order_invariance():
    from paper_2307_15333_b200.render import render_and_backprop
    tree, o, d, t = _scene(93)
    p = np.random.default_rng(0).permutation(o.shape[0])
    for det in (False, True):
        l1, g1, s1 = render_and_backprop(tree, o, d, t, 0.5, deterministic=det)
        l2, g2, s2 = render_and_backprop(tree, o[p], d[p], t[p], 0.5, deterministic=det)
        assert l2 == pytest.approx(l1, rel=1e-12)
        assert_grads_close(g2.dsh, g1.dsh, what="dsh")
        np.testing.assert_allclose(s2, s1, rtol=1e-12, atol=1e-15)


def test_occluded_leaves_get_no_signal():
    """An opaque wall in front of a dense block: the block's leaves behind the
    cut receive no Q signal; the wall's leaves take it all."""
    from paper_2307_15333_b200.octree import build_dense
    from paper_2307_15333_b200.render import render_and_backprop

    def init(c):
        sig = np.where(c[:, 0] < -0.5, 60.0, np.where(c[:, 0] > 0.25, 30.0, 0.0))
        return sig, np.zeros((len(c), 12))

    tree = build_dense(3, (0.0, 0.0, 0.0), 1.0, 4, init, max_depth=4, device="cuda")
    rng = np.random.default_rng(7)
    n = 4000
    o = np.stack([np.full(n, -3.0), rng.uniform(-0.9, 0.9, n), rng.uniform(-0.9, 0.9, n)], axis=1)
    d = np.tile([1.0, 0.0, 0.0], (n, 1))
    _, g, sig = render_and_backprop(tree, o, d, np.zeros((n, 3)), 1.0)
    c = tree._center
    leaves = tree.leaf_ids()
    wall = leaves[c[leaves, 0] < -0.5]
    block = leaves[c[leaves, 0] > 0.25]
    assert sig[wall].sum() > 100.0
    assert sig[block].max() < 1e-6
    assert set(block.tolist()) <= set(g.touched.tolist())  # walked past the cut: touched


def test_refine_fixed_point_and_recursion_monotone():
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
    from paper_2307_15333_b200.signals import SignalBuffer
    tree, o, d, t = _scene(95, B=1)
    blob = tree_bytes(tree)
    rng = np.random.default_rng(3)

    def run(recursive, tau, gamma, acc_scale=1.0):
        tr = load_tree_bytes(blob, device="cuda")
        buf = SignalBuffer(tr)
        acc = np.where(tr.topology().node.cpu().numpy() < 0, rng.uniform(0, 1, tr.capacity) * acc_scale, 0.0)
        buf.accumulator.copy_(torch.from_numpy(acc))
        rep = calibrate(tr, buf, CalibrationConfig(tau=tau, gamma=gamma, recursive=recursive))
        return tr, rep

    tr, rep = run(False, 0.0, 0.0, acc_scale=1.0)  # nothing <= 0 among positive signals, no sampling
    assert (rep.merges_applied, rep.splits_applied) == (0, 0) and tree_bytes(tr) == blob
    rng = np.random.default_rng(4)
    _, one = run(False, 0.9, 0.0)
    rng = np.random.default_rng(4)
    _, rec = run(True, 0.9, 0.0)
    assert rec.merges_applied >= one.merges_applied and rec.recursion_rounds >= one.recursion_rounds


def test_untouched_leaves_never_move():
    from paper_2307_15333_b200.optim import RmsPropState, StepWorkspace, train_step
    from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
    from paper_2307_15333_b200.signals import SignalBuffer
    tree, o, d, t = _scene(97, B=9)
    tree = load_tree_bytes(tree_bytes(tree), device="cuda")
    keep = o[:, 1] > 0.5  # rays from one side only
    o, d, t = (torch.from_numpy(x[keep]).cuda() for x in (o, d, t))
    st, buf = RmsPropState(tree), SignalBuffer(tree)
    sws = StepWorkspace(tree, buf)
    sig0, sh0 = tree.sigma.clone(), tree.sh.clone()
    train_step(tree, o, d, t, st, buf, sws, 1.0)
    touched = sws.ws.touched.bool()
    assert bool(touched.any()) and not bool(touched.all())
    assert torch.equal(tree.sigma[~touched], sig0[~touched])
    assert torch.equal(tree.sh[~touched], sh0[~touched])
    assert not bool(st.v_sh[~touched].any())
