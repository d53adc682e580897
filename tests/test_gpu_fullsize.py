"""Size-independent properties at BASELINE.json's full sizes (the oracle is
too slow there): configs[1]/[2] scene (2.6M leaves, 800x800 views, 2^20-ray
batches) and the configs[4] refine on a 16M-leaf depth-10 tree."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def scene():
    from paper_2307_15333_b200 import scenes
    return scenes.config2_scene(device="cuda")


def _view_rays(scene, seed=4, i=0):
    import bench
    from paper_2307_15333_b200 import scenes
    focal, poses = scenes.hemisphere_cameras(8, 800, 800, 4.03, seed=seed)
    return bench.view_rays_torch(focal, poses[i], torch.device("cuda"))


def test_config2_view_weight_conservation(scene):
    """sum_i T_i Q_i + T_final = 1 for every pixel of an 800x800 view (eps 0
    and 1e-4), and T_final in [0, 1]."""
    from paper_2307_15333_b200.render import render_rays
    o, d = _view_rays(scene)
    for eps in (0.0, 1e-4):
        rgb, tf, ws = render_rays(scene, o, d, 1.0, eps, return_aux=True)
        assert float((ws - 1.0).abs().max()) < 1e-5
        assert float(tf.min()) >= 0.0 and float(tf.max()) <= 1.0
        assert torch.isfinite(rgb).all()


def test_config2_full_batch_deterministic_and_atomic_agree(scene):
    """A 2^20-ray training batch: the deterministic path is bit-identical run
    to run; the default (atomic, learned-schedule) path agrees with it within
    the float tolerance and has the identical touched set."""
    import bench
    from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop
    o, d, t = bench.build_training_pool(scene, torch.device("cuda"))
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    idx = torch.randperm(o.shape[0], generator=g, device="cuda")[: 1 << 20]
    outs = []
    for _ in range(2):
        ws = BackpropWorkspace.for_tree(scene)
        loss, gr, sig = render_and_backprop(scene, o, d, t, 1.0, ray_index=idx, workspace=ws,
                                            deterministic=True)
        outs.append((float(loss), gr.dsigma.clone(), gr.dsh.clone(), sig.clone(), gr.touched_mask.clone()))
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1:], outs[1][1:]):
        assert torch.equal(a, b)
    for _ in range(3):  # warm the schedule table, then compare
        ws = BackpropWorkspace.for_tree(scene)
        loss, gr, sig = render_and_backprop(scene, o, d, t, 1.0, ray_index=idx, workspace=ws)
    assert float(loss) == pytest.approx(outs[0][0], rel=1e-9)
    torch.testing.assert_close(gr.dsigma, outs[0][1], atol=1e-7, rtol=1e-3)
    torch.testing.assert_close(gr.dsh, outs[0][2], atol=1e-7, rtol=1e-3)
    torch.testing.assert_close(sig, outs[0][3], atol=1e-9, rtol=1e-9)
    assert torch.equal(gr.touched_mask, outs[0][4])
    del o, d, t


def test_config5_refine_structure():
    """configs[4] refine (16M leaves): the result is a valid canonical octree
    with L = 7I + 1 and the counts the plan predicted; refining twice more
    keeps it valid."""
    import bench
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.signals import SignalBuffer
    tree = bench.config5_tree(torch.device("cuda"))
    n0, l0 = tree.topology().n_nodes, tree.leaf_count
    buf = SignalBuffer(tree)
    g = torch.Generator(device="cuda")
    g.manual_seed(55)
    node = tree.topology().node
    leaf = node < 0
    acc = torch.zeros(node.shape[0], dtype=torch.float64, device="cuda")
    acc[leaf] = torch.exp(-6.0 + 2.0 * torch.randn(int(leaf.sum()), generator=g, device="cuda",
                                                  dtype=torch.float64))
    buf.accumulator.copy_(acc)
    rep = calibrate(tree, buf, CalibrationConfig(tau=0.01, gamma=0.10), events=False)
    assert rep.leaves_before == l0
    assert tree.leaf_count == l0 - 7 * rep.merges_applied + 7 * rep.splits_applied
    assert tree.topology().n_nodes == n0 - 8 * rep.merges_applied + 8 * rep.splits_applied
    w = tree.topology().node
    internal = w[w >= 0]
    assert int((w < 0).sum()) == 7 * int(internal.numel()) + 1
    assert int(internal.max()) + 8 <= w.shape[0] and int(internal.min()) >= 1
    # every non-root node is the child of exactly one internal node
    kids = (internal[:, None] + torch.arange(8, device="cuda")).reshape(-1)
    assert int(kids.numel()) == w.shape[0] - 1
    assert torch.equal(torch.sort(kids).values, torch.arange(1, w.shape[0], device="cuda", dtype=kids.dtype))
    # leaves carry their own pool row (canonical: pool id == BFS index)
    lid = torch.nonzero(w < 0).reshape(-1)
    assert torch.equal((~w[lid]).to(torch.int64), lid)
