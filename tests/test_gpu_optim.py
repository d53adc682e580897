"""Optimizer-state remap and a short training run against the reference.

* RmsPropState.remap across a 3-round recursive calibrate: merged parents take
  the mean of their children's second moments (round by round), split
  children copy their parent's -- compared leaf by leaf in canonical order,
  bit-exactly (optim.py:89-104).
* train(): same data, config and seed as a reference train() run; leaf counts
  per epoch must match exactly, epoch losses within 1e-3 relative (the CUDA
  gradients are fp32 sums in atomic order, the reference's fp64 serial).
"""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_rmsprop_remap_matches_reference():
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.octree import from_pool_arrays
    from paper_2307_15333_b200.optim import RmsPropState
    from paper_2307_15333_b200.signals import SignalBuffer
    z = np.load(os.path.join(GOLDEN, "optim_remap.npz"))
    tree = from_pool_arrays(z, device="cuda")
    state = RmsPropState(tree)
    state.v_sigma.copy_(torch.from_numpy(z["v_sigma"]))
    state.v_sh.copy_(torch.from_numpy(z["v_sh"]))
    buf = SignalBuffer(tree)
    buf.accumulator.copy_(torch.from_numpy(z["acc"]))
    rep = calibrate(tree, buf, CalibrationConfig(tau=float(z["tau"]), gamma=float(z["gamma"]),
                                                 recursive=True), events=False)
    assert (rep.recursion_rounds, rep.merges_applied, rep.splits_applied) == (
        int(z["rounds"]), int(z["merges"]), int(z["splits"]))
    state.remap(rep)
    leaf = z["canon_is_leaf"]
    node = tree.topology().node.cpu().numpy()
    np.testing.assert_array_equal(node < 0, leaf)
    np.testing.assert_array_equal(state.v_sigma.cpu().numpy()[leaf], z["canon_v_sigma"][leaf])
    np.testing.assert_array_equal(state.v_sh.cpu().numpy()[leaf], z["canon_v_sh"][leaf])


class _Bundle:
    def __init__(self, origins, dirs, targets):
        self.origins, self.dirs, self.targets, self.heldout = origins, dirs, targets, []


def test_short_training_run_matches_reference():
    from paper_2307_15333_b200.octree import LeafPayload, build_dense
    from paper_2307_15333_b200.optim import TrainConfig, train
    from paper_2307_15333_b200.scene_io import load_tree_bytes
    z = np.load(os.path.join(GOLDEN, "train_small.npz"))
    trainee = build_dense(2, (0.0, 0.0, 0.0), 1.0, 1, LeafPayload(0.3, [0.0, 0.0, 0.0]),
                          max_depth=5, device="cuda")
    cfg = TrainConfig(epochs=6, interval=2, tau=0.5, gamma=0.1, batch_size=500, seed=3)
    _, hist = train(trainee, _Bundle(z["origins"], z["dirs"], z["targets"]), cfg)
    np.testing.assert_array_equal([h["leaf_count"] for h in hist], z["leaf_count"])
    np.testing.assert_allclose([h["loss"] for h in hist], z["loss"], rtol=1e-3)
    ref = load_tree_bytes(z["final_dot1"].tobytes(), device="cuda")
    np.testing.assert_array_equal(trainee.topology().node.cpu().numpy(),
                                  ref.topology().node.cpu().numpy())
    np.testing.assert_allclose(trainee.sigma.cpu().numpy(), ref.sigma.cpu().numpy(),
                               atol=1e-3, rtol=1e-3)
