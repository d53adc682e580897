"""The fused multi-GPU update (dot_rmsprop_step_peers), checked on one GPU:
W "ranks" are W buffer sets on the same device and each rank's kernel runs
in turn (none waits on another), exactly as it would after the barrier on W
GPUs.  The result must equal the single-process update on the rank-order
f64 sum of the partial gradients, bit for bit, in every payload replica."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_peer_update_equals_summed_update(oracle, world):
    from helpers import irregular_tree
    from paper_2307_15333_b200.optim import RmsPropState
    from paper_2307_15333_b200.parallel import owned_rows, rmsprop_step_peers
    rng = np.random.default_rng(world)
    tree = irregular_tree(60 + world, 16, depth=3, splits=10, max_depth=5, device="cuda")
    cap, S, nsh = tree.capacity, tree.sh_stride, 48
    sig0 = tree.sigma.cpu().numpy().copy()
    sh0 = tree._sh_store.cpu().numpy().copy()
    v0s = rng.uniform(0, 1e-3, cap)
    v0h = rng.uniform(0, 1e-3, (cap, nsh))
    gs = [rng.normal(0, 1e-2, cap).astype(np.float32) for _ in range(world)]
    gh = [rng.normal(0, 1e-2, (cap, S)).astype(np.float32) for _ in range(world)]
    masks = [(rng.uniform(size=cap) < 0.4).astype(np.uint8) for _ in range(world)]
    for r in range(world):  # untouched rows carry no gradient
        gs[r][masks[r] == 0] = 0
        gh[r][masks[r] == 0] = 0
    dev = "cuda"
    P_sig = [torch.from_numpy(sig0).to(dev) for _ in range(world)]
    P_sh = [torch.from_numpy(sh0).to(dev) for _ in range(world)]
    G_sig = [torch.from_numpy(x).to(dev) for x in gs]
    G_sh = [torch.from_numpy(x).to(dev) for x in gh]
    T = [torch.from_numpy(m).to(dev) for m in masks]
    states = []
    for r in range(world):
        st = RmsPropState(tree)
        st.v_sigma.copy_(torch.from_numpy(v0s))
        st.v_sh.copy_(torch.from_numpy(v0h))
        states.append(st)
    for r in range(world):
        rmsprop_step_peers(P_sig, P_sh, G_sig, G_sh, T, r, states[r], owned_rows(cap, r, world), S, nsh)
    torch.cuda.synchronize()
    # expected: rank-order f64 sums, the reference's update (oracle)
    g_sig = np.zeros(cap)
    g_sh = np.zeros((cap, nsh))
    for r in range(world):
        g_sig = g_sig + gs[r].astype(np.float64)
        g_sh = g_sh + gh[r][:, :nsh].astype(np.float64)
    touched = np.nonzero(np.logical_or.reduce(masks))[0]
    e_sig, e_sh = sig0.copy(), sh0[:, :nsh].copy()
    e_vs, e_vh = v0s.copy(), v0h.copy()
    oracle.rmsprop_step(e_sig, e_sh, e_vs, e_vh, g_sig, g_sh, touched)
    for r in range(world):
        np.testing.assert_array_equal(P_sig[r].cpu().numpy(), e_sig)
        np.testing.assert_array_equal(P_sh[r].cpu().numpy()[:, :nsh], e_sh)
        assert not G_sig[r][torch.from_numpy(touched).to(dev)].any()
        assert not G_sh[r][torch.from_numpy(touched).to(dev)].any()
        lo, hi = owned_rows(cap, r, world)
        np.testing.assert_array_equal(states[r].v_sigma.cpu().numpy()[lo:hi], e_vs[lo:hi])
        np.testing.assert_array_equal(states[r].v_sh.cpu().numpy()[lo:hi], e_vh[lo:hi])


def test_peer_exchange_end_to_end_under_torchrun():
    """PeerExchange (torch symmetric memory + device barriers + the fused
    kernel) through train_step under torchrun on the GPUs of this box (one
    here), against the same steps without an exchange."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    n = max(1, min(torch.cuda.device_count(), 8))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29541", os.path.join(root, "tests", "peer_worker.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-2000:]
    assert res.stdout.count("PEER_OK") == n, res.stdout[-2000:]
