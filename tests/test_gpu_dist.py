"""The data-parallel training step with the real CUDA kernels at world 2.

Only one GPU is available to this build, so both ranks run on cuda:0 and
talk over gloo (NCCL refuses two ranks on one device); the kernels never
wait on each other -- the collectives are host-side.  Each rank runs
``optim.train_step`` on its contiguous shard of a global batch with the
global gradient scale 2/n_global and ``parallel.allreduce_grads_overlapped``
as the exchange (chunked all-reduce, RMSProp per landed chunk) -- exactly
what bench.py runs under torchrun with NCCL.  Checked against one process
doing the full batch: payload, RMSProp state and touched set; then the
signal all-reduce + refine leaves bit-identical trees on both ranks
(SURVEY.md section 8e).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

N_GLOBAL = 1 << 16
STEPS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup():
    from helpers import irregular_tree, ray_batch
    from paper_2307_15333_b200.scene_io import load_tree_bytes, tree_bytes
    tree = irregular_tree(61, 16, depth=3, splits=60, merges=5, resplits=10, max_depth=6, device="cuda")
    tree = load_tree_bytes(tree_bytes(tree), device="cuda")  # canonical, like a loaded scene
    o, d = ray_batch(62, 3 * N_GLOBAL)
    t = np.random.default_rng(63).uniform(0, 1, (o.shape[0], 3))
    o, d, t = (torch.from_numpy(x).cuda() for x in (o, d, t))
    batches = [torch.randperm(o.shape[0], generator=torch.Generator().manual_seed(k))[:N_GLOBAL].cuda()
               for k in range(STEPS)]
    return tree, o, d, t, batches


def _run(rank, world, out_path, port=None):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here]
    import torch.distributed as dist
    torch.cuda.set_device(0)
    if world > 1:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    import hashlib
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.optim import RmsPropState, StepWorkspace, train_step
    from paper_2307_15333_b200.parallel import (allreduce_grads_overlapped, allreduce_signal, grad_scale,
                                                shard_bounds)
    from paper_2307_15333_b200.scene_io import tree_bytes
    from paper_2307_15333_b200.signals import SignalBuffer
    tree, o, d, t, batches = _setup()
    state, buf = RmsPropState(tree), SignalBuffer(tree)
    sws = StepWorkspace(tree, buf)
    ws = sws.ws

    def exchange(update):
        allreduce_grads_overlapped(ws.dsigma, ws.dsh_store, ws.touched, update, chunks=3)

    touched = []
    for idx in batches:
        lo, hi = shard_bounds(N_GLOBAL, rank, world)
        # the exchange zeroes the consumed gradients; keep this step's
        # reduced touched set before the next step clears it
        train_step(tree, o, d, t, state, buf, sws, 0.7, ray_index=idx[lo:hi], grad_scale=grad_scale(N_GLOBAL),
                   exchange=exchange if world > 1 else None)
        touched.append(ws.touched.clone())
    torch.cuda.synchronize()
    out = {"sigma": tree.sigma.cpu().numpy(), "sh": tree.sh.cpu().numpy(),
           "v_sigma": state.v_sigma.cpu().numpy(), "v_sh": state.v_sh.cpu().numpy(),
           "touched": torch.stack(touched).cpu().numpy(), "rays": buf.epoch_rays}
    if world > 1:
        allreduce_signal(buf.accumulator)
    out["signal"] = buf.accumulator.cpu().numpy()
    rep = calibrate(tree, buf, CalibrationConfig(tau=0.02, gamma=0.05))
    out["sha"] = hashlib.sha256(tree_bytes(tree)).hexdigest()
    out["counts"] = (rep.merges_applied, rep.splits_applied)
    np.savez(out_path, **{k: np.asarray(v) for k, v in out.items()})
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def test_train_step_world2_equals_single_process(tmp_path):
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_run, args=(r, 2, str(tmp_path / f"rank{r}.npz"), port)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    _run(0, 1, str(tmp_path / "single.npz"))
    r0, r1, one = (np.load(tmp_path / f"{k}.npz") for k in ("rank0", "rank1", "single"))
    # replicas stay identical: every rank applied the same all-reduced update
    for k in ("sigma", "sh", "v_sigma", "v_sh", "touched", "signal"):
        np.testing.assert_array_equal(r0[k], r1[k], err_msg=k)
    # ... and equal the single-process full-batch step up to fp32-atomic order
    np.testing.assert_array_equal(r0["touched"], one["touched"])
    np.testing.assert_allclose(r0["sigma"], one["sigma"], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(r0["sh"], one["sh"], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(r0["v_sigma"], one["v_sigma"], rtol=1e-3, atol=1e-18)
    np.testing.assert_allclose(r0["v_sh"], one["v_sh"], rtol=1e-3, atol=1e-18)
    # steps 2-3 run on payloads that already differ by fp32-atomic rounding
    np.testing.assert_allclose(r0["signal"], one["signal"], rtol=1e-5, atol=1e-12)
    assert int(r0["rays"]) + int(r1["rays"]) == int(one["rays"]) == STEPS * N_GLOBAL
    # the refine after the signal all-reduce: identical trees on both ranks
    assert str(r0["sha"]) == str(r1["sha"])
    assert tuple(r0["counts"]) == tuple(r1["counts"])
