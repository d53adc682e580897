"""Multi-rank host logic on CPU (gloo, world_size 2).

The per-rank compute is the C oracle (test stand-in for the GPU kernel); the
sharding, global gradient scale and the collectives are the product's
``paper_2307_15333_b200.parallel`` functions.  The rank partials summed by
all-reduce must equal the single-process full batch.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2307_15333_b200.parallel import allreduce_grads, allreduce_signal, grad_scale, shard_bounds
    from helpers import irregular_tree, ray_batch
    tree = irregular_tree(31, 4, depth=2, splits=6, merges=2, max_depth=4, device="cpu")
    o, d = ray_batch(32, 501)
    tg = np.random.default_rng(3).uniform(0, 1, (501, 3))
    lo, hi = shard_bounds(501, rank, world)
    loss, g, sig = O.render_and_backprop(tree, o[lo:hi], d[lo:hi], tg[lo:hi], 0.5,
                                         grad_scale=grad_scale(501))
    ds = torch.from_numpy(g.dsigma.copy())
    dh = torch.from_numpy(g.dsh.copy())
    touched = torch.zeros(tree.capacity, dtype=torch.uint8)
    touched[torch.from_numpy(g.touched)] = 1
    loss_sum = torch.tensor([loss * (hi - lo)], dtype=torch.float64)
    allreduce_grads(ds, dh, touched, loss_sum)
    s = torch.from_numpy(sig.copy())
    allreduce_signal(s)
    if rank == 0:
        np.savez(out_path, dsigma=ds.numpy(), dsh=dh.numpy(), touched=touched.numpy(),
                 loss=loss_sum.numpy() / 501, signal=s.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _worker_overlap(rank, world, port, out_path):
    """Chunked all-reduce + per-chunk optimizer update (parallel.allreduce_grads_overlapped)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2307_15333_b200.parallel import allreduce_grads_overlapped, grad_scale, shard_bounds
    from helpers import irregular_tree, ray_batch
    tree = irregular_tree(41, 4, depth=2, splits=9, merges=2, max_depth=4, device="cpu")
    o, d = ray_batch(42, 777)
    tg = np.random.default_rng(4).uniform(0, 1, (777, 3))
    lo, hi = shard_bounds(777, rank, world)
    loss, g, sig = O.render_and_backprop(tree, o[lo:hi], d[lo:hi], tg[lo:hi], 0.5,
                                         grad_scale=grad_scale(777))
    ds = torch.from_numpy(g.dsigma.copy())
    dh = torch.from_numpy(g.dsh.copy())
    touched = torch.zeros(tree.capacity, dtype=torch.uint8)
    touched[torch.from_numpy(g.touched)] = 1
    sigma = tree.sigma.numpy().copy()
    sh = tree.sh.numpy().copy()
    vs = np.full(tree.capacity, 1e-4)
    vh = np.full((tree.capacity, 12), 1e-4)
    seen = []

    def on_chunk(a, b):
        seen.append((a, b))
        idx = a + np.nonzero(touched[a:b].numpy())[0]
        O.rmsprop_step(sigma, sh, vs, vh, ds.numpy(), dh.numpy(), idx)

    allreduce_grads_overlapped(ds, dh, touched, on_chunk, chunks=3)
    assert seen[0][0] == 0 and seen[-1][1] == tree.capacity and len(seen) >= 2
    if rank == 0:
        np.savez(out_path, sigma=sigma, sh=sh, vs=vs, vh=vh)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_overlapped_allreduce_and_update(tmp_path, oracle):
    from helpers import irregular_tree, ray_batch
    out = str(tmp_path / "o.npz")
    mp.start_processes(_worker_overlap, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    tree = irregular_tree(41, 4, depth=2, splits=9, merges=2, max_depth=4, device="cpu")
    o, d = ray_batch(42, 777)
    tg = np.random.default_rng(4).uniform(0, 1, (777, 3))
    _, g, _ = oracle.render_and_backprop(tree, o, d, tg, 0.5)
    sigma = tree.sigma.numpy().copy()
    sh = tree.sh.numpy().copy()
    vs = np.full(tree.capacity, 1e-4)
    vh = np.full((tree.capacity, 12), 1e-4)
    oracle.rmsprop_step(sigma, sh, vs, vh, g.dsigma, g.dsh, g.touched)
    np.testing.assert_allclose(got["vs"], vs, rtol=1e-9, atol=1e-20)
    np.testing.assert_allclose(got["vh"], vh, rtol=1e-9, atol=1e-20)
    np.testing.assert_allclose(got["sigma"], sigma, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(got["sh"], sh, rtol=1e-6, atol=1e-7)


def test_shard_bounds_partition():
    from paper_2307_15333_b200.parallel import shard_bounds
    for n in (0, 1, 7, 1000, 1 << 20):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_two_rank_allreduce_equals_full_batch(tmp_path, oracle):
    from helpers import irregular_tree, ray_batch
    out = str(tmp_path / "r.npz")
    mp.start_processes(_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    tree = irregular_tree(31, 4, depth=2, splits=6, merges=2, max_depth=4, device="cpu")
    o, d = ray_batch(32, 501)
    tg = np.random.default_rng(3).uniform(0, 1, (501, 3))
    loss, g, sig = oracle.render_and_backprop(tree, o, d, tg, 0.5)
    np.testing.assert_allclose(got["dsigma"], g.dsigma, rtol=1e-12, atol=1e-18)
    np.testing.assert_allclose(got["dsh"], g.dsh, rtol=1e-12, atol=1e-18)
    np.testing.assert_array_equal(np.nonzero(got["touched"])[0], g.touched)
    np.testing.assert_allclose(got["signal"], sig, rtol=1e-12, atol=1e-15)
    assert float(got["loss"][0]) == pytest.approx(loss, rel=1e-12)


def test_owned_rows_partition():
    from paper_2307_15333_b200.parallel import owned_rows
    for cap in (1, 63, 64, 1000, 123457):
        for world in (1, 2, 3, 8):
            parts = [owned_rows(cap, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == cap
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b
