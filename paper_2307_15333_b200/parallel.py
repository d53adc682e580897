"""Ray-sharded data parallelism over one node (one process per GPU).

The tree is replicated; a global ray batch of ``n_global`` rays is split into
contiguous per-rank shards; every rank runs the fused backward on its shard
with the *global* gradient scale 2/n_global (render.py:217 uses the batch n),
so the per-rank partial leaf gradients sum to the full-batch gradient.  One
collective per step then sums them (NCCL all-reduce over NVLink/NVSwitch):
grad_sigma, grad_sh, the touched mask (MAX) and the loss sum.  Signals are
accumulated locally and summed once per refine interval
(``allreduce_signal``); NCCL results are bitwise identical on every rank,
so every rank can run the refine itself and stay in lock-step without a
broadcast.

Everything here is plain ``torch.distributed``; it runs with ``gloo`` on CPU
tensors in the tests and ``nccl`` on the GPU in ``bench.py``.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(n_global: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) block of rank ``rank``; sizes differ by at most one."""
    base, extra = divmod(n_global, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def grad_scale(n_global: int) -> float:
    return 2.0 / n_global if n_global else 0.0


def allreduce_grads(dsigma: torch.Tensor, dsh: torch.Tensor, touched: torch.Tensor,
                    loss_sum: torch.Tensor | None = None, group=None) -> None:
    """Sum partial leaf gradients (and loss sums); OR the touched masks."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    dist.all_reduce(dsigma, group=group)
    dist.all_reduce(dsh, group=group)
    dist.all_reduce(touched, op=dist.ReduceOp.MAX, group=group)
    if loss_sum is not None:
        dist.all_reduce(loss_sum, group=group)


def chunk_bounds(n_rows: int, chunks: int) -> list[tuple[int, int]]:
    """Row ranges of a chunked gradient exchange (aligned to 64 rows)."""
    cuts = sorted({min(n_rows, ((n_rows * k) // chunks + 63) // 64 * 64) for k in range(chunks + 1)})
    cuts[0], cuts[-1] = 0, n_rows
    return [(a, b) for a, b in zip(cuts, cuts[1:]) if b > a]


def allreduce_grads_overlapped(dsigma: torch.Tensor, dsh: torch.Tensor, touched: torch.Tensor,
                               on_chunk, loss_sum: torch.Tensor | None = None, chunks: int = 4,
                               group=None) -> None:
    """All-reduce the per-leaf gradients in row chunks (async) and call
    ``on_chunk(lo, hi)`` -- the optimizer update of rows [lo, hi) -- as soon
    as each chunk's reduction has landed, so the collective of chunk k+1
    overlaps the update of chunk k.  Equivalent to allreduce_grads followed
    by one update over all rows."""
    n = dsigma.shape[0]
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        on_chunk(0, n)
        return
    parts = chunk_bounds(n, chunks)
    pending = []
    for lo, hi in parts:
        pending.append((
            dist.all_reduce(dsigma[lo:hi], group=group, async_op=True),
            dist.all_reduce(dsh[lo:hi], group=group, async_op=True),
            dist.all_reduce(touched[lo:hi], op=dist.ReduceOp.MAX, group=group, async_op=True)))
    if loss_sum is not None:
        pending.append((dist.all_reduce(loss_sum, group=group, async_op=True),))
    for (lo, hi), handles in zip(parts, pending):
        for h in handles:
            h.wait()
        on_chunk(lo, hi)
    for h in pending[len(parts):]:
        for hh in h:
            hh.wait()


def allreduce_signal(accumulator: torch.Tensor, group=None) -> None:
    """Sum per-rank signal accumulators before a refine."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(accumulator, group=group)


def sharded_render_and_backprop(tree, origins, dirs, targets, background, early_stop_eps,
                                workspace, group=None):
    """This rank's shard of a global batch through the fused kernel, then the
    gradient all-reduce.  ``origins``/``dirs``/``targets`` are the global
    batch (device tensors); returns (global mean loss tensor, GradBuffer, local signal)."""
    from .render import render_and_backprop
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = origins.shape[0]
    lo, hi = shard_bounds(n, rank, world)
    _, grads, signal = render_and_backprop(tree, origins[lo:hi], dirs[lo:hi], targets[lo:hi],
                                           background, early_stop_eps, grad_scale=grad_scale(n),
                                           workspace=workspace)
    allreduce_grads(workspace.dsigma, workspace.dsh_store, workspace.touched, workspace.loss, group)
    return workspace.loss[0] / max(n, 1), grads, signal
