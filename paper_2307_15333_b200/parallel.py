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


# ---------------------------------------------------------------------------
# Fused update + collective over peer memory (NVLink / NVSwitch, one node)

def owned_rows(capacity: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [lo, hi) whose update rank ``rank`` owns (64-row aligned blocks)."""
    cuts = chunk_bounds(capacity, world)
    cuts += [(capacity, capacity)] * (world - len(cuts))
    return cuts[rank]


def rmsprop_step_peers(payload_sigma, payload_sh, grad_sigma, grad_sh, touched, rank: int, state,
                       rows: tuple[int, int], sh_stride: int, n_sh: int, consume: bool = True,
                       stream=None) -> None:
    """One rank's share of the fused data-parallel update (dot_rmsprop_step_peers):
    for rows [lo, hi) sum the W ranks' partial gradients (rank order, f64),
    apply RMSProp with this rank's second moments (``state.v_*``), write the
    updated rows into all W payload replicas and zero the consumed gradient
    rows.  The five arguments are length-W lists of device pointers (ints)
    or tensors, index r = rank r's buffer as mapped on this GPU."""
    from . import _lib
    world = len(payload_sigma)
    pr = _lib.DotPeerRows()
    for r in range(world):
        for name, arr in (("sigma", payload_sigma), ("sh", payload_sh), ("grad_sigma", grad_sigma),
                          ("grad_sh", grad_sh), ("touched", touched)):
            x = arr[r]
            getattr(pr, name)[r] = int(x.data_ptr()) if hasattr(x, "data_ptr") else int(x)
    pr.world, pr.rank = world, rank
    lo, hi = rows
    _lib.call("dot_rmsprop_step_peers", _lib.ctypes.byref(pr), sh_stride, n_sh, sh_stride,
              _lib.ptr(state.v_sigma), _lib.ptr(state.v_sh), lo, hi, state.beta, state.eps,
              state.lr_sigma, state.lr_sh, 1 if consume else 0, _lib.stream_ptr(stream))


class PeerExchange:
    """``train_step(exchange=...)`` for N > 1 GPUs of one node without NCCL
    on the data path: the payload replica and the gradient buffers of every
    rank live in torch symmetric memory (peer-mapped over NVLink), and after
    a device-side barrier each rank runs ``rmsprop_step_peers`` over the rows
    it owns -- reduce-scatter, update and all-gather fused in one kernel --
    followed by a second barrier before the next backward.  The second
    moments are current only on each row's owner; ``sync_state`` all-gathers
    them (needed before ``RmsPropState.remap`` at a refine)."""

    def __init__(self, tree, state, step_ws, group=None):
        import torch.distributed._symmetric_memory as symm_mem
        self.tree, self.state, self.ws = tree, state, step_ws.ws
        self.group = group if group is not None else dist.group.WORLD
        self.world, self.rank = dist.get_world_size(self.group), dist.get_rank(self.group)
        dev, cap, S = tree.device, tree.capacity, tree.sh_stride

        def sym(shape, dtype, init=None):
            t = symm_mem.empty(*shape, dtype=dtype, device=dev)
            t.copy_(init) if init is not None else t.zero_()
            return t, symm_mem.rendezvous(t, self.group)

        self._bufs = {}
        for name, shape, dtype, init in (("sigma", (cap,), torch.float32, tree._sigma),
                                         ("sh", (cap, S), torch.float32, tree._sh_store),
                                         ("gsig", (cap,), torch.float32, None),
                                         ("gsh", (cap, S), torch.float32, None),
                                         ("touched", (cap,), torch.uint8, None)):
            self._bufs[name] = sym(shape, dtype, init)
        tree._sigma, tree._sh_store = self._bufs["sigma"][0], self._bufs["sh"][0]
        self.ws.dsigma, self.ws.dsh_store = self._bufs["gsig"][0], self._bufs["gsh"][0]
        self.ws.touched = self._bufs["touched"][0]
        self.rows = owned_rows(cap, self.rank, self.world)
        self.generation = tree.generation
        self._ptrs = {k: list(h.buffer_ptrs) for k, (_, h) in self._bufs.items()}

    def _barrier(self):
        self._bufs["touched"][1].barrier()

    def __call__(self, update=None) -> None:
        if self.tree.generation != self.generation:
            raise RuntimeError("tree was refined: build a new PeerExchange")
        self._barrier()  # every rank's backward has landed
        rmsprop_step_peers(self._ptrs["sigma"], self._ptrs["sh"], self._ptrs["gsig"], self._ptrs["gsh"],
                           self._ptrs["touched"], self.rank, self.state, self.rows, self.tree.sh_stride,
                           3 * self.tree.basis_count)
        self._barrier()  # every replica is updated before the next backward reads it

    def sync_state(self) -> None:
        """All-gather the owners' second-moment rows into every rank's state."""
        for v in (self.state.v_sigma, self.state.v_sh):
            parts = [v[lo:hi].contiguous() for lo, hi in
                     (owned_rows(v.shape[0], r, self.world) for r in range(self.world))]
            dist.all_gather(parts, parts[self.rank].clone(), group=self.group)
            for (lo, hi), p in zip((owned_rows(v.shape[0], r, self.world) for r in range(self.world)), parts):
                v[lo:hi].copy_(p)
