"""Host-fed training batches: double-buffered pinned-host -> HBM staging.

The reference trains from numpy ray arrays in host memory
(``optim.py:138-154`` slices ``dataset.origins/dirs/targets`` per batch).  On
the GPU every batch costs a 72 B/ray host->device copy (fp64 origin,
direction, target) -- about 1.3 ms for a 2^20-ray batch over PCIe, a third of
the fused step.  ``RayBatchStager`` moves that copy onto a side copy stream so
batch k+1 is in flight while batch k renders, back-propagates and updates:

    stager = RayBatchStager(device, max_rays=n)
    stager.stage(o_host[0], d_host[0], t_host[0])
    for k in range(steps):
        o, d, t = stager.take()                       # compute stream waits for the copy
        if k + 1 < steps:
            stager.stage(o_host[k + 1], d_host[k + 1], t_host[k + 1])
        loss, grads, sig = render_and_backprop(tree, o, d, t, ...)
        rmsprop_step(tree, grads, state)
        stager.release()                              # slot reusable once this step is done
        losses.push(loss)                             # LossReader: lagged D2H read

Source tensors should be pinned (``tensor.pin_memory()``); pageable sources
are accepted but the copy then serialises with the host.  Slots are recycled
only after the compute stream has passed the ``release`` fence, so a staged
batch can never overwrite rays a running kernel still reads.
"""

from __future__ import annotations

from collections import deque

import numpy as np
import torch

from .errors import InputError


class _Slot:
    __slots__ = ("bufs", "n", "ready", "free", "busy", "plan", "cost", "ids", "meta", "plan_args", "plan_out")

    def __init__(self):
        self.bufs = None
        self.cost = None
        self.ids = None
        self.meta = torch.cuda.Event()  # costs and ids copied (all a ranked plan reads)
        self.plan_args = None           # a plan not launched yet (plan_next / take_with_plan)
        self.plan_out = None            # the slot's plan index / warp order (reused with the slot)
        self.plan = None
        self.n = 0
        self.ready = torch.cuda.Event()
        self.free = None
        self.busy = False


class RayBatchStager:
    """Double-buffered (``depth`` slots) host->HBM staging of ray batches."""

    def __init__(self, device, max_rays: int = 0, depth: int = 2, plan_tree=None, plan_rank=None):
        """``plan_tree``: also compute each staged batch's coherence order
        (render.plan_batch) on the copy stream right after its copy, so the
        step that takes it skips the key sort (``take_with_plan``).
        ``plan_rank`` (render.PoolRank of the host dataset, e.g.
        ``pool_rank`` of its rays computed once): batches staged with their
        dataset ``ids`` are ordered by the rank without a sort
        (``dot_plan_ranked`` in slot mode)."""
        if depth < 2:
            raise InputError("depth must be >= 2 for copy/compute overlap")
        self.device = torch.device(device)
        self.plan_tree = plan_tree
        self.plan_rank = plan_rank
        self.plan_stream = None
        self.copy_stream = torch.cuda.Stream(self.device)
        self.slots = [_Slot() for _ in range(depth)]
        self.pending: deque[int] = deque()
        self.in_use: deque[int] = deque()
        self.next_slot = 0
        self.bytes_staged = 0
        if max_rays:
            for s in self.slots:
                self._ensure(s, max_rays)

    def _ensure(self, slot: _Slot, n: int) -> None:
        if slot.bufs is None or slot.bufs[0].shape[0] < n:
            # allocated on (and owned by) the compute stream, never freed while
            # a copy or kernel may touch it: the free/ready events order all uses
            torch.cuda.current_stream(self.device).synchronize()
            slot.bufs = tuple(torch.empty(n, 3, dtype=torch.float64, device=self.device) for _ in range(3))
            slot.cost = torch.empty(n, dtype=torch.int16, device=self.device)
            slot.ids = torch.empty(n, dtype=torch.int64, device=self.device)
            slot.plan_out = (torch.empty(n, dtype=torch.int64, device=self.device),
                             torch.empty((n + 31) // 32, dtype=torch.int32, device=self.device))

    @staticmethod
    def _host(x, name: str) -> torch.Tensor:
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
        if t.device.type != "cpu":
            raise InputError(f"{name}: RayBatchStager stages host tensors (got {t.device})")
        t = t.reshape(-1, 3)
        if t.dtype != torch.float64:
            t = t.double()
        return t.contiguous()

    def stage(self, origins, dirs, targets, costs=None, ids=None) -> None:
        """Queue the H2D copy of one batch on the copy stream (returns at once).
        ``costs`` (host int16 per ray, optional, e.g. a slice of
        ``render.ray_costs`` kept with the dataset): staged too and used for the
        batch's warp launch order (``plan_batch(costs=)``).  ``ids`` (host
        int64 per ray, optional): the rays' dataset ids, staged too; with
        ``plan_rank`` the batch is ordered by the dataset's rank."""
        o, d, t = (self._host(x, nm) for x, nm in ((origins, "origins"), (dirs, "dirs"), (targets, "targets")))
        n = o.shape[0]
        if d.shape[0] != n or t.shape[0] != n:
            raise InputError(f"batch length mismatch: {n} origins, {d.shape[0]} dirs, {t.shape[0]} targets")
        c = None
        if costs is not None:
            c = costs if isinstance(costs, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(costs))
            if c.device.type != "cpu" or c.dtype != torch.int16 or c.numel() != n:
                raise InputError("costs must be a host int16 tensor with one entry per ray")
        ih = None
        if ids is not None:
            ih = ids if isinstance(ids, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(ids))
            if ih.device.type != "cpu" or ih.dtype != torch.int64 or ih.numel() != n:
                raise InputError("ids must be a host int64 tensor with one entry per ray")
        i = self.next_slot
        slot = self.slots[i]
        if slot.busy:
            raise InputError("all staging slots are in flight: take()/release() before staging more")
        self._ensure(slot, n)
        ranked = self.plan_tree is not None and self.plan_rank is not None and ih is not None
        with torch.cuda.stream(self.copy_stream):
            if slot.free is not None:
                self.copy_stream.wait_event(slot.free)  # the last step reading this slot is done
            # costs and ids first: a ranked plan needs only them
            if c is not None:
                slot.cost[:n].copy_(c.reshape(-1), non_blocking=True)
            if ih is not None:
                slot.ids[:n].copy_(ih.reshape(-1), non_blocking=True)
            slot.meta.record(self.copy_stream)
            for dst, src in zip(slot.bufs, (o, d, t)):
                dst[:n].copy_(src, non_blocking=True)
            slot.plan = None
            slot.plan_args = (n, c is not None, ranked) if self.plan_tree is not None else None
            if self.plan_tree is not None and not ranked:  # key sort: needs the rays, right after the copy
                self._launch_plan(slot, self.copy_stream)
            slot.ready.record(self.copy_stream)
        slot.n = n
        slot.busy = True
        self.bytes_staged += 3 * n * 24 + (2 * n if c is not None else 0) + (8 * n if ih is not None else 0)
        self.pending.append(i)
        self.next_slot = (i + 1) % len(self.slots)

    def _launch_plan(self, slot: _Slot, stream, wait_current: bool = False) -> None:
        from .render import plan_batch
        n, has_cost, ranked = slot.plan_args
        slot.plan_args = None
        slot.plan = plan_batch(self.plan_tree, slot.bufs[0][:n], slot.bufs[1][:n], stream=stream,
                               wait_current=wait_current, costs=slot.cost[:n] if has_cost else None,
                               rank=self.plan_rank if ranked else None, ids=slot.ids[:n] if ranked else None,
                               out=slot.plan_out if ranked else None)

    def plan_next(self) -> None:
        """Launch the ranked plan of the most recently staged batch now, on the
        stager's plan stream, ordered after the work queued so far on the
        current stream and after the batch's costs / ids copies.  Call it once
        the current step's backward is queued (``train_step(after_backward=
        stager.plan_next)``): the plan then runs beside the optimizer update
        instead of the backward.  Without it ``take_with_plan`` launches the
        plan itself."""
        if not self.pending:
            return
        slot = self.slots[self.pending[-1]]
        if slot.plan_args is None:
            return
        if self.plan_stream is None:
            self.plan_stream = torch.cuda.Stream(self.device)
        self.plan_stream.wait_event(slot.meta)
        self._launch_plan(slot, self.plan_stream, wait_current=True)

    def take(self):
        """Device (origins, dirs, targets) of the oldest staged batch; the
        current stream waits for its copy (no host synchronisation)."""
        if not self.pending:
            raise InputError("take() with no staged batch")
        i = self.pending.popleft()
        slot = self.slots[i]
        torch.cuda.current_stream(self.device).wait_event(slot.ready)
        self.in_use.append(i)
        return tuple(b[:slot.n] for b in slot.bufs)

    def take_with_plan(self):
        """``take()`` plus the batch's coherence plan (None without plan_tree)."""
        i = self.pending[0] if self.pending else None
        if i is not None and self.slots[i].plan_args is not None:  # not launched by plan_next
            slot = self.slots[i]
            with torch.cuda.stream(self.copy_stream):
                self.copy_stream.wait_event(slot.meta)
                self._launch_plan(slot, self.copy_stream)
                slot.ready.record(self.copy_stream)
        out = self.take()
        return out + (self.slots[i].plan,)

    def release(self) -> None:
        """Mark the oldest taken batch consumed by the work queued so far."""
        if not self.in_use:
            raise InputError("release() without a taken batch")
        slot = self.slots[self.in_use.popleft()]
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        slot.free = ev
        slot.busy = False


class LossReader:
    """Per-step device->host loss read, lagged by one step so the host never
    stalls the queue: ``push(loss)`` starts the 8-byte copy of this step's loss
    and returns the PREVIOUS step's value (None on the first call);
    ``flush()`` returns the last one."""

    def __init__(self):
        self.host = [torch.empty((), dtype=torch.float64).pin_memory() for _ in range(2)]
        self.events = [torch.cuda.Event(), torch.cuda.Event()]
        self.k = 0
        self.values: list[float] = []
        self.stream = None  # the 8-byte copies run on their own stream, off the compute queue

    def push(self, loss: torch.Tensor):
        j = self.k % 2
        if self.stream is None:
            self.stream = torch.cuda.Stream(loss.device)
        self.stream.wait_stream(torch.cuda.current_stream(loss.device))
        with torch.cuda.stream(self.stream):
            self.host[j].copy_(loss.detach().reshape(()), non_blocking=True)
            self.events[j].record(self.stream)
        loss.record_stream(self.stream)
        prev = None
        if self.k > 0:
            p = (self.k - 1) % 2
            self.events[p].synchronize()
            prev = float(self.host[p])
            self.values.append(prev)
        self.k += 1
        return prev

    def flush(self):
        if self.k == 0:
            return None
        p = (self.k - 1) % 2
        self.events[p].synchronize()
        v = float(self.host[p])
        self.values.append(v)
        return v


__all__ = ["RayBatchStager", "LossReader"]
