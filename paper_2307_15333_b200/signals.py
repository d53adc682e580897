"""Per-leaf training signals over one calibration interval.

Same semantics as ``octrf.signals`` (/root/reference/pkg/src/octrf/signals.py:17-88):
the buffer sums each leaf's light contribution Q over every training ray of
the interval, is bound to one tree generation and must be reset after any
structural mutation.  The accumulator is a float64 tensor on the tree's
device (the backward kernel's per-leaf signal output adds into it).
"""

from __future__ import annotations

import enum

import numpy as np
import torch

from .errors import HandleError, InputError, StaleBufferError


class SignalTarget(enum.Enum):
    RAY_WEIGHT_Q = "q"
    DENSITY_SIGMA = "sigma"


class SignalBuffer:
    """Interval-windowed sum_r Q_{i,r} accumulator, bound to one topology."""

    def __init__(self, tree, target: SignalTarget = SignalTarget.RAY_WEIGHT_Q):
        self.target = SignalTarget(target)
        self._tree = tree
        self.accumulator = torch.zeros(0, dtype=torch.float64, device=tree.device)
        self.epoch_rays = 0
        self.generation = -1
        self.reset()

    @property
    def tree(self):
        return self._tree

    def reset(self) -> None:
        self.accumulator = torch.zeros(self._tree.capacity, dtype=torch.float64,
                                       device=self._tree.device)
        self.epoch_rays = 0
        self.generation = self._tree.generation

    def is_fresh(self) -> bool:
        return self.generation == self._tree.generation

    def check_fresh(self) -> None:
        if not self.is_fresh():
            raise StaleBufferError(
                f"signal buffer bound to generation {self.generation}, "
                f"tree is at {self._tree.generation}; reset() required")

    def accumulate(self, contributions, ray_count: int, validate: bool = True) -> None:
        """Add one batch's per-leaf Q contributions (signals.py:58-69).

        ``validate=False`` skips the negativity check, which costs a device
        synchronisation (the kernel never produces negative Q)."""
        self.check_fresh()
        c = torch.as_tensor(contributions, dtype=torch.float64).to(self.accumulator.device)
        if tuple(c.shape) != tuple(self.accumulator.shape):
            raise InputError(f"contribution array shape {tuple(c.shape)} does not match "
                             f"buffer shape {tuple(self.accumulator.shape)}")
        if validate and bool((c < 0).any()):
            raise InputError("negative Q contribution")
        self.accumulator += c
        self.epoch_rays += int(ray_count)


def signal_value(buffer: SignalBuffer, tree, leaf: int) -> float:
    return float(signal_values(buffer, tree, np.asarray([leaf]))[0])


def signal_values(buffer: SignalBuffer, tree, leaves) -> np.ndarray:
    if tree is not buffer.tree:
        raise InputError("buffer is bound to a different tree")
    buffer.check_fresh()
    leaves = np.asarray(leaves, dtype=np.int64)
    if leaves.size and not (tree._alive[leaves].all() and tree._leaf[leaves].all()):
        raise HandleError("signal lookup on a dead or internal node")
    if buffer.target is SignalTarget.DENSITY_SIGMA:
        return tree.sigma.detach().cpu().numpy()[leaves].astype(np.float64)
    return buffer.accumulator.detach().cpu().numpy()[leaves].copy()
