"""Memory schedules: the strategy plug-ins and the device schedule generator.

Mirror of /root/reference/pkg/src/fracgrid/schedule.py.  The strategy objects
(``FullMemory`` / ``ShortMemory`` / ``AdaptiveMemory``, :198-254) keep the
reference's protocol — ``.tag``, ``.param``, ``.schedule_at(k, dt)`` — and the
fused step kernel regenerates the same schedule on the device every step
(``fg_segments`` in csrc/fg_schedule.cuh).  ``schedule_at`` here asks that same
device generator (``fg_schedule_expand``) and wraps the result in a validated
:class:`MemorySchedule`, so what a user inspects is what the kernel visits.
Any object with a matching ``.tag`` / ``.length`` / ``.base`` (e.g. the
reference's own strategies) is accepted by :func:`solver.run`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Union

import numpy as np

from . import _lib


@dataclass(frozen=True)
class MemorySchedule:
    """Weighted history offsets of one backward sum (schedule.py:21-60)."""

    offsets: np.ndarray
    weights: np.ndarray

    def __post_init__(self) -> None:
        offsets = np.asarray(self.offsets, dtype=np.int64)
        weights = np.asarray(self.weights, dtype=np.int64)
        if offsets.ndim != 1 or weights.ndim != 1 or offsets.size != weights.size:
            raise ValueError("offsets and weights must be 1D arrays of equal length")
        if offsets.size == 0:
            raise ValueError("a schedule must contain at least one entry")
        if offsets[0] < 0:
            raise ValueError("offsets must be >= 0")
        if offsets.size > 1 and not np.all(np.diff(offsets) > 0):
            raise ValueError("offsets must be strictly increasing")
        if np.any(weights < 1):
            raise ValueError("weights must be positive integers")
        offsets.setflags(write=False)
        weights.setflags(write=False)
        object.__setattr__(self, "offsets", offsets)
        object.__setattr__(self, "weights", weights)

    def __len__(self) -> int:
        return int(self.offsets.size)

    def pairs(self) -> list[tuple[int, int]]:
        return [(int(m), int(w)) for m, w in zip(self.offsets, self.weights)]

    @property
    def weight_sum(self) -> int:
        return int(self.weights.sum())


def _checked_step(k: int) -> int:
    k = int(k)
    if k < 0:
        raise ValueError(f"step index k must be >= 0, got {k}")
    return k


def device_schedules(kind: str, k0: int, nk: int, *, base: int = 0, horizon: int = 0, row_cap: int | None = None):
    """Expand schedule(k) for k = k0..k0+nk-1 on the device.

    Returns device tensors (offsets int32 [nk, row_cap], weights int32 [nk, row_cap],
    lens int64 [nk]).  Used by the parity tests to compare every step's schedule
    with the reference bit for bit.
    """
    import torch

    dev = _lib.require_cuda()
    L = _lib.load()
    if row_cap is None:
        import ctypes as C

        n = C.c_int64(0)
        _lib.check(L.fg_schedule_len(_lib.MEM_KINDS[kind], k0 + nk - 1, base, horizon, C.byref(n)))
        row_cap = max(1, int(n.value))
        # lengths are not monotone in k for adaptive memory; take a safe bound
        row_cap = max(row_cap, k0 + nk) if kind == "adaptive" else row_cap
    offs = torch.empty((nk, row_cap), dtype=torch.int32, device=dev)
    wts = torch.empty((nk, row_cap), dtype=torch.int32, device=dev)
    lens = torch.empty((nk,), dtype=torch.int64, device=dev)
    _lib.check(L.fg_schedule_expand(_lib.MEM_KINDS[kind], k0, nk, base, horizon, offs.data_ptr(), wts.data_ptr(),
                                    row_cap, lens.data_ptr(), _lib.stream_handle()), "fg_schedule_expand")
    return offs, wts, lens


def _device_schedule(kind: str, k: int, base: int = 0, horizon: int = 0) -> MemorySchedule:
    offs, wts, lens = device_schedules(kind, k, 1, base=base, horizon=horizon)
    n = int(lens[0].item())
    return MemorySchedule(offsets=offs[0, :n].cpu().numpy().astype(np.int64),
                          weights=wts[0, :n].cpu().numpy().astype(np.int64))


def full_schedule(k: int) -> MemorySchedule:
    """schedule.py:70-76."""
    return _device_schedule("full", _checked_step(k))


def short_schedule(k: int, length: float, dt: float) -> MemorySchedule:
    """schedule.py:79-94 (horizon floor(length/dt) evaluated on the host, as there)."""
    k = _checked_step(k)
    if not length > 0 or not math.isfinite(length):
        raise ValueError(f"memory length must be positive and finite, got {length!r}")
    if not dt > 0 or not math.isfinite(dt):
        raise ValueError(f"dt must be positive and finite, got {dt!r}")
    horizon = min(int(math.floor(length / dt)), 1 << 62)
    return _device_schedule("short", k, horizon=horizon)


def adaptive_schedule(k: int, base: int) -> MemorySchedule:
    """schedule.py:97-151."""
    k = _checked_step(k)
    base = int(base)
    if base < 2:
        raise ValueError(f"adaptive base must be >= 2, got {base}")
    return _device_schedule("adaptive", k, base=base)


@dataclass(frozen=True)
class FullMemory:
    """Visit the entire history every step (schedule.py:198-209)."""

    tag = "full"

    @property
    def param(self) -> float:
        return 0.0

    def schedule_at(self, k: int, dt: float) -> MemorySchedule:
        return full_schedule(k)


@dataclass(frozen=True)
class ShortMemory:
    """Visit only the most recent ``length`` units of simulation time (schedule.py:212-231)."""

    length: float
    tag = "short"

    def __post_init__(self) -> None:
        if not self.length > 0 or not math.isfinite(self.length):
            raise ValueError(f"short-memory length must be positive and finite, got {self.length!r}")
        object.__setattr__(self, "length", float(self.length))

    @property
    def param(self) -> float:
        return self.length

    def schedule_at(self, k: int, dt: float) -> MemorySchedule:
        return short_schedule(k, self.length, dt)


@dataclass(frozen=True)
class AdaptiveMemory:
    """Dense recent window of ``base`` steps, geometric thinning beyond it (schedule.py:234-254)."""

    base: int
    tag = "adaptive"

    def __post_init__(self) -> None:
        base = self.base
        if not isinstance(base, (int, np.integer)) or isinstance(base, bool):
            raise ValueError(f"adaptive base must be an integer, got {base!r}")
        if base < 2:
            raise ValueError(f"adaptive base must be >= 2, got {base}")
        object.__setattr__(self, "base", int(base))

    @property
    def param(self) -> float:
        return float(self.base)

    def schedule_at(self, k: int, dt: float) -> MemorySchedule:
        return adaptive_schedule(k, self.base)


MemoryStrategy = Union[FullMemory, ShortMemory, AdaptiveMemory]
