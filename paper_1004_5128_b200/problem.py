"""Additive extension of the reference API: 1D/3D grids, nonlinear reaction, ensembles.

The reference solver is 2D / five-point / linear decay only
(/root/reference/pkg/src/fracgrid/solver.py:95-106, grid.py:95-97); BASELINE.json
also asks for 1D (c1), 3D with a saturating reaction (c4) and a batched ensemble
with per-member γ and Δt (c5).  ``FieldConfig`` + :func:`run_field` cover those
on the same engine, with the same semantics as ``solver.run``: snapshots at 0 /
every cadence / final, ``DivergenceError`` on the first non-finite step,
``MemoryBudgetError`` before allocation, loop-only ``elapsed_seconds``.

Update forms (rounding order is part of the contract):
    LinearDecay(beta):      u*(1 - beta*dt) + diffuse*S          (the reference's form)
    Saturating(vmax, km):   u + dt*f(u) + diffuse*S,  f(u) = -vmax*u/(km+u)
with diffuse = alpha*dt**gamma/dx**2 evaluated per member on the host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Sequence, Union

import numpy as np

from ._engine import DEFAULT_HISTORY_BYTE_CAP, Problem, Stepper, strategy_spec
from .schedule import FullMemory, MemoryStrategy


@dataclass(frozen=True)
class LinearDecay:
    beta: float = 0.0

    def spec(self) -> tuple:
        if not self.beta >= 0.0 or not math.isfinite(self.beta):
            raise ValueError(f"beta must be finite and >= 0, got {self.beta!r}")
        return ("linear", float(self.beta))


@dataclass(frozen=True)
class Saturating:
    """f(u) = -vmax·u/(km + u) (Michaelis–Menten consumption)."""

    vmax: float
    km: float

    def spec(self) -> tuple:
        if not (math.isfinite(self.vmax) and math.isfinite(self.km) and self.km > 0.0):
            raise ValueError(f"saturating reaction needs finite vmax and km > 0, got {self!r}")
        return ("saturating", float(self.vmax), float(self.km))


Reaction = Union[LinearDecay, Saturating]


def _ring_is_zero(u: np.ndarray) -> bool:
    for ax in range(u.ndim):
        if np.any(np.take(u, 0, axis=ax) != 0.0) or np.any(np.take(u, -1, axis=ax) != 0.0):
            return False
    return True


@dataclass(frozen=True)
class FieldConfig:
    """One run on a 1-3 dimensional grid, optionally an ensemble of members.

    ``initial`` has shape ``shape`` (single problem) or ``(B, *shape)`` with
    ``batched=True``.  ``gamma`` / ``dt`` are scalars or per-member sequences.
    Every member's boundary faces must be exactly zero (Dirichlet u = 0).
    """

    initial: np.ndarray
    dx: float
    gamma: Union[float, Sequence[float]]
    dt: Union[float, Sequence[float]]
    n_steps: int
    alpha: float = 1.0
    reaction: Reaction = field(default_factory=LinearDecay)
    strategy: MemoryStrategy = field(default_factory=FullMemory)
    batched: bool = False
    snapshot_every: int | None = None
    history_byte_cap: int | None = DEFAULT_HISTORY_BYTE_CAP

    def members(self) -> int:
        return int(np.asarray(self.initial).shape[0]) if self.batched else 1

    @property
    def snapshot_cadence(self) -> int:
        if self.snapshot_every is not None:
            return int(self.snapshot_every)
        return max(1, math.ceil(self.n_steps / 100))

    def to_problem(self) -> Problem:
        u0 = np.asarray(self.initial, dtype=np.float64)
        if not self.batched:
            u0 = u0[None]
        B = u0.shape[0]
        if not 1 <= u0.ndim - 1 <= 3:
            raise ValueError(f"fields must have 1-3 dimensions, got {u0.ndim - 1}")
        if any(s < 3 for s in u0.shape[1:]):
            raise ValueError(f"grid must be at least 3 points per axis, got {u0.shape[1:]}")
        if not np.isfinite(u0).all():
            raise ValueError("initial field contains non-finite values")
        for b in range(B):
            if not _ring_is_zero(u0[b]):
                raise ValueError("boundary ring must be exactly zero")
        gamma = np.broadcast_to(np.asarray(self.gamma, dtype=np.float64), (B,)).copy()
        dt = np.broadcast_to(np.asarray(self.dt, dtype=np.float64), (B,)).copy()
        if not np.all((gamma > 0.0) & (gamma <= 1.0)):
            raise ValueError(f"gamma must lie in (0, 1], got {self.gamma!r}")
        if not np.all(np.isfinite(dt) & (dt > 0.0)):
            raise ValueError(f"dt must be positive and finite, got {self.dt!r}")
        if not self.dx > 0.0 or not math.isfinite(self.dx):
            raise ValueError(f"dx must be positive and finite, got {self.dx!r}")
        if not self.alpha >= 0.0 or not math.isfinite(self.alpha):
            raise ValueError(f"alpha must be finite and >= 0, got {self.alpha!r}")
        if int(self.n_steps) < 0:
            raise ValueError(f"n_steps must be >= 0, got {self.n_steps}")
        if self.snapshot_every is not None and self.snapshot_every < 1:
            raise ValueError(f"snapshot_every must be >= 1, got {self.snapshot_every}")
        kind, param = strategy_spec(self.strategy)
        return Problem(u0=u0, gamma=gamma, dt=dt, alpha=float(self.alpha), dx=float(self.dx),
                       reaction=self.reaction.spec(), kind=kind, param=param, n_steps=int(self.n_steps),
                       cadence=self.snapshot_cadence, history_byte_cap=self.history_byte_cap)


@dataclass(frozen=True)
class FieldResult:
    """Snapshots ``(step, array)`` with arrays shaped like ``config.initial``."""

    config: FieldConfig
    snapshots: tuple
    final: np.ndarray
    elapsed_seconds: float


def run_field(config: FieldConfig, *, progress_every: int = 0, split: int = 0, flags: int | None = None,
              tblock: int | None = None) -> FieldResult:
    """Run an n-D / batched problem on the GPU (solver.run semantics).

    ``flags`` / ``split`` / ``tblock`` select the launch pipeline, the warp split
    of the history sum and the temporal blocking factor; all
    choices agree with the reference within the 1e-10 parity bound.
    """
    prob = config.to_problem()
    stepper = Stepper(prob, split=split, flags=flags, tblock=tblock)
    elapsed = stepper.run(progress_every=progress_every)
    snaps = stepper.fetch_snapshots()
    if not config.batched:
        snaps = [(s, u[0]) for s, u in snaps]
    snaps = tuple(snaps)
    return FieldResult(config=config, snapshots=snaps, final=snaps[-1][1], elapsed_seconds=elapsed)
