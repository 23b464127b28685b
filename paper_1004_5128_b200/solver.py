"""Reference-compatible solver API on the B200 stepper.

Mirror of /root/reference/pkg/src/fracgrid/solver.py: same ``SimulationConfig``
(fields, validation, messages, ``StabilityWarning``), ``SimulationResult``,
``DivergenceError`` and the three entry points ``run`` / ``step`` /
``history_sum`` — but every step is one fused sm_100a kernel over an
HBM-resident history.  ``run`` also accepts the reference's own
``fracgrid.solver.SimulationConfig`` (duck-typed), so rebinding
``fracgrid.benchmark.run`` / ``fracgrid.cli.run`` to this ``run`` swaps the
engine under the reference's drivers.

Differences that are allowed by the parity contract: the history sum is
FMA-accumulated in a different order (fields agree to ≤1e-10 relative; ψ,
schedules and the stencil are bit-exact), and ``elapsed_seconds`` is device
time of the stepping loop measured with a synchronise on both sides.
"""

from __future__ import annotations

import ctypes as C
import math
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._engine import (
    DEFAULT_HISTORY_BYTE_CAP,
    DivergenceError,
    HistoryCapacityError,
    Problem,
    Stepper,
    divergence,
    error_class,
    host_scalars,
    short_horizon,
    strategy_spec,
)
from .coefficients import PsiTable
from .grid import Grid2D, HistoryBuffer
from .schedule import FullMemory, MemorySchedule, MemoryStrategy

__all__ = ["STABILITY_LIMIT", "DivergenceError", "StabilityWarning", "SimulationConfig", "SimulationResult",
           "history_sum", "step", "run", "problem_from_config"]

STABILITY_LIMIT = 0.25  # solver.py:35


class StabilityWarning(UserWarning):
    """The explicit-step stability heuristic is exceeded; results may blow up."""


@dataclass(frozen=True)
class SimulationConfig:
    """Fully-resolved parameters of one 2D run (solver.py:53-145)."""

    gamma: float
    alpha: float
    beta: float
    dt: float
    dx: float
    nx: int
    ny: int
    n_steps: int
    sources: tuple[tuple[int, int, float], ...] = ()
    strategy: MemoryStrategy = field(default_factory=FullMemory)
    snapshot_every: int | None = None
    history_byte_cap: int | None = DEFAULT_HISTORY_BYTE_CAP

    def __post_init__(self) -> None:
        if not 0.0 < self.gamma <= 1.0:
            raise ValueError(f"gamma must lie in (0, 1], got {self.gamma!r}")
        if not self.alpha >= 0.0 or not math.isfinite(self.alpha):
            raise ValueError(f"alpha must be finite and >= 0, got {self.alpha!r}")
        if not self.beta >= 0.0 or not math.isfinite(self.beta):
            raise ValueError(f"beta must be finite and >= 0, got {self.beta!r}")
        if not self.dt > 0.0 or not math.isfinite(self.dt):
            raise ValueError(f"dt must be positive and finite, got {self.dt!r}")
        if not self.dx > 0.0 or not math.isfinite(self.dx):
            raise ValueError(f"dx must be positive and finite, got {self.dx!r}")
        if self.nx < 3 or self.ny < 3:
            raise ValueError(f"grid must be at least 3x3, got {self.nx}x{self.ny}")
        if self.n_steps < 0:
            raise ValueError(f"n_steps must be >= 0, got {self.n_steps}")
        if self.snapshot_every is not None and self.snapshot_every < 1:
            raise ValueError(f"snapshot_every must be >= 1, got {self.snapshot_every}")
        seen: set[tuple[int, int]] = set()
        for j, l, value in self.sources:
            if not (1 <= j <= self.nx - 2 and 1 <= l <= self.ny - 2):
                raise ValueError(f"source ({j}, {l}) is outside the interior of a {self.nx}x{self.ny} grid")
            if not math.isfinite(value):
                raise ValueError(f"source ({j}, {l}) has non-finite value {value!r}")
            if (j, l) in seen:
                raise ValueError(f"duplicate source at ({j}, {l})")
            seen.add((j, l))
        if self.stability_ratio > STABILITY_LIMIT:
            warnings.warn(
                f"stability ratio alpha*dt**gamma/dx**2 = {self.stability_ratio:.4g} "
                f"exceeds {STABILITY_LIMIT}; the explicit step may diverge",
                StabilityWarning,
                stacklevel=2,
            )

    @property
    def stability_ratio(self) -> float:
        return self.alpha * self.dt**self.gamma / self.dx**2

    @property
    def snapshot_cadence(self) -> int:
        if self.snapshot_every is not None:
            return self.snapshot_every
        return max(1, math.ceil(self.n_steps / 100))

    def initial_grid(self) -> Grid2D:
        return Grid2D.from_sources(self.nx, self.ny, self.dx, self.sources)


@dataclass(frozen=True)
class SimulationResult:
    """Snapshots, final state and stepping-loop time of one run (solver.py:148-159)."""

    config: object
    snapshots: tuple[tuple[int, Grid2D], ...]
    final: Grid2D
    elapsed_seconds: float

    @property
    def n_steps(self) -> int:
        return self.config.n_steps


def _cadence(config) -> int:
    cad = getattr(config, "snapshot_cadence", None)
    if cad is not None:
        return int(cad)
    if config.snapshot_every is not None:
        return int(config.snapshot_every)
    return max(1, math.ceil(config.n_steps / 100))


def problem_from_config(config) -> Problem:
    """Normalise a (reference or local) ``SimulationConfig`` into an engine problem."""
    grid = config.initial_grid()
    kind, param = strategy_spec(config.strategy)
    return Problem(
        u0=np.asarray(grid.data, dtype=np.float64)[None],
        gamma=np.array([float(config.gamma)]),
        dt=np.array([float(config.dt)]),
        alpha=float(config.alpha),
        dx=float(config.dx),
        reaction=("linear", float(config.beta)),
        kind=kind,
        param=param,
        n_steps=int(config.n_steps),
        cadence=_cadence(config),
        history_byte_cap=config.history_byte_cap,
    )


def run(config, *, progress_every: int = 0) -> SimulationResult:
    """Run a complete simulation on the GPU (solver.py:230-265 semantics).

    Snapshots at step 0, every ``snapshot_cadence`` steps and the final step;
    ``progress_every`` > 0 logs ``step k/n`` on the ``fracgrid`` logger.  Raises
    ``DivergenceError(step, peak)`` for the first non-finite step and
    ``MemoryBudgetError`` before allocating an over-cap history.
    """
    prob = problem_from_config(config)
    stepper = Stepper(prob)
    elapsed = stepper.run(progress_every=progress_every)
    snaps = [(s, Grid2D(u[0], config.dx)) for s, u in stepper.fetch_snapshots()]
    return SimulationResult(config=config, snapshots=tuple(snaps), final=snaps[-1][1], elapsed_seconds=elapsed)


# --------------------------------------------------------------------------------
# single-step building blocks (device equivalents of solver.py:162-227)

def _to_device_i64(a, dev):
    import torch

    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int64), device=dev)


def history_sum(history: HistoryBuffer, schedule: MemorySchedule, table: PsiTable, k: int):
    """S_k = Σ w·ψ(m)·δ[k-m] on the device (solver.py:162-197).

    Same validation and errors as the reference; the result is a device tensor of
    the field shape (reduction order differs: FMA, newest first).
    """
    import torch

    k = int(k)
    if k < 0 or len(history) <= k:
        raise ValueError(f"step {k} needs {k + 1} history entries, buffer holds {len(history)}")
    offsets = np.asarray(schedule.offsets, dtype=np.int64)
    weights = np.asarray(schedule.weights, dtype=np.int64)
    oldest = int(offsets[-1])
    if oldest > k:
        raise ValueError(f"schedule reaches offset {oldest}, beyond step {k}")
    if oldest > table.capacity:
        raise ValueError(f"psi table covers offsets up to {table.capacity}, schedule needs {oldest}")
    dev = history.device
    out = torch.empty(history.ms, dtype=torch.float64, device=dev)
    n = int(np.prod(history.field_shape))
    o = _to_device_i64(offsets, dev)
    w = _to_device_i64(weights, dev)
    _lib.check(_lib.load().fg_history_sum(history.storage.data_ptr(), history.ms, n, o.data_ptr(), w.data_ptr(),
                                          int(offsets.size), table.values.data_ptr(), table.capacity + 1, k,
                                          out.data_ptr(), _lib.stream_handle()), "fg_history_sum")
    return out[:n].reshape(history.field_shape)


def step(u, history: HistoryBuffer, k: int, config, table: PsiTable):
    """Advance u^k → u^{k+1} and append stencil(u^{k+1}) (solver.py:200-227).

    One fused-step kernel (schedule generated on the device from
    ``config.strategy``), then the stencil kernel for the append.  Raises
    ``DivergenceError(k+1, peak)`` and leaves the history untouched if the new
    field is non-finite.  Returns the same array type it was given.
    """
    import torch

    k = int(k)
    is_np = not isinstance(u, torch.Tensor)
    kind, param = strategy_spec(config.strategy)
    sched = config.strategy.schedule_at(k, config.dt)
    if k < 0 or len(history) <= k:
        raise ValueError(f"step {k} needs {k + 1} history entries, buffer holds {len(history)}")
    oldest = int(np.asarray(sched.offsets)[-1])
    if oldest > table.capacity:
        raise ValueError(f"psi table covers offsets up to {table.capacity}, schedule needs {oldest}")
    dev = history.device
    shape = history.field_shape
    n = int(np.prod(shape))
    f64 = dict(dtype=torch.float64, device=dev)
    fields = torch.zeros((2, history.ms), **f64)
    fields[k & 1, :n] = torch.as_tensor(np.asarray(u, dtype=np.float64) if is_np else u, **f64).reshape(-1)
    decay, diffuse = host_scalars(config.alpha, config.beta, config.gamma, config.dt, config.dx)
    decay_t = torch.tensor([decay], **f64)
    diffuse_t = torch.tensor([diffuse], **f64)
    dt_t = torch.tensor([float(config.dt)], **f64)
    hz = torch.tensor([short_horizon(param, config.dt) if kind == "short" else 0], dtype=torch.int64, device=dev)
    status = torch.full((2,), _lib.FG_NO_BAD_STEP, dtype=torch.int64, device=dev)
    from .grid import field_plan

    plan = field_plan(shape)
    plan.reaction = 0
    plan.kind = _lib.MEM_KINDS[kind]
    plan.base = int(param) if kind == "adaptive" else 0
    plan.horizon_dev = hz.data_ptr()
    plan.psi_dev = table.values.data_ptr()
    plan.psi_stride = table.capacity + 1
    plan.decay_dev, plan.diffuse_dev, plan.dt_dev = decay_t.data_ptr(), diffuse_t.data_ptr(), dt_t.data_ptr()
    plan.H_dev = history.storage.data_ptr()
    plan.h_slices = history.capacity
    plan.u_dev[0], plan.u_dev[1] = fields[0].data_ptr(), fields[1].data_ptr()
    plan.status_dev = status.data_ptr()
    plan.step_flags = _lib.FG_STEP_M0_FROM_HISTORY
    L = _lib.load()
    st = _lib.stream_handle()
    _lib.check(L.fg_step(C.byref(plan), k, None, st), "fg_step")
    nxt = fields[(k + 1) & 1]
    bad = int(status[0].item())
    if bad != _lib.FG_NO_BAD_STEP:
        view = nxt[:n]
        fin = view[torch.isfinite(view)]
        peak = float(fin.abs().max().item()) if fin.numel() else math.inf
        raise divergence(bad, peak)
    # append at len(history) after the divergence check, like HistoryBuffer.append
    # in solver.py:222-226 (a full buffer raises only once the step is known good)
    at = len(history)
    if at >= history.capacity:
        raise error_class(HistoryCapacityError)(f"buffer holds {history.capacity} entries and is full")
    _lib.check(L.fg_stencil(C.byref(plan), nxt.data_ptr(), history.storage[at].data_ptr(), st), "fg_stencil")
    history._mark(at + 1)
    res = nxt[:n].reshape(shape).clone()
    return res.cpu().numpy() if is_np else res
