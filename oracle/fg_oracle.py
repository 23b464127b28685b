"""NumPy restatement of the reference GL history stepper — TEST INFRASTRUCTURE ONLY.

Checker for ``paper_1004_5128_b200`` (see ``oracle/__init__.py``).  Every function
cites the reference line(s) it restates; paths are relative to
``/root/reference/pkg/src/fracgrid/``.

Scope beyond the reference: the reference solver is 2D,
5-point, linear decay only.  BASELINE.json also asks for 1D, 3D, a saturating
reaction and a batched ensemble.  For those the restatement composes exactly the
reference's own pieces (ψ recursion, schedules, ``history_sum`` contraction,
update/append order) around an n-D stencil written in the same operation pattern
as ``grid.py:98-106``.  ``tests/golden/make_golden.py`` builds the same
composition out of the *imported* reference functions, which is what pins these
extensions.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "OracleDivergence",
    "OracleProblem",
    "psi",
    "build_table",
    "schedule_segments",
    "schedule",
    "stencil",
    "history_sum",
    "host_scalars",
    "run",
    "count_terms",
]


class OracleDivergence(RuntimeError):
    """Mirror of ``solver.DivergenceError`` (solver.py:38-46)."""

    def __init__(self, step: int, peak: float):
        super().__init__(f"solution diverged at step {step}: max |u| reached {peak!r}")
        self.step = step
        self.peak = peak


# --------------------------------------------------------------------------- ψ ---

def psi(gamma: float, m: int) -> float:
    """ψ(γ, m) by the two-term recursion — coefficients.py:30-51.

    Evaluated as ``((-v) * ((2.0 - γ) - m)) / m``, which is how Python parses the
    reference's ``-value * (2.0 - gamma - j) / j`` (each op one fp64 rounding).
    """
    v = 1.0
    for j in range(1, int(m) + 1):
        v = -v * (2.0 - gamma - j) / j
    return v


def build_table(gamma: float, n: int) -> np.ndarray:
    """ψ(γ, 0..n) in one sequential pass — coefficients.py:76-92 (bitwise = psi())."""
    gamma = float(gamma)
    if not (math.isfinite(gamma) and 0.0 < gamma < 2.0):
        raise ValueError(f"gamma must lie in the open interval (0.0, 2.0), got {gamma!r}")
    out = np.empty(int(n) + 1, dtype=np.float64)
    v = 1.0
    out[0] = v
    for j in range(1, int(n) + 1):
        v = -v * (2.0 - gamma - j) / j
        out[j] = v
    return out


# -------------------------------------------------------------------- schedules ---

def schedule_segments(kind: str, k: int, param: float = 0.0, dt: float = 1.0):
    """Schedule for step ``k`` as arithmetic segments ``(m0, count, stride)``.

    Weight equals stride in every segment (dense runs: 1/1; thinned intervals:
    2i-1 / 2i-1), so the segment list is the whole schedule.  Restates
    schedule.py:70-76 (full), :79-94 (short, horizon ``min(floor(L/dt), k)``) and
    :97-151 (adaptive, including the ``k > a**last_i`` tail branch at :137-141).
    """
    k = int(k)
    if k < 0:
        raise ValueError(f"step index k must be >= 0, got {k}")
    if kind == "full":
        return [(0, k + 1, 1)]
    if kind == "short":
        length = float(param)
        if not length > 0 or not math.isfinite(length):
            raise ValueError(f"memory length must be positive and finite, got {length!r}")
        if not dt > 0 or not math.isfinite(dt):
            raise ValueError(f"dt must be positive and finite, got {dt!r}")
        horizon = min(int(math.floor(length / dt)), k)
        return [(0, horizon + 1, 1)]
    if kind != "adaptive":
        raise ValueError(f"unknown memory kind {kind!r}")
    a = int(param)
    if a < 2:
        raise ValueError(f"adaptive base must be >= 2, got {a}")
    if k <= a:
        return [(0, k + 1, 1)]
    segs = [(0, a + 1, 1)]
    last = None  # (last sampled offset, its interval index i, a**i)
    i, a_prev = 2, a  # a_prev = a**(i-1)
    while True:
        start = a_prev + i
        if start > k:
            break
        a_i = a_prev * a
        stride = 2 * i - 1
        hi = min(a_i, k - i + 1)
        if hi >= start:
            count = (hi - start) // stride + 1
            segs.append((start, count, stride))
            last = (start + (count - 1) * stride, i, a_i)
        a_prev = a_i
        i += 1
    if last is None:
        tail = a + 1
    elif k > last[2]:
        tail = last[2] + 1
    else:
        tail = last[0] + last[1]
    if tail <= k:
        segs.append((tail, k - tail + 1, 1))
    return segs


def schedule(kind: str, k: int, param: float = 0.0, dt: float = 1.0):
    """Expanded ``(offsets, weights)`` int64 arrays — the ``MemorySchedule`` pair."""
    segs = schedule_segments(kind, k, param, dt)
    offs = np.concatenate([m0 + np.arange(n, dtype=np.int64) * s for m0, n, s in segs])
    wts = np.concatenate([np.full(n, s, dtype=np.int64) for _, n, s in segs])
    return offs, wts


def count_terms(kind: str, n_steps: int, param: float = 0.0, dt: float = 1.0) -> int:
    """Σ_k len_k over k = 0..n_steps-1 (history terms per grid point per run)."""
    return int(sum(sum(n for _, n, _ in schedule_segments(kind, k, param, dt))
                   for k in range(int(n_steps))))


# ---------------------------------------------------------------------- stencil ---

def stencil(u: np.ndarray) -> np.ndarray:
    """Discrete Laplacian numerator with a zero output ring, no /dx².

    2D is grid.py:88-106 verbatim in operation order:
    ``((((x+ + x-) - 4c) + y+) + y-)``.  1D / 3D follow the same left-to-right
    pattern: ``(x+ + x-) - 2c`` and ``((((((x+ + x-) - 6c) + y+) + y-) + z+) + z-)``.
    """
    u = np.asarray(u, dtype=np.float64)
    out = np.zeros_like(u)
    if u.ndim == 1:
        out[1:-1] = u[2:] + u[:-2] - 2.0 * u[1:-1]
    elif u.ndim == 2:
        out[1:-1, 1:-1] = (
            u[2:, 1:-1] + u[:-2, 1:-1] - 4.0 * u[1:-1, 1:-1] + u[1:-1, 2:] + u[1:-1, :-2]
        )
    elif u.ndim == 3:
        c = (slice(1, -1),) * 3
        out[c] = (
            u[2:, 1:-1, 1:-1] + u[:-2, 1:-1, 1:-1] - 6.0 * u[c]
            + u[1:-1, 2:, 1:-1] + u[1:-1, :-2, 1:-1]
            + u[1:-1, 1:-1, 2:] + u[1:-1, 1:-1, :-2]
        )
    else:
        raise ValueError(f"stencil supports 1-3 dimensions, got {u.ndim}")
    return out


def zero_ring(u: np.ndarray) -> None:
    """Pin every boundary face to zero in place — solver.py:218-221 generalised."""
    for ax in range(u.ndim):
        idx = [slice(None)] * u.ndim
        idx[ax] = 0
        u[tuple(idx)] = 0.0
        idx[ax] = -1
        u[tuple(idx)] = 0.0


# ------------------------------------------------------------------ history sum ---

def history_sum(H: np.ndarray, offsets: np.ndarray, weights: np.ndarray,
                table: np.ndarray, k: int) -> np.ndarray:
    """S_k = Σ w·ψ[m]·H[k-m] — solver.py:162-197.

    ``H`` is ``(T, *field)`` oldest first.  Coefficients ``w * ψ[m]`` (one
    rounding, :190).  Contiguous schedules 0..M contract the block H[k-M..k] with
    flipped coefficients (oldest first, :191-195); anything else gathers
    H[k-offsets] (newest first, :196-197).  Same ``np.einsum`` contraction.
    """
    offsets = np.asarray(offsets, dtype=np.int64)
    weights = np.asarray(weights, dtype=np.int64)
    oldest = int(offsets[-1])
    if oldest > k:
        raise ValueError(f"schedule reaches offset {oldest}, beyond step {k}")
    if oldest > table.size - 1:
        raise ValueError(f"psi table covers offsets up to {table.size - 1}, schedule needs {oldest}")
    coeffs = weights * table[offsets]
    flat = H.reshape(H.shape[0], -1)
    if int(offsets[0]) == 0 and oldest == offsets.size - 1:
        out = np.einsum("t,tn->n", coeffs[::-1], flat[k - oldest:k + 1])
    else:
        out = np.einsum("t,tn->n", coeffs, flat[k - offsets])
    return out.reshape(H.shape[1:])


# ---------------------------------------------------------------------- problem ---

@dataclass
class OracleProblem:
    """Fully resolved run, normalised to ``B`` members of one n-D field shape.

    ``u0`` has shape ``(B, *shape)``; ``gamma`` and ``dt`` are per member.
    ``reaction`` is ``("linear", beta)`` (the reference's decay form,
    solver.py:215) or ``("saturating", vmax, km)`` for f(u) = -vmax·u/(km+u).
    ``strategy`` is ``(kind, param)`` with kind in {full, short, adaptive}.
    """

    u0: np.ndarray
    gamma: np.ndarray
    dt: np.ndarray
    alpha: float
    dx: float
    reaction: tuple
    strategy: tuple
    n_steps: int
    snapshot_every: int | None = None
    extra: dict = field(default_factory=dict)

    @property
    def batch(self) -> int:
        return self.u0.shape[0]

    @property
    def cadence(self) -> int:
        """solver.py:137-142."""
        if self.snapshot_every is not None:
            return int(self.snapshot_every)
        return max(1, math.ceil(self.n_steps / 100))


def host_scalars(alpha: float, beta: float, gamma: float, dt: float, dx: float):
    """(decay, diffuse) exactly as solver.py:215-216 evaluates them (Python floats)."""
    decay = 1.0 - float(beta) * float(dt)
    diffuse = float(alpha) * float(dt) ** float(gamma) / float(dx) ** 2
    return decay, diffuse


def _update(u, acc, reaction, dt, decay, diffuse):
    """u_next before ring pinning — solver.py:215-217; saturating form per Appendix B."""
    if reaction[0] == "linear":
        return u * decay + diffuse * acc
    if reaction[0] == "saturating":
        vmax, km = float(reaction[1]), float(reaction[2])
        f = -vmax * u / (km + u)
        return u + dt * f + diffuse * acc
    raise ValueError(f"unknown reaction {reaction!r}")


def run(p: OracleProblem):
    """Restatement of ``solver.run`` (solver.py:230-265) for B members in lockstep.

    Members never interact; each has its own ψ table and history, and the
    contraction per member is exactly the reference's.  Returns a dict with
    ``snapshots`` [(step, (B,*shape) array)], ``final`` and ``elapsed_seconds``
    (stepping loop only, solver.py:248-257).  Raises OracleDivergence(k+1, peak)
    at the first step whose (whole-batch) field is non-finite (solver.py:222-225).
    """
    B = p.batch
    shape = p.u0.shape[1:]
    n = int(p.n_steps)
    kind, param = p.strategy
    tables = [build_table(float(p.gamma[b]), n) for b in range(B)]
    beta = float(p.reaction[1]) if p.reaction[0] == "linear" else 0.0
    scal = [host_scalars(p.alpha, beta, float(p.gamma[b]), float(p.dt[b]), p.dx) for b in range(B)]
    u = np.array(p.u0, dtype=np.float64, copy=True)
    H = np.empty((n + 1, B) + shape, dtype=np.float64)
    for b in range(B):
        H[0, b] = stencil(u[b])
    snaps = [(0, u.copy())]
    cadence = p.cadence
    t0 = time.perf_counter()
    for k in range(n):
        nxt = np.empty_like(u)
        for b in range(B):
            offs, wts = schedule(kind, k, param, float(p.dt[b]))
            acc = history_sum(H[: k + 1, b], offs, wts, tables[b], k)
            decay, diffuse = scal[b]
            nb = _update(u[b], acc, p.reaction, float(p.dt[b]), decay, diffuse)
            zero_ring(nb)
            nxt[b] = nb
        if not np.isfinite(nxt).all():
            fin = nxt[np.isfinite(nxt)]
            peak = float(np.abs(fin).max()) if fin.size else math.inf
            raise OracleDivergence(k + 1, peak)
        for b in range(B):
            H[k + 1, b] = stencil(nxt[b])
        u = nxt
        done = k + 1
        if (done % cadence == 0 or done == n) and snaps[-1][0] != done:
            snaps.append((done, u.copy()))
    elapsed = time.perf_counter() - t0
    return {"snapshots": snaps, "final": snaps[-1][1], "elapsed_seconds": elapsed}
