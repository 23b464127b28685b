"""Device engine: owns every HBM buffer of one run and drives the fused step kernel.

This is the B200 replacement for the body of ``solver.run``
(/root/reference/pkg/src/fracgrid/solver.py:230-265).  It is shared by the
reference-compatible 2D API (:mod:`.solver`) and the n-D / batched extension
(:mod:`.problem`).  PyTorch is used only as the device allocator and stream
provider; all arithmetic on the path runs in the kernels of ``libfgb200.so``.

HBM layout:
    H      [n_steps+1][B][ms]  fp64   δ^t = stencil(u^t), one slice per step
    u      [2][B][ms]          fp64   ping-pong fields, u^k in slot k & 1
    psi    [B][n_steps+1]      fp64   ψ_b(m), generated on the device
    snaps  [n_snap][B][ms]     fp64   snapshot pool written by the step kernel
``ms`` = points per member rounded up to 32 (256-byte aligned member rows).
"""

from __future__ import annotations

import ctypes as C
import logging
import math
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _lib

log = logging.getLogger("fracgrid")

DEFAULT_HISTORY_BYTE_CAP = 4 * 1024**3  # grid.py:13
_INT64_BIG = 1 << 62


class MemoryBudgetError(ValueError):
    """History storage for the requested run would exceed the byte cap (grid.py:16-17)."""


class HistoryCapacityError(ValueError):
    """An append would exceed the buffer's preallocated step count (grid.py:20-21)."""


class DivergenceError(RuntimeError):
    """A step produced non-finite concentrations (solver.py:38-46)."""

    def __init__(self, step: int, peak: float):
        # not super(): a bridged subclass (below) puts the reference's class,
        # whose __init__ takes (step, peak), next in the MRO
        RuntimeError.__init__(self, f"solution diverged at step {step}: max |u| reached {peak!r}")
        self.step = step
        self.peak = peak


# The reference's callers catch the reference's own exception classes
# (benchmark.py:114-128 records a diverging cell as a NaN row, cli.py:469-479
# maps it to exit code 3).  When ``fracgrid`` is loaded in this process, every
# error this package raises is an instance of BOTH its own class and the
# reference's class of the same name, so those handlers keep working when
# ``run`` is rebound to this package's (integrate.install).  Nothing is
# imported: the reference module is looked up in sys.modules only.
_REFERENCE_HOME = {
    DivergenceError: ("fracgrid.solver", "DivergenceError"),
    MemoryBudgetError: ("fracgrid.grid", "MemoryBudgetError"),
    HistoryCapacityError: ("fracgrid.grid", "HistoryCapacityError"),
}
_BRIDGED: dict = {}


def error_class(ours: type) -> type:
    """``ours``, or a cached subclass of ``ours`` and the reference's same-named
    class when that reference module is loaded (see _REFERENCE_HOME)."""
    import sys

    module, name = _REFERENCE_HOME[ours]
    mod = sys.modules.get(module)
    ref = getattr(mod, name, None) if mod is not None else None
    if not isinstance(ref, type) or not issubclass(ref, BaseException) or issubclass(ours, ref):
        return ours
    cls = _BRIDGED.get((ours, ref))
    if cls is None:
        cls = type(ours.__name__, (ours, ref), {"__module__": ours.__module__, "__doc__": ours.__doc__,
                                                "__qualname__": ours.__qualname__})
        _BRIDGED[(ours, ref)] = cls
    return cls


def divergence(step: int, peak: float) -> DivergenceError:
    return error_class(DivergenceError)(step, peak)


def budget_error(msg: str) -> MemoryBudgetError:
    return error_class(MemoryBudgetError)(msg)


def default_flags() -> int:
    env = os.environ.get("FGB200_RUN_FLAGS")
    if env is not None:
        return int(env)
    # per-step launches chained with programmatic dependent launch measured
    # fastest on B200 (profiles/): the next step's A phase fills this step's tail
    return _lib.FG_RUN_PDL


def env_flags() -> int:
    """Launch-shape options from the environment, read per call (tests toggle them);
    results are bitwise identical either way: FGB200_BLOCK_OVERLAP=0 (no side
    stream for the main block-stage launches), FGB200_PAIRS=0/1 (fused step
    pairs off / also in 2D)."""
    f = 0
    if os.environ.get("FGB200_BLOCK_OVERLAP") == "0":
        f |= _lib.FG_RUN_NO_OVERLAP
    pairs = os.environ.get("FGB200_PAIRS")
    if pairs == "0":
        f |= _lib.FG_RUN_NO_PAIRS
    elif pairs == "1":
        f |= _lib.FG_RUN_PAIRS
    return f


def default_tblock(p: "Problem | None" = None) -> int:
    """Temporal blocking factor (0 = off): one history pass feeds this many steps.

    Measured on B200 (profiles/r01_summary.md, tblock sweep): single-member
    full memory at 32 (the dense block kernel turns fp64-tensor bound);
    adaptive at 128 with 16-column items for large fields (c3, c4, c5) and at
    56 with 8-column items otherwise (c2); short memory on large single fields
    at 32 too (the solo dense main launch), other short memory and ensembles
    (per-member tables built in the CTA) at 24.
    """
    env = os.environ.get("FGB200_TBLOCK")
    if env is not None:
        return int(env)
    if p is None:
        return 24
    thinned = p.kind == "adaptive" and int(p.param) < int(p.n_steps)  # base >= n: the full schedule
    if thinned and large_field(p):
        # 16-column items (see item_cols): one history pass per 112 (single
        # field: the stride-7 interval then has exactly 16 steps per residue
        # class; c3-adaptive 302 vs 314 ms at 128, c4-adaptive 621 vs 644) or
        # 128 steps (ensembles: c5 1312 vs 1346 ms at 112)
        return 128 if p.batch > 1 else 112
    if p.batch > 1:
        # ensembles: itemized (per-member coefficient rows) when thinned; dense otherwise
        return 64 if thinned else 24
    # a short memory at least as long as the run is the full schedule, and must
    # give the full schedule's bits (reference property, test_covering_strategies)
    truncating = p.kind == "short" and short_horizon(p.param, float(p.dt[0])) < int(p.n_steps)
    if truncating:
        # large single fields: 32, the solo dense main launch (c3-short 240 -> 231 ms,
        # 220 ms with sub-blocks of 8, default_subblock); 24 measured best otherwise
        return 32 if large_field(p) else 24
    # thinned schedules: the itemized block stage does work proportional to the
    # schedule's terms, so a wider block (fewer history passes) pays off up to
    # 56 (c2, one box: 35.8 ms at 40, 33.5 at 48, 32.7 at 56, 33.3 at 64 and 72 —
    # at 56 the stride-7 interval has exactly 8 steps per residue class, so its
    # 8-column items read it once; wider blocks lengthen the step chain's recent sums)
    return 56 if thinned else 32


def item_cols(p: "Problem") -> int:
    """Step columns per item of the itemized block stage (fg_plan.item_cols).

    16-column items stream a residue class of up to 16 steps once (narrow
    tiles); 8-column items use wider tiles.  Measured on B200 (ms per run):
    c2 8/64 30.2, 16/128 37.8; c3-adaptive 8/64 352, 16/128 336; c4-adaptive
    8/64 716, 16/128 687; c5 8/64 1780, 16/128 1400.  FGB200_ITEM_COLS overrides.
    """
    env = os.environ.get("FGB200_ITEM_COLS")
    if env in ("8", "16"):
        return int(env)
    return 16 if large_field(p) else 8


def large_field(p: "Problem") -> bool:
    """Fields of >= 2^19 points in all (c3, c4, c5): their step chain keeps up
    with a block stage at tblock 128 and 16-column items; smaller ones (c2)
    are step-chain bound and run best at tblock 64 with 8-column items."""
    return p.batch * p.n_m >= 1 << 19


def default_subblock(p: "Problem", tblock: int) -> int:
    """Sub-block length S of the sub-block launches (fg_plan.subblock, 0 = off).

    Large fields (c3, c4, c5) at tblock 112/128: the block's own slices do not
    fit in L2, so every step re-reads its recent slices from HBM; with
    sub-blocks each finished one is streamed once into the later steps' partial
    sums.  Measured on B200 at tblock 128 (ms per run, S = 0 / 8 / 16 / 32 /
    64): c5 1403 / 1492 / 1372 / 1350 / 1374, c3-adaptive 335 / 423 / 339 / 323
    / 326 (tblock 112: S = 28 302, S = 56 312) — the steps' recent sums are
    bound by their rounds of loads in flight more than by their count, so a
    quarter block pays and shorter ones do not.  FGB200_SUBBLOCK overrides (0
    disables).
    """
    env = os.environ.get("FGB200_SUBBLOCK")
    if env is not None:
        s = int(env)
    elif p.kind != "adaptive":
        # dense schedules (one field): every step sums all its recent offsets,
        # so even short sub-blocks pay (c3-short 278 -> 262 ms at S = 4,
        # c3-full 693 -> 675 and c4-full 1414 -> 1370 at S = 8)
        # (c3-short at tblock 32, S/D: 4/4 231-235, 8/8 231, 8/4 220, 8/2 225 ms)
        s = (8 if p.kind == "full" or tblock == 32 else 4) if large_field(p) and p.batch == 1 else 0
    else:
        s = tblock // 4 if large_field(p) and tblock >= 112 else 0
    if s and (tblock % s or tblock // s > 16 or s < 2):
        return 0
    return s


def default_subdelay(p: "Problem", subblock: int) -> int:
    """Steps a sub-block launch has to finish (fg_plan.subdelay, 0 = one whole
    sub-block): sub-block i feeds the steps from (i+1)·S + D on, so the steps
    themselves sum offsets < S + D.  FGB200_SUBDELAY overrides."""
    env = os.environ.get("FGB200_SUBDELAY")
    if env is not None:
        d = int(env)
    elif p.kind in ("adaptive", "full"):
        # a quarter sub-block: measured on B200 (ms per run, D = S / 14 / 7 / 4 at
        # S = 28): c4-adaptive 579 / 571 / 562 / 570, c3-adaptive 262 / 258 / 257 /
        # 258, c5 (S = 32) 1128 / 1096 / 1088 / 1083; c4-full (S = 8, D = 8 / 4 / 2)
        # 1342 / 1317 / 1312 — the launch still finishes in time and the steps sum
        # fewer recent slices.  Short memory (S = 4) keeps D = S (c3-short 247 vs
        # 267 at D = 2).
        d = subblock // 4
    elif subblock == 8:
        d = 4  # short memory at tblock 32 (see default_subblock)
    else:
        d = 0
    return d if 0 <= d <= subblock else 0


def history_pad(p: "Problem", tblock: int) -> int:
    """Slices allocated past H[n] for a blocked run (fg_history_pad): the 16-column
    item stage reads whole TMA boxes of 16 slices of a strided progression (the
    itemized stages of adaptive runs, and the sub-block launches of dense ones)."""
    n = int(p.n_steps)
    if not tblock or n <= tblock or item_cols(p) != 16:
        return 0
    pad = C.c_int64(0)
    base = int(p.param) if p.kind == "adaptive" else 0
    _lib.check(_lib.load().fg_history_pad(_lib.MEM_KINDS[p.kind], n, base, C.byref(pad)), "fg_history_pad")
    return int(pad.value)


def single_coef_rows(tblock: int, n_steps: int) -> int:
    """Coefficient rows per block of a single-member blocked run (fg_plan.coef_rows):
    rows for the tail, every slice of the main launch and the slices two
    strides' items share; itemized blocks re-read a dense class per 8-step item."""
    if tblock > 32:
        return (tblock // 8 + 2) * (n_steps + 1)
    return 2 * (n_steps + 1) + 4 * tblock


def round_up(n: int, m: int) -> int:
    return (n + m - 1) // m * m


def strategy_spec(strategy) -> tuple[str, float]:
    """Duck-type a memory strategy by ``.tag`` (schedule.py:198-257)."""
    tag = getattr(strategy, "tag", None)
    if tag == "full":
        return "full", 0
    if tag == "short":
        length = float(strategy.length)
        if not length > 0 or not math.isfinite(length):
            raise ValueError(f"short-memory length must be positive and finite, got {length!r}")
        return "short", length
    if tag == "adaptive":
        base = strategy.base
        if isinstance(base, bool) or int(base) != base or int(base) < 2:
            raise ValueError(f"adaptive base must be an integer >= 2, got {base!r}")
        return "adaptive", int(base)
    raise TypeError(f"not a memory strategy: {strategy!r}")


def short_horizon(length: float, dt: float) -> int:
    """floor(L/dt) exactly as schedule.py:92 evaluates it (then clamped for int64)."""
    if not dt > 0 or not math.isfinite(dt):
        raise ValueError(f"dt must be positive and finite, got {dt!r}")
    return min(int(math.floor(float(length) / float(dt))), _INT64_BIG)


def host_scalars(alpha: float, beta: float, gamma: float, dt: float, dx: float) -> tuple[float, float]:
    """(decay, diffuse) with the reference's Python-float evaluation (solver.py:215-216)."""
    decay = 1.0 - float(beta) * float(dt)
    diffuse = float(alpha) * float(dt) ** float(gamma) / float(dx) ** 2
    return decay, diffuse


def snapshot_steps(n_steps: int, cadence: int) -> list[int]:
    """0, every ``cadence`` steps, and the final step (solver.py:245-256)."""
    steps = [0]
    for done in range(cadence, n_steps + 1, cadence):
        steps.append(done)
    if steps[-1] != n_steps:
        steps.append(n_steps)
    return steps


@dataclass
class Problem:
    """Normalised run: ``B`` members sharing one field shape (1-3 dims)."""

    u0: np.ndarray            # (B, *shape) float64, boundary ring zero
    gamma: np.ndarray         # (B,)
    dt: np.ndarray            # (B,)
    alpha: float
    dx: float
    reaction: tuple           # ("linear", beta) | ("saturating", vmax, km)
    kind: str                 # full | short | adaptive
    param: float
    n_steps: int
    cadence: int
    history_byte_cap: int | None = DEFAULT_HISTORY_BYTE_CAP

    @property
    def batch(self) -> int:
        return int(self.u0.shape[0])

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(int(s) for s in self.u0.shape[1:])

    @property
    def n_m(self) -> int:
        return int(np.prod(self.shape))

    def terms(self) -> int:
        """Σ_k len_k · N over the run — the metric's numerator."""
        L = _lib.load()
        out = C.c_int64(0)
        total = 0
        for b in range(self.batch if self.kind == "short" else 1):
            hz = short_horizon(self.param, float(self.dt[b])) if self.kind == "short" else 0
            base = int(self.param) if self.kind == "adaptive" else 0
            s = 0
            for k in range(self.n_steps):
                _lib.check(L.fg_schedule_len(_lib.MEM_KINDS[self.kind], k, base, hz, C.byref(out)))
                s += out.value
            total += s * self.n_m
        if self.kind != "short":
            total *= self.batch
        return total


def recent_entries(kind: str, k: int, param: float, horizon: int, mmax: int) -> int:
    """Entries of schedule(k) with 1 <= m <= mmax (host accounting, schedule.py:70-151)."""
    if kind in ("full", "short"):
        top = k if kind == "full" else min(horizon, k)
        return max(0, min(mmax, top))
    a = int(param)
    if k <= a:
        return max(0, min(mmax, k))
    n = min(mmax, a)  # dense window 1..a
    i, a_prev, last = 2, a, None
    while True:
        start = a_prev + i
        if start > k:
            break
        a_i, stride = a_prev * a, 2 * i - 1
        hi = min(a_i, k - i + 1)
        if hi >= start:
            cnt = (hi - start) // stride + 1
            if start <= mmax:
                n += min(cnt, (mmax - start) // stride + 1)
            last = (start + (cnt - 1) * stride, i, a_i)
        a_prev, i = a_i, i + 1
    tail = a + 1 if last is None else (last[2] + 1 if k > last[2] else last[0] + last[1])
    if tail <= min(k, mmax):
        n += min(k, mmax) - tail + 1
    return n


def block_launch_bytes(p: Problem, tblock: int, with_flops: bool = False) -> list[tuple]:
    """(kb0, bt, algorithmic bytes[, algorithmic flops]) of every block stage of one run.

    A block stage (main + tail launch) reads the union of its steps' old slices
    (t < kb0) once and writes bt partial-sum slices; its flops are 2 per point
    per old schedule entry (m > b for step kb0+b).  The first block (kb0 = 0)
    has no old slices and is a memset, not a launch.
    """
    L = _lib.load()
    out = C.c_int64(0)
    base = int(p.param) if p.kind == "adaptive" else 0
    kind = _lib.MEM_KINDS[p.kind]
    members = range(p.batch) if p.kind == "short" else [0]
    scale = p.n_m * (1 if p.kind == "short" else p.batch)
    n = int(p.n_steps)
    hzs = {b: (short_horizon(p.param, float(p.dt[b])) if p.kind == "short" else 0) for b in members}
    res = []
    for kb0 in range(tblock, n, tblock):
        bt = min(tblock, n - kb0)
        slices = 0
        terms = 0
        for b in members:
            hz = hzs[b]
            _lib.check(L.fg_block_union(kind, kb0, bt, base, hz, C.byref(out)))
            slices += out.value + bt
            if with_flops:
                for bb in range(bt):
                    k = kb0 + bb
                    _lib.check(L.fg_schedule_len(kind, k, base, hz, C.byref(out)))
                    terms += out.value - 1 - recent_entries(p.kind, k, p.param, hz, bb)
        rec = (kb0, bt, slices * scale * 8)
        res.append(rec + (2 * terms * scale,) if with_flops else rec)
    return res


def execution_bytes(p: Problem, tblock: int) -> tuple[int, int]:
    """(single-pass algorithmic bytes, bytes of the algorithm as executed) for one run.

    Single pass: 8·N per history term + 3·8·N per step (u^k read,
    u^{k+1} write, δ^k write).  With temporal blocking of factor tb the history
    is read once per block over the union of the block's old slices, plus the
    partial sums P (written once, read once per step) and each step's recent
    entries (1 <= m <= b).
    """
    N = p.batch * p.n_m
    n = int(p.n_steps)
    single = 8 * p.terms() + 3 * 8 * N * n
    if not tblock:
        return single, single
    L = _lib.load()
    out = C.c_int64(0)
    base = int(p.param) if p.kind == "adaptive" else 0
    members = range(p.batch) if p.kind == "short" else [0]
    total = 0
    for b in members:
        hz = short_horizon(p.param, float(p.dt[b])) if p.kind == "short" else 0
        for kb0 in range(0, n, tblock):
            bt = min(tblock, n - kb0)
            _lib.check(L.fg_block_union(_lib.MEM_KINDS[p.kind], kb0, bt, base, hz, C.byref(out)))
            total += out.value + bt  # union slices + P write
            for bb in range(bt):
                total += 1 + recent_entries(p.kind, kb0 + bb, p.param, hz, bb)  # P read + recent slices
    scale = p.n_m * 8 * (1 if p.kind == "short" else p.batch)
    return single, total * scale + 3 * 8 * N * n


def check_history_budget(p: Problem) -> None:
    """MemoryBudgetError before any allocation (grid.py:141-146, same formula)."""
    n, B, shape = int(p.n_steps), p.batch, p.shape
    needed = (n + 1) * B * p.n_m * 8
    if p.history_byte_cap is not None and needed > p.history_byte_cap:
        members = f" x{B} members" if B > 1 else ""
        raise budget_error(
            f"history of {n + 1} fields of shape {'x'.join(map(str, shape))}{members} needs "
            f"{needed} bytes, over the cap of {p.history_byte_cap}")


_TOTALS: dict = {}


def _device_total(device) -> int:
    """Total device memory (cached; the properties call is cheap only once)."""
    import torch

    key = str(device)
    if key not in _TOTALS:
        _TOTALS[key] = int(torch.cuda.get_device_properties(device).total_memory)
    return _TOTALS[key]


class Stepper:
    """All device state of one run plus the loop driver."""

    def __init__(self, problem: Problem, *, device=None, split: int = 0, flags: int | None = None,
                 snapshots: bool = True, tblock: int | None = None):
        import torch

        self.torch = torch
        self.p = problem
        p = problem
        B, shape, n = p.batch, p.shape, int(p.n_steps)
        if not 1 <= len(shape) <= 3:
            raise ValueError(f"fields must have 1-3 dimensions, got shape {shape}")
        if any(s < 3 for s in shape):
            raise ValueError(f"grid must be at least 3 points per axis, got {shape}")
        self.n_m = p.n_m
        self.ms = round_up(self.n_m, 32)
        check_history_budget(p)
        self.device = device if device is not None else _lib.require_cuda()
        self.flags = default_flags() if flags is None else int(flags)
        L = self.L = _lib.load()
        slice_elems = B * self.ms
        self.snap_steps = snapshot_steps(n, p.cadence) if snapshots else []
        pool_slices = max(0, len([s for s in self.snap_steps if s > 0]))
        tb = default_tblock(p) if tblock is None else int(tblock)
        p_slices = 2 * tb if tb and n > tb else 0
        ens_rows = 0
        if tb and n > tb and B > 1 and p.kind == "adaptive":
            # itemized ensembles: per-member item coefficient rows
            # ([2][B][rows][36]; the shared schedule fixes the items, ψ_b the values)
            need = C.c_int64(0)
            icols = item_cols(p)
            _lib.check(L.fg_block_item_rows(_lib.MEM_KINDS["adaptive"], n, tb, int(p.param), 0, icols,
                                            C.byref(need)), "fg_block_item_rows")
            ens_rows = max(1, -(-need.value * _lib.FG_ITEM_PITCH[icols] // _lib.FG_COEF_ROW))
        self.h_pad = history_pad(p, tb)
        dev_bytes = ((n + 1) + self.h_pad + 2 + pool_slices + p_slices) * slice_elems * 8 + B * (n + 1) * 8
        dev_bytes += 2 * B * ens_rows * _lib.FG_COEF_ROW * 8
        if tb and n > tb and B == 1:
            dev_bytes += 2 * single_coef_rows(tb, n) * _lib.FG_COEF_ROW * 8
        self.pairs_possible = bool(tb and n > tb and len(shape) <= 2 and p.kind != "short")
        if self.pairs_possible:
            dev_bytes += (slice_elems + 1) * 8
        # cudaMemGetInfo costs ~1 ms per call: ask it only when the request is
        # not obviously small next to what torch already holds or the device has
        idle = torch.cuda.memory_reserved(self.device) - torch.cuda.memory_allocated(self.device)
        if dev_bytes > idle and dev_bytes > _device_total(self.device) // 4:
            free, _total = torch.cuda.mem_get_info(self.device)
            free += idle
            if dev_bytes > free:
                raise budget_error(
                    f"device history and fields need {dev_bytes} bytes, only {free} free on {self.device}")
        f64 = dict(dtype=torch.float64, device=self.device)
        try:
            self._allocate(p, shape, split, slice_elems, pool_slices, ens_rows, tb, f64)
        except torch.cuda.OutOfMemoryError as exc:
            # a device that is mostly taken by another process: same error type
            # as the byte-cap refusal (grid.py:141-146), before any step runs
            raise budget_error(f"device history and fields need {dev_bytes} bytes, more than is free on "
                               f"{self.device} ({exc.__class__.__name__})") from None

    def _allocate(self, p, shape, split, slice_elems, pool_slices, ens_rows, tb, f64) -> None:
        """Every device buffer of the run (allocated once, before the loop) and the plan."""
        import torch

        L = self.L
        B, n = p.batch, int(p.n_steps)
        self.H = torch.empty((n + 1 + self.h_pad, slice_elems), **f64)
        self.u = torch.zeros((2, slice_elems), **f64)
        self.psi = torch.empty((B, n + 1), **f64)
        self.status = torch.full((2,), _lib.FG_NO_BAD_STEP, dtype=torch.int64, device=self.device)
        beta = float(p.reaction[1]) if p.reaction[0] == "linear" else 0.0
        scal = [host_scalars(p.alpha, beta, float(p.gamma[b]), float(p.dt[b]), p.dx) for b in range(B)]
        self.decay = torch.tensor([s[0] for s in scal], **f64)
        self.diffuse = torch.tensor([s[1] for s in scal], **f64)
        self.dt = torch.tensor([float(x) for x in p.dt], **f64)
        gam = torch.tensor([float(x) for x in p.gamma], **f64)
        hz = [short_horizon(p.param, float(p.dt[b])) if p.kind == "short" else 0 for b in range(B)]
        self.horizon = torch.tensor(hz, dtype=torch.int64, device=self.device)
        self.pool = torch.empty((pool_slices, slice_elems), **f64) if pool_slices else None
        self.snap_slot = torch.empty((n + 2,), dtype=torch.int32, device=self.device) if pool_slices else None
        st = _lib.stream_handle()
        _lib.check(L.fg_psi_tables(gam.data_ptr(), B, n, n + 1, self.psi.data_ptr(), st), "fg_psi_tables")
        # upload u^0 (padded rows) — the run's host→device input copy
        u0 = np.zeros((B, self.ms), dtype=np.float64)
        u0[:, : self.n_m] = np.asarray(p.u0, dtype=np.float64).reshape(B, self.n_m)
        self.h2d_bytes = u0.nbytes
        self.u[0].copy_(torch.from_numpy(u0).reshape(-1).pin_memory(), non_blocking=True)
        self.d2h_bytes = 0

        plan = _lib.FgPlan()
        plan.B, plan.n_m, plan.ms = B, self.n_m, self.ms
        plan.ndim = len(shape)
        plan.reaction = _lib.REACTIONS[p.reaction[0]]
        for i in range(3):
            plan.shape[i] = shape[i] if i < len(shape) else 1
        plan.kind = _lib.MEM_KINDS[p.kind]
        plan.split = int(split)
        plan.base = int(p.param) if p.kind == "adaptive" else 0
        plan.horizon_dev = self.horizon.data_ptr()
        plan.psi_dev = self.psi.data_ptr()
        plan.psi_stride = n + 1
        plan.decay_dev = self.decay.data_ptr()
        plan.diffuse_dev = self.diffuse.data_ptr()
        plan.dt_dev = self.dt.data_ptr()
        if p.reaction[0] == "saturating":
            plan.vmax, plan.km = float(p.reaction[1]), float(p.reaction[2])
        plan.H_dev = self.H.data_ptr()
        plan.h_slices = n + 1
        plan.h_alloc = n + 1 + self.h_pad
        plan.u_dev[0] = self.u[0].data_ptr()
        plan.u_dev[1] = self.u[1].data_ptr()
        plan.status_dev = self.status.data_ptr()
        plan.snap_slot_dev = self.snap_slot.data_ptr() if self.snap_slot is not None else None
        plan.horizon_max = max(hz) if p.kind == "short" else 0
        plan.item_cols = item_cols(p)
        self.P = None
        if self.pairs_possible:  # fused step pairs: u^{k+2} buffer + the step it holds
            self.pair = torch.empty(slice_elems + 1, **f64)
            plan.pair_dev = self.pair.data_ptr()
        if tb and n > tb:
            # two buffers: block j's steps read one while block j+1's main launch
            # fills the other (fg_run's side-stream pipeline)
            self.P = torch.empty((2, tb, slice_elems), **f64)
            plan.tblock = tb
            plan.P_dev = self.P.data_ptr()
            if ens_rows:
                self.blkcoef = torch.empty((2, B, ens_rows, _lib.FG_COEF_ROW), **f64)
                plan.blkcoef_dev = self.blkcoef.data_ptr()
                plan.coef_rows = ens_rows
            if B == 1:  # per-block coefficient rows shared by all tiles
                # two blocks in flight; rows for the tail, every slice of the main
                # launch and the slices two strides' items share
                rows = single_coef_rows(tb, n)
                self.blkcoef = torch.empty((2, rows, _lib.FG_COEF_ROW), **f64)
                plan.blkcoef_dev = self.blkcoef.data_ptr()
                plan.coef_rows = rows
                # host copy of ψ(0..tb): the library hands the blocked steps their
                # coefficients as launch parameters (no ψ loads in the step chain)
                self.psi_host = np.ascontiguousarray(self.psi[0, : tb + 1].cpu().numpy())
                plan.psi_host = self.psi_host.ctypes.data

        if plan.tblock and plan.blkcoef_dev and (p.kind == "adaptive" or B == 1):
            plan.subblock = default_subblock(p, int(plan.tblock))
            plan.subdelay = default_subdelay(p, int(plan.subblock))
        self.tblock = int(plan.tblock)
        self.plan = plan
        self.k = 0
        self.pool_host = None
        self.copy_stream = None
        self.copied: set[int] = set()
        self._p_block: int | None = None  # block whose partial sums P holds

    # ---------------------------------------------------------------- driving --
    def block_partials(self, kb0: int):
        """View of the partial-sum buffer that holds the block starting at kb0."""
        return self.P[(kb0 // self.tblock) & 1]

    def reset(self, u0_dev) -> None:
        """Rewind to step 0 from a device-resident padded u^0 (benchmark re-runs)."""
        self.u[0].copy_(u0_dev)
        self.status.fill_(_lib.FG_NO_BAD_STEP)
        self.k = 0
        self.copied = set()
        self._p_block = None

    def geometry(self) -> tuple[int, int, int]:
        ctas, thr, spl = C.c_int64(0), C.c_int32(0), C.c_int32(0)
        _lib.check(self.L.fg_step_geometry(C.byref(self.plan), C.byref(ctas), C.byref(thr), C.byref(spl)))
        return ctas.value, thr.value, spl.value

    def advance(self, k1: int, *, flags: int | None = None, stream_snapshots: bool = False) -> None:
        """Launch steps self.k .. k1-1 (asynchronous, stream-ordered).

        With ``stream_snapshots`` every snapshot is copied to pinned host memory
        by the library (fg_run_ex) on its copy stream as soon as the step that
        produced it is done, overlapping the following steps; the copies are
        joined into the current stream.
        """
        k0 = self.k
        if k1 <= k0:
            return
        snaps = [s for s in self.snap_steps if s > 0]
        arr = (C.c_int64 * max(1, len(snaps)))(*snaps)
        pool = self.pool.data_ptr() if self.pool is not None else None
        host = None
        if stream_snapshots and self.pool is not None:
            if self.pool_host is None:
                self.pool_host = self.torch.empty(self.pool.shape, dtype=self.torch.float64, pin_memory=True)
            host = self.pool_host.data_ptr()
            self.copied.update(i for i, s in enumerate(snaps) if k0 < s <= k1)
        fl = (self.flags if flags is None else flags) | env_flags()
        _lib.check(self.L.fg_run_ex(C.byref(self.plan), k0, k1, arr, len(snaps), pool, host,
                                    fl | self._continue_flag(k0), _lib.stream_handle()), "fg_run_ex")
        if self.tblock:
            self._p_block = (k1 - 1) - (k1 - 1) % self.tblock
        self.k = k1

    def _continue_flag(self, start: int) -> int:
        """FG_RUN_CONTINUE when P already holds the partial sums of start's block."""
        if self.tblock and self._p_block is not None and start - start % self.tblock == self._p_block:
            return _lib.FG_RUN_CONTINUE
        return 0

    def run(self, progress_every: int = 0) -> float:
        """Run every step; return the loop's wall time (solver.py:248-257 semantics)."""
        torch = self.torch
        n = int(self.p.n_steps)
        torch.cuda.synchronize(self.device)
        t0 = time.perf_counter()
        if progress_every and progress_every > 0:
            for stop in list(range(progress_every, n + 1, progress_every)) + [n]:
                if stop <= self.k:
                    continue
                self.advance(stop, stream_snapshots=True)
                torch.cuda.synchronize(self.device)
                if stop % progress_every == 0:
                    self.raise_if_diverged()
                    log.info("step %d/%d", stop, n)
        else:
            self.advance(n, stream_snapshots=True)
        torch.cuda.synchronize(self.device)
        elapsed = time.perf_counter() - t0
        self.raise_if_diverged()
        return elapsed

    def first_bad_step(self) -> int | None:
        v = int(self.status[0].item())
        return None if v == _lib.FG_NO_BAD_STEP else v

    def raise_if_diverged(self) -> None:
        bad = self.first_bad_step()
        if bad is None:
            return
        field = self.u[bad & 1].reshape(self.p.batch, self.ms)[:, : self.n_m]
        fin = field[self.torch.isfinite(field)]
        peak = float(fin.abs().max().item()) if fin.numel() else math.inf
        raise divergence(bad, peak)

    # -------------------------------------------------------------- results --
    def fetch_snapshots(self) -> list[tuple[int, np.ndarray]]:
        """Snapshots as host arrays; step 0 is the input field itself.

        Snapshots already streamed to pinned memory during the run are returned
        as zero-copy views of that buffer; any others come over in one D2H copy.
        """
        torch = self.torch
        B, shape = self.p.batch, self.p.shape
        out = [(0, np.array(self.p.u0, dtype=np.float64).reshape((B,) + shape))]
        later = [s for s in self.snap_steps if s > 0]
        self.d2h_bytes = 0
        if later:
            torch.cuda.current_stream(self.device).synchronize()  # joins the library's snapshot copies
            missing = [i for i in range(len(later)) if i not in self.copied]
            if self.pool_host is None:
                self.pool_host = torch.empty(self.pool.shape, dtype=torch.float64, pin_memory=True)
            if missing:
                torch.cuda.synchronize(self.device)
                if len(missing) == len(later):
                    self.pool_host.copy_(self.pool)
                else:
                    for i in missing:
                        self.pool_host[i].copy_(self.pool[i])
            self.d2h_bytes = self.pool_host.numel() * 8
            arr = self.pool_host.numpy().reshape(len(later), B, self.ms)[:, :, : self.n_m]
            for i, s in enumerate(later):
                out.append((s, arr[i].reshape((B,) + shape)))
        return out

    def field(self, k: int | None = None) -> np.ndarray:
        k = self.k if k is None else k
        arr = self.u[k & 1].reshape(self.p.batch, self.ms)[:, : self.n_m].cpu().numpy()
        return arr.reshape((self.p.batch,) + self.p.shape)
