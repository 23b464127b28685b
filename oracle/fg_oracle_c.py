"""ctypes front end of ``oracle/fg_oracle.c`` — TEST INFRASTRUCTURE ONLY.

Same inputs and outputs as :func:`oracle.fg_oracle.run`, bitwise-identical
results, multi-threaded over grid points.  Used by the tests as a fast checker and
by ``bench.py`` as the timed CPU baseline (``kind: "port"``).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

from .fg_oracle import OracleDivergence, OracleProblem, host_scalars

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libfgoracle.so")

_KINDS = {"full": 0, "short": 1, "adaptive": 2}


class _Problem(C.Structure):
    _fields_ = [
        ("B", C.c_int64), ("n_m", C.c_int64), ("ndim", C.c_int32), ("reaction", C.c_int32),
        ("shape", C.c_int64 * 3),
        ("gamma", C.POINTER(C.c_double)), ("dt", C.POINTER(C.c_double)),
        ("decay", C.POINTER(C.c_double)), ("diffuse", C.POINTER(C.c_double)),
        ("vmax", C.c_double), ("km", C.c_double),
        ("kind", C.c_int32), ("pad_", C.c_int32), ("param", C.c_double), ("n_steps", C.c_int64),
    ]


_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.fgo_run.restype = C.c_int
        L.fgo_run.argtypes = [C.POINTER(_Problem), C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                              C.POINTER(C.c_int64), C.c_int, C.c_int64, C.POINTER(C.c_double)]
        L.fgo_build_table.restype = C.c_int
        L.fgo_build_table.argtypes = [C.c_double, C.c_int64, C.c_void_p]
        L.fgo_schedule.restype = C.c_int64
        L.fgo_schedule.argtypes = [C.c_int32, C.c_int64, C.c_double, C.c_double, C.c_void_p,
                                   C.c_void_p, C.c_int64]
        L.fgo_max_threads.restype = C.c_int
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().fgo_max_threads())


def snapshot_steps(n_steps: int, cadence: int) -> list[int]:
    """Snapshot steps of solver.run (solver.py:245-256): 0, every cadence, final."""
    steps = [0]
    for done in range(1, n_steps + 1):
        if (done % cadence == 0 or done == n_steps) and steps[-1] != done:
            steps.append(done)
    return steps


def run(p: OracleProblem, *, nthreads: int = 0, max_steps: int = -1, snapshots: bool = True):
    """Run the C restatement.  ``max_steps`` truncates to a prefix (bounded
    samples for the CPU baseline); the prefix is exact."""
    u0 = np.ascontiguousarray(p.u0, dtype=np.float64)
    B = u0.shape[0]
    shape = u0.shape[1:]
    if not 1 <= len(shape) <= 3:
        raise ValueError("1-3 spatial dimensions")
    T = int(p.n_steps)
    steps_run = T if max_steps < 0 else min(T, int(max_steps))
    gamma = np.ascontiguousarray(np.broadcast_to(np.asarray(p.gamma, np.float64), (B,)))
    dt = np.ascontiguousarray(np.broadcast_to(np.asarray(p.dt, np.float64), (B,)))
    beta = float(p.reaction[1]) if p.reaction[0] == "linear" else 0.0
    sc = [host_scalars(p.alpha, beta, float(gamma[b]), float(dt[b]), p.dx) for b in range(B)]
    decay = np.array([s[0] for s in sc])
    diffuse = np.array([s[1] for s in sc])
    kind, param = p.strategy
    prob = _Problem()
    prob.B, prob.n_m, prob.ndim = B, int(np.prod(shape)), len(shape)
    prob.reaction = 0 if p.reaction[0] == "linear" else 1
    for i, s in enumerate(shape):
        prob.shape[i] = s
    dp = C.POINTER(C.c_double)
    prob.gamma, prob.dt = gamma.ctypes.data_as(dp), dt.ctypes.data_as(dp)
    prob.decay, prob.diffuse = decay.ctypes.data_as(dp), diffuse.ctypes.data_as(dp)
    if p.reaction[0] == "saturating":
        prob.vmax, prob.km = float(p.reaction[1]), float(p.reaction[2])
    prob.kind, prob.param, prob.n_steps = _KINDS[kind], float(param), T
    if snapshots:
        ss = [s for s in snapshot_steps(T, p.cadence) if s <= steps_run]
    else:
        ss = []
    ss_arr = np.asarray(ss, dtype=np.int64)
    snaps = np.empty((len(ss),) + u0.shape, dtype=np.float64)
    u = u0.copy()
    bad = C.c_int64(0)
    el = C.c_double(0.0)
    rc = lib().fgo_run(C.byref(prob), u.ctypes.data, len(ss), ss_arr.ctypes.data, snaps.ctypes.data,
                       C.byref(bad), int(nthreads), int(steps_run), C.byref(el))
    if rc == 1:
        fin = u[np.isfinite(u)]
        peak = float(np.abs(fin).max()) if fin.size else math.inf
        raise OracleDivergence(int(bad.value), peak)
    if rc != 0:
        raise RuntimeError(f"fgo_run failed with code {rc}")
    return {"snapshots": list(zip(ss, snaps)), "final": u, "elapsed_seconds": el.value,
            "steps_run": steps_run}
