"""Freeze reference outputs as golden fixtures (run in the BUILD container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the real reference package ``fracgrid`` from ``/root/reference/pkg/src``
(read-only; nothing is copied) and writes ``tests/golden/golden.npz`` plus
``tests/golden/golden.json``.  ``/root/reference`` does not exist on the GPU box,
so the tests read only these committed fixtures there.

What is pinned (reference file:line relative to pkg/src/fracgrid/):

* ψ tables — ``coefficients.build_table`` (coefficients.py:76-92): full values for
  short tables, SHA-256 of the raw fp64 bytes for 10 001-entry tables.
* schedules — ``schedule.adaptive_schedule`` / ``short_schedule`` / ``full_schedule``
  (schedule.py:70-151): explicit pairs at selected k, and per-base SHA-256 over
  every k in 0..10000 of (len, offsets, weights) as little-endian int64.
* ``solver.history_sum`` (solver.py:162-197) on seeded random histories.
* ``solver.run`` (solver.py:230-265) on small 2D configs: every snapshot.
* n-D / saturating / batched compositions built from the reference's own
  ``build_table``, strategies, ``HistoryBuffer`` and ``history_sum`` around a
  restated n-D stencil (grid.py:98-106 operation pattern) — SURVEY.md §8(c).
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
from dataclasses import replace

import numpy as np

REF = os.environ.get("FRACGRID_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

from fracgrid.coefficients import build_table  # noqa: E402
from fracgrid.grid import HistoryBuffer, stencil as ref_stencil  # noqa: E402
from fracgrid.schedule import (  # noqa: E402
    AdaptiveMemory,
    FullMemory,
    ShortMemory,
    adaptive_schedule,
    full_schedule,
    short_schedule,
)
from fracgrid.solver import DivergenceError, SimulationConfig, history_sum, run  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

SCHED_BASES = (2, 3, 4, 5, 8, 12, 20, 40, 100, 1500)
SCHED_KMAX = 10000
PSI_GAMMAS = (0.1, 0.3, 0.35, 0.5, 0.6, 0.7, 0.75, 0.8, 0.9, 1.0, 1.5, 1.99)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).astype("<i8" if a.dtype.kind in "iu" else "<f8").tobytes())
    return h.hexdigest()


def schedule_hash(make, kmax: int) -> str:
    h = hashlib.sha256()
    for k in range(kmax + 1):
        s = make(k)
        h.update(np.int64(len(s)).astype("<i8").tobytes())
        h.update(s.offsets.astype("<i8").tobytes())
        h.update(s.weights.astype("<i8").tobytes())
    return h.hexdigest()


# ---- n-D composition out of reference pieces ----------------------

def nd_stencil(u: np.ndarray) -> np.ndarray:
    if u.ndim == 2:
        return ref_stencil(u)
    out = np.zeros_like(u)
    if u.ndim == 1:
        out[1:-1] = u[2:] + u[:-2] - 2.0 * u[1:-1]
    else:
        c = (slice(1, -1),) * 3
        out[c] = (
            u[2:, 1:-1, 1:-1] + u[:-2, 1:-1, 1:-1] - 6.0 * u[c]
            + u[1:-1, 2:, 1:-1] + u[1:-1, :-2, 1:-1]
            + u[1:-1, 1:-1, 2:] + u[1:-1, 1:-1, :-2]
        )
    return out


def composed_run(u0, gamma, dt, alpha, dx, reaction, strategy, n_steps, snapshot_every):
    """One member: reference ψ / schedule / HistoryBuffer / history_sum, fields
    flattened to (1, N) exactly as SURVEY.md §8(c) prescribes."""
    shape = u0.shape
    N = int(np.prod(shape))
    table = build_table(gamma, n_steps)
    hist = HistoryBuffer(n_steps + 1, (1, N), byte_cap=None)
    u = u0.copy()
    hist.append(nd_stencil(u).reshape(1, N))
    snaps = [(0, u.copy())]
    cadence = snapshot_every or max(1, math.ceil(n_steps / 100))
    beta = reaction[1] if reaction[0] == "linear" else 0.0
    decay = 1.0 - beta * dt
    diffuse = alpha * dt**gamma / dx**2
    for k in range(n_steps):
        sched = strategy.schedule_at(k, dt)
        acc = history_sum(hist, sched, table, k).reshape(shape)
        if reaction[0] == "linear":
            nxt = u * decay + diffuse * acc
        else:
            vmax, km = reaction[1], reaction[2]
            f = -vmax * u / (km + u)
            nxt = u + dt * f + diffuse * acc
        for ax in range(nxt.ndim):
            idx = [slice(None)] * nxt.ndim
            idx[ax] = 0
            nxt[tuple(idx)] = 0.0
            idx[ax] = -1
            nxt[tuple(idx)] = 0.0
        if not np.isfinite(nxt).all():
            raise DivergenceError(k + 1, float("nan"))
        hist.append(nd_stencil(nxt).reshape(1, N))
        u = nxt
        done = k + 1
        if (done % cadence == 0 or done == n_steps) and snaps[-1][0] != done:
            snaps.append((done, u.copy()))
    return snaps


def dense_sources(u: np.ndarray):
    return tuple((int(j), int(l), float(u[j, l])) for j, l in zip(*np.nonzero(u)))


def main() -> None:
    arrays: dict[str, np.ndarray] = {}
    meta: dict = {"reference": REF, "numpy": np.__version__, "cases": {}}

    # ---- ψ --------------------------------------------------------------------
    meta["psi"] = {}
    for g in PSI_GAMMAS:
        arrays[f"psi_{g}_64"] = build_table(g, 64).values.copy()
        meta["psi"][str(g)] = sha(build_table(g, 10000).values)
    arrays["psi_0.5_1000"] = build_table(0.5, 1000).values.copy()

    # ---- schedules ------------------------------------------------------------
    meta["sched_hash"] = {str(a): schedule_hash(lambda k, a=a: adaptive_schedule(k, a), SCHED_KMAX)
                          for a in SCHED_BASES}
    meta["sched_hash"]["full"] = schedule_hash(full_schedule, 2000)
    shorts = [(100.0, 1.0), (10.5, 1.0), (100.0, 0.5), (4.0, 0.5), (0.3, 0.1), (7.25, 0.25)]
    meta["short_hash"] = {f"{L}/{dt}": schedule_hash(lambda k, L=L, dt=dt: short_schedule(k, L, dt), 3000)
                          for L, dt in shorts}
    meta["sched_pairs"] = {}
    for a, k in ((3, 9), (3, 20), (4, 260), (5, 5000), (5, 4999), (5, 3999), (5, 9999), (2, 777), (12, 2000)):
        meta["sched_pairs"][f"{a}/{k}"] = adaptive_schedule(k, a).pairs()

    # ---- history_sum ----------------------------------------------------------
    rng = np.random.default_rng(17)
    k = 30
    table = build_table(0.6, k)
    buf = HistoryBuffer(k + 1, (5, 5))
    fields = []
    for _ in range(k + 1):
        f = np.zeros((5, 5))
        f[1:-1, 1:-1] = rng.normal(size=(3, 3))
        fields.append(f)
        buf.append(f)
    arrays["hs_fields"] = np.stack(fields)
    for name, sched in (("full", full_schedule(k)), ("adaptive3", adaptive_schedule(k, 3)),
                        ("short7", short_schedule(k, 7.0, 1.0))):
        arrays[f"hs_out_{name}"] = history_sum(buf, sched, table, k)
    rng = np.random.default_rng(23)
    k = 700
    table = build_table(0.8, k)
    buf = HistoryBuffer(k + 1, (8, 16), byte_cap=None)
    fields = rng.normal(size=(k + 1, 8, 16))
    for f in fields:
        buf.append(f)
    arrays["hs2_fields"] = fields
    for name, sched in (("full", full_schedule(k)), ("adaptive5", adaptive_schedule(k, 5)),
                        ("adaptive2", adaptive_schedule(k, 2))):
        arrays[f"hs2_out_{name}"] = history_sum(buf, sched, table, k)

    # ---- 2D solver.run cases ---------------------------------------------------
    def record_run(name, config, *, inputs=None):
        result = run(config)
        steps = np.array([s for s, _ in result.snapshots], dtype=np.int64)
        arrays[f"run_{name}_steps"] = steps
        arrays[f"run_{name}_snaps"] = np.stack([g.data for _, g in result.snapshots])
        if inputs is not None:
            arrays[f"run_{name}_u0"] = inputs
        meta["cases"][name] = {
            "kind": "run2d",
            "gamma": config.gamma, "alpha": config.alpha, "beta": config.beta,
            "dt": config.dt, "dx": config.dx, "nx": config.nx, "ny": config.ny,
            "n_steps": config.n_steps, "snapshot_every": config.snapshot_every,
            "sources": [list(s) for s in config.sources] if inputs is None else None,
            "strategy": [config.strategy.tag, config.strategy.param],
        }

    base = dict(gamma=0.5, alpha=1.0, beta=0.0, dt=1.0, dx=10.0, nx=8, ny=8, n_steps=10,
                sources=((4, 4, 10.0),))
    record_run("small", SimulationConfig(**base))
    record_run("small_decay", SimulationConfig(**{**base, "beta": 0.07, "dt": 0.5, "n_steps": 30,
                                                  "snapshot_every": 1}))
    point = SimulationConfig(gamma=0.75, alpha=1.0, beta=0.0, dt=1.0, dx=10.0, nx=20, ny=20,
                             n_steps=1500, sources=((10, 10, 10.0),))
    record_run("point_full", point)
    record_run("point_short100", replace(point, strategy=ShortMemory(100.0)))
    record_run("point_adaptive3", replace(point, strategy=AdaptiveMemory(3)))
    record_run("point_adaptive5", replace(point, strategy=AdaptiveMemory(5)))
    record_run("point_g05_adaptive1500", replace(point, gamma=0.5, strategy=AdaptiveMemory(1500)))
    record_run("ftcs_g1", SimulationConfig(gamma=1.0, alpha=1.0, beta=0.0, dt=0.5, dx=5.0, nx=9, ny=9,
                                           n_steps=25, sources=((4, 4, 2.0),)))
    spread = SimulationConfig(gamma=0.9, alpha=1.0, beta=0.0, dt=0.5, dx=5.0, nx=100, ny=100, n_steps=200,
                              sources=((50, 50, 0.1), (49, 50, 0.05), (51, 50, 0.05), (50, 49, 0.05),
                                       (50, 51, 0.05)), snapshot_every=20)
    record_run("spread_g09_adaptive4", replace(spread, strategy=AdaptiveMemory(4)))
    # c2-like (reduced): dense seeded field, gamma 0.8, r 0.1, beta 0.1, adaptive:5
    n = 48
    dx = 1.0 / (n - 1)
    x = np.arange(n) * dx
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0 = np.exp(-((X - 0.5) ** 2 + (Y - 0.5) ** 2) / (2 * 0.1**2))
    u0 = u0 + np.random.default_rng(2).uniform(0.0, 0.01, size=u0.shape)
    u0[0, :] = u0[-1, :] = 0.0
    u0[:, 0] = u0[:, -1] = 0.0
    dt = (0.1 * dx**2 / 1.0) ** (1 / 0.8)
    c2s = SimulationConfig(gamma=0.8, alpha=1.0, beta=0.1, dt=dt, dx=dx, nx=n, ny=n, n_steps=600,
                           sources=dense_sources(u0), strategy=AdaptiveMemory(5), snapshot_every=50)
    record_run("c2_small", c2s, inputs=u0)
    record_run("c2_small_full", replace(c2s, strategy=FullMemory(), n_steps=300), inputs=u0)
    record_run("c2_small_short", replace(c2s, strategy=ShortMemory(37.5 * dt), n_steps=300), inputs=u0)
    # divergence: the reference test configuration (tests/test_solver.py:245-251)
    try:
        run(SimulationConfig(**{**base, "gamma": 1.0, "dt": 1.0, "dx": 1.0, "n_steps": 500}))
        raise SystemExit("expected divergence")
    except DivergenceError as exc:
        meta["divergence"] = {"step": exc.step, "peak": exc.peak}

    # ---- n-D compositions --------------------------------------------------------
    def record_nd(name, u0s, gammas, dts, alpha, dx, reaction, strategy, n_steps, snapshot_every):
        snaps_all = []
        steps = None
        for b in range(len(u0s)):
            snaps = composed_run(u0s[b], float(gammas[b]), float(dts[b]), alpha, dx, reaction, strategy,
                                 n_steps, snapshot_every)
            steps = [s for s, _ in snaps]
            snaps_all.append(np.stack([u for _, u in snaps]))
        arrays[f"nd_{name}_u0"] = np.stack(u0s)
        arrays[f"nd_{name}_gamma"] = np.asarray(gammas, dtype=np.float64)
        arrays[f"nd_{name}_dt"] = np.asarray(dts, dtype=np.float64)
        arrays[f"nd_{name}_steps"] = np.asarray(steps, dtype=np.int64)
        arrays[f"nd_{name}_snaps"] = np.stack(snaps_all, axis=1)  # (S, B, *shape)
        meta["cases"][name] = {
            "kind": "nd", "alpha": alpha, "dx": dx, "reaction": list(reaction),
            "strategy": [strategy.tag, strategy.param], "n_steps": n_steps,
            "snapshot_every": snapshot_every,
        }

    # c1 exactly (BASELINE.json configs[0])
    dx = 0.01
    x = np.arange(101) * dx
    u0 = np.exp(-((x - 0.5) ** 2) / (2 * 0.05**2))
    u0[0] = u0[-1] = 0.0
    dt = (0.2 * dx**2 / 1.0) ** (1 / 0.5)
    record_nd("c1", [u0], [0.5], [dt], 1.0, dx, ("linear", 0.0), FullMemory(), 2000, 100)
    # 1D adaptive with decay
    record_nd("1d_adaptive", [u0], [0.7], [(0.2 * dx**2) ** (1 / 0.7)], 1.0, dx, ("linear", 0.05),
              AdaptiveMemory(4), 900, 150)
    # 3D saturating, full and adaptive (c4 shape family, reduced)
    n = 14
    dx = 1.0 / (n - 1)
    rng = np.random.default_rng(3)
    v = rng.uniform(0.0, 1.0, size=(n, n, n))
    for _ in range(3):
        w = np.zeros_like(v)
        c = (slice(1, -1),) * 3
        w[c] = (v[2:, 1:-1, 1:-1] + v[:-2, 1:-1, 1:-1] + v[1:-1, 2:, 1:-1] + v[1:-1, :-2, 1:-1]
                + v[1:-1, 1:-1, 2:] + v[1:-1, 1:-1, :-2]) / 6.0
        v = w
    dt = (0.05 * dx**2) ** (1 / 0.7)
    record_nd("3d_sat_full", [v], [0.7], [dt], 1.0, dx, ("saturating", 0.5, 0.2), FullMemory(), 250, 50)
    record_nd("3d_sat_adaptive", [v], [0.7], [dt], 1.0, dx, ("saturating", 0.5, 0.2), AdaptiveMemory(5),
              400, 80)
    # batched 1D ensemble, per-member gamma (c5 family, reduced)
    rng = np.random.default_rng(4)
    B, n = 6, 64
    dx = 1.0 / (n - 1)
    x = np.arange(n) * dx
    gammas = rng.uniform(0.3, 0.9, size=B)
    centres = rng.uniform(0.2, 0.8, size=B)
    u0s = []
    for c in centres:
        u = np.exp(-((x - c) ** 2) / (2 * 0.03**2))
        u[0] = u[-1] = 0.0
        u0s.append(u)
    dts = [(0.2 * dx**2) ** (1 / g) for g in gammas]
    record_nd("batch_adaptive", u0s, gammas, dts, 1.0, dx, ("linear", 0.0), AdaptiveMemory(5), 1200, 200)
    # batched short memory: per-member horizon floor(L/dt_b)
    dts2 = [0.01 * (b + 1) for b in range(B)]
    record_nd("batch_short", u0s, [0.6] * B, dts2, 1.0e-4, dx, ("linear", 0.0), ShortMemory(0.4), 300, 60)

    # ---- drivers on top of the path: benchmark.py:69-193 ------------------------------
    from fracgrid.benchmark import gamma_sweep, run_comparison

    cmp_cfg = replace(point, n_steps=300)
    recs = run_comparison(cmp_cfg, (0.5, 0.9), (10.0, 50.0), (3, 5))
    meta["comparison"] = [[r.strategy, r.param, r.gamma, r.err_l2_pct, r.err_linf_pct, r.message] for r in recs]
    sweep_cfg = replace(spread, n_steps=60, snapshot_every=10)
    meta["sweep_gammas"] = [0.5, 0.75, 1.0]
    for e in gamma_sweep(sweep_cfg, (0.5, 0.75, 1.0)):
        arrays[f"sweep_{e.gamma}_profile"] = e.profile
        arrays[f"sweep_{e.gamma}_steps"] = e.trace_steps
        arrays[f"sweep_{e.gamma}_values"] = e.trace_values

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    size = os.path.getsize(os.path.join(HERE, "golden.npz"))
    print(f"wrote {len(arrays)} arrays ({size/1e6:.2f} MB) and {len(meta['cases'])} run cases")


if __name__ == "__main__":
    main()
