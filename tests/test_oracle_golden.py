"""Pin the CPU oracle against the reference's own outputs (golden fixtures).

CPU only.  Bit-exact where the reference is bit-exact: ψ, schedules, and every
``solver.run`` / composed n-D case (same contraction, same op order).
"""

import hashlib

import numpy as np
import pytest

from oracle import fg_oracle as fo


def _sched_hash(kind, kmax, param, dt=1.0):
    h = hashlib.sha256()
    for k in range(kmax + 1):
        offs, wts = fo.schedule(kind, k, param, dt)
        h.update(np.int64(offs.size).astype("<i8").tobytes())
        h.update(offs.astype("<i8").tobytes())
        h.update(wts.astype("<i8").tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("gamma", [0.1, 0.3, 0.35, 0.5, 0.6, 0.7, 0.75, 0.8, 0.9, 1.0, 1.5, 1.99])
def test_psi_tables_bitwise(golden, gamma):
    assert np.array_equal(fo.build_table(gamma, 64), golden[f"psi_{gamma}_64"])
    digest = hashlib.sha256(fo.build_table(gamma, 10000).astype("<f8").tobytes()).hexdigest()
    assert digest == golden.meta["psi"][str(gamma)]


def test_psi_frozen_values():
    # coefficients tests/test_coefficients.py:18-22,30-34,51-55
    assert [fo.psi(0.5, m) for m in range(4)] == [1.0, -0.5, -0.125, -0.0625]
    assert all(fo.psi(1.0, m) == 0.0 for m in (1, 2, 3, 10, 100))
    t = fo.build_table(0.5, 1000)
    assert np.cumsum(t[:3]).tolist() == [1.0, 0.5, 0.375]
    np.testing.assert_allclose(np.sum(t[:101]), 0.05634847900925633, rtol=1e-13)
    np.testing.assert_allclose(np.sum(t), 0.017839011145854074, rtol=1e-13)
    for bad in (0.0, 2.0, -1.0, float("nan")):
        with pytest.raises(ValueError, match="gamma"):
            fo.build_table(bad, 3)


def test_schedule_pairs(golden):
    for key, pairs in golden.meta["sched_pairs"].items():
        a, k = map(int, key.split("/"))
        offs, wts = fo.schedule("adaptive", k, a)
        assert list(zip(offs.tolist(), wts.tolist())) == [tuple(p) for p in pairs], key


@pytest.mark.parametrize("base", ["2", "3", "4", "5", "8", "12", "20", "40", "100", "1500"])
def test_adaptive_schedule_hash_all_k(golden, base):
    assert _sched_hash("adaptive", 10000, int(base)) == golden.meta["sched_hash"][base]


def test_full_and_short_schedule_hash(golden):
    assert _sched_hash("full", 2000, 0) == golden.meta["sched_hash"]["full"]
    for key, digest in golden.meta["short_hash"].items():
        L, dt = map(float, key.split("/"))
        assert _sched_hash("short", 3000, L, dt) == digest, key


def test_history_sum_bitwise(golden):
    table = fo.build_table(0.6, 30)
    H = golden["hs_fields"]
    for name, (kind, p, dt) in {"full": ("full", 0, 1.0), "adaptive3": ("adaptive", 3, 1.0),
                                "short7": ("short", 7.0, 1.0)}.items():
        offs, wts = fo.schedule(kind, 30, p, dt)
        assert np.array_equal(fo.history_sum(H, offs, wts, table, 30), golden[f"hs_out_{name}"]), name
    table = fo.build_table(0.8, 700)
    H = golden["hs2_fields"]
    for name, (kind, p) in {"full": ("full", 0), "adaptive5": ("adaptive", 5),
                            "adaptive2": ("adaptive", 2)}.items():
        offs, wts = fo.schedule(kind, 700, p)
        assert np.array_equal(fo.history_sum(H, offs, wts, table, 700), golden[f"hs2_out_{name}"]), name


def test_stencil_known_answers():
    # grid tests/test_grid.py:18-29, 62-69
    d = np.zeros((5, 5))
    d[2, 2] = 10.0
    out = fo.stencil(d)
    assert out[2, 2] == -40.0 and out[1, 2] == out[3, 2] == out[2, 1] == out[2, 3] == 10.0
    assert out[1, 1] == 0.0
    d = np.zeros((9, 9))
    d[4, 4] = 3.0
    d[3, 4] = d[5, 4] = d[4, 3] = d[4, 5] = 1.0
    out = fo.stencil(d)
    assert np.array_equal(out, out.T) and np.array_equal(out, out[::-1])


FAST_CASES = ["small", "small_decay", "ftcs_g1", "c2_small", "c2_small_full", "c2_small_short",
              "point_adaptive5", "1d_adaptive", "3d_sat_full", "3d_sat_adaptive", "batch_adaptive",
              "batch_short", "c1", "spread_g09_adaptive4"]


@pytest.mark.parametrize("name", FAST_CASES)
def test_oracle_run_bitwise(golden, name):
    p = golden.problem_params(name)
    res = fo.run(fo.OracleProblem(**p))
    steps, snaps = golden.expected(name)
    assert [s for s, _ in res["snapshots"]] == steps.tolist()
    got = np.stack([u for _, u in res["snapshots"]])
    assert np.array_equal(got, snaps), f"{name}: max |diff| {np.abs(got - snaps).max()}"


def test_oracle_divergence(golden):
    u0 =np.zeros((1, 8, 8))
    u0[0, 4, 4] = 10.0
    prob = fo.OracleProblem(u0=u0, gamma=np.array([1.0]), dt=np.array([1.0]), alpha=1.0, dx=1.0,
                            reaction=("linear", 0.0), strategy=("full", 0), n_steps=500)
    with np.errstate(over="ignore", invalid="ignore"), pytest.raises(fo.OracleDivergence) as exc:
        fo.run(prob)
    assert exc.value.step == golden.meta["divergence"]["step"]
    assert exc.value.peak == golden.meta["divergence"]["peak"]
