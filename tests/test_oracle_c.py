"""The C restatement is bitwise identical to the NumPy one and to the goldens (CPU)."""

import numpy as np
import pytest

from oracle import fg_oracle as fo
from oracle import fg_oracle_c as foc

CASES = ["small", "small_decay", "ftcs_g1", "c2_small", "c2_small_full", "c2_small_short",
         "point_full", "point_short100", "point_adaptive3", "point_adaptive5", "point_g05_adaptive1500",
         "spread_g09_adaptive4", "c1", "1d_adaptive", "3d_sat_full", "3d_sat_adaptive",
         "batch_adaptive", "batch_short"]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("threads", [1, 3])
def test_c_oracle_matches_golden(golden, name, threads):
    p = fo.OracleProblem(**golden.problem_params(name))
    res = foc.run(p, nthreads=threads)
    steps, snaps = golden.expected(name)
    assert [s for s, _ in res["snapshots"]] == steps.tolist()
    got = np.stack([u for _, u in res["snapshots"]])
    assert np.array_equal(got, snaps), f"{name}: max |diff| {np.abs(got - snaps).max()}"


def test_c_schedule_and_table_match():
    import ctypes as C

    L = foc.lib()
    offs = np.empty(20000, np.int64)
    wts = np.empty(20000, np.int64)
    for kind, param, dt in (("adaptive", 5, 1.0), ("adaptive", 2, 1.0), ("short", 7.25, 0.25), ("full", 0, 1.0)):
        for k in list(range(0, 300)) + [999, 4096, 9999]:
            n = L.fgo_schedule(foc._KINDS[kind], k, float(param), dt, offs.ctypes.data, wts.ctypes.data, 20000)
            eo, ew = fo.schedule(kind, k, param, dt)
            assert n == eo.size and np.array_equal(offs[:n], eo) and np.array_equal(wts[:n], ew)
    t = np.empty(10001)
    assert L.fgo_build_table(C.c_double(0.37), 10000, t.ctypes.data) == 0
    assert np.array_equal(t, fo.build_table(0.37, 10000))


def test_c_prefix_is_exact(golden):
    p = fo.OracleProblem(**golden.problem_params("c2_small"))
    full = foc.run(p)
    pre = foc.run(p, max_steps=250)
    by_step = dict(full["snapshots"])
    for s, u in pre["snapshots"]:
        assert np.array_equal(u, by_step[s])


def test_c_divergence(golden):
    u0 = np.zeros((1, 8, 8))
    u0[0, 4, 4] = 10.0
    p = fo.OracleProblem(u0=u0, gamma=np.array([1.0]), dt=np.array([1.0]), alpha=1.0, dx=1.0,
                         reaction=("linear", 0.0), strategy=("full", 0), n_steps=500)
    with pytest.raises(fo.OracleDivergence) as exc:
        foc.run(p)
    assert exc.value.step == golden.meta["divergence"]["step"]
    assert exc.value.peak == golden.meta["divergence"]["peak"]
