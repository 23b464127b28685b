"""The rebind seam on the CPU: exception classes and ``install``.

The reference's drivers catch ``fracgrid.solver.DivergenceError``
(/root/reference/pkg/src/fracgrid/benchmark.py:114-128, cli.py:469-479); this
package's errors must be instances of it whenever ``fracgrid`` is loaded.  The
stand-in-module tests run anywhere; the ones marked ``reference`` import the
real reference from /root/reference (this container only) and mirror its own
fault-injection test (pkg/tests/test_benchmark.py:105-124) with the bridged
error raised by a rebound ``run``.
"""

import math
import os
import sys
import types

import numpy as np
import pytest

from paper_1004_5128_b200 import _engine, integrate

REF_SRC = "/root/reference/pkg/src"


def _standin(monkeypatch):
    """A minimal ``fracgrid`` with the reference's exception classes (solver.py:38-46, grid.py:16-21)."""
    pkg = types.ModuleType("fracgrid")
    solver = types.ModuleType("fracgrid.solver")
    grid = types.ModuleType("fracgrid.grid")

    class DivergenceError(RuntimeError):
        def __init__(self, step, peak):
            super().__init__(f"solution diverged at step {step}: max |u| reached {peak!r}")
            self.step = step
            self.peak = peak

    class MemoryBudgetError(ValueError):
        pass

    class HistoryCapacityError(ValueError):
        pass

    solver.DivergenceError = DivergenceError
    grid.MemoryBudgetError = MemoryBudgetError
    grid.HistoryCapacityError = HistoryCapacityError
    pkg.solver, pkg.grid = solver, grid
    for name, mod in (("fracgrid", pkg), ("fracgrid.solver", solver), ("fracgrid.grid", grid)):
        monkeypatch.setitem(sys.modules, name, mod)
    return pkg


def test_own_classes_without_reference(monkeypatch):
    for name in ("fracgrid", "fracgrid.solver", "fracgrid.grid"):
        monkeypatch.delitem(sys.modules, name, raising=False)
    err = _engine.divergence(7, math.inf)
    assert type(err) is _engine.DivergenceError
    assert str(err) == "solution diverged at step 7: max |u| reached inf"
    assert _engine.error_class(_engine.MemoryBudgetError) is _engine.MemoryBudgetError


def test_bridged_errors_are_both_classes(monkeypatch):
    ref = _standin(monkeypatch)
    err = _engine.divergence(7, 2.5)
    assert isinstance(err, _engine.DivergenceError) and isinstance(err, ref.solver.DivergenceError)
    assert (err.step, err.peak) == (7, 2.5)
    assert str(err) == str(ref.solver.DivergenceError(7, 2.5))
    assert _engine.error_class(_engine.DivergenceError) is type(err)  # cached, one class per pair
    with pytest.raises(ref.grid.MemoryBudgetError, match="cap"):
        raise _engine.budget_error("over the cap")
    cap = _engine.error_class(_engine.HistoryCapacityError)
    assert issubclass(cap, ref.grid.HistoryCapacityError) and issubclass(cap, ValueError)


def test_budget_check_raises_reference_class(monkeypatch):
    ref = _standin(monkeypatch)
    p = _engine.Problem(u0=np.zeros((1, 64, 64)), gamma=np.array([0.5]), dt=np.array([1.0]), alpha=1.0, dx=1.0,
                        reaction=("linear", 0.0), kind="full", param=0, n_steps=1000, cadence=10,
                        history_byte_cap=1024)
    with pytest.raises(ref.grid.MemoryBudgetError, match="over the cap of 1024"):
        _engine.check_history_budget(p)


def test_install_rebinds_and_undoes(monkeypatch):
    ref = _standin(monkeypatch)
    bench = types.ModuleType("fracgrid.benchmark")
    cli = types.ModuleType("fracgrid.cli")
    sentinel = object()
    bench.run = cli.run = sentinel
    ref.benchmark, ref.cli = bench, cli
    undo = integrate.install(ref)
    assert bench.run is integrate.gpu_run and cli.run is integrate.gpu_run
    undo()
    assert bench.run is sentinel and cli.run is sentinel


# ------------------------------------------------------------- real reference --

@pytest.fixture
def fracgrid_ref(monkeypatch):
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference tree not present (GPU box)")
    monkeypatch.syspath_prepend(REF_SRC)
    import fracgrid
    import fracgrid.benchmark
    import fracgrid.cli

    return fracgrid


def _small(fr, **kw):
    d = dict(gamma=0.5, alpha=1.0, beta=0.0, dt=1.0, dx=10.0, nx=10, ny=10, n_steps=40,
             sources=((5, 5, 10.0),), snapshot_every=40)
    d.update(kw)
    return fr.solver.SimulationConfig(**d)


def test_reference_run_comparison_records_bridged_divergence(fracgrid_ref):
    """benchmark.py:114-128 turns our DivergenceError into a NaN record (test_benchmark.py:105-124)."""
    fr = fracgrid_ref
    real_run = fr.benchmark.run

    def gpu_like_run(config, **kw):  # stands in for the GPU run: raises this package's (bridged) error
        if isinstance(config.strategy, fr.schedule.ShortMemory) and config.strategy.length == 13.0:
            raise _engine.divergence(7, float("inf"))
        return real_run(config, **kw)

    undo = integrate.install(fr, run=gpu_like_run)
    try:
        records = fr.benchmark.run_comparison(_small(fr), gammas=(0.5,), short_lengths=(13.0, 20.0),
                                              adaptive_bases=())
    finally:
        undo()
    failed = [r for r in records if r.failed]
    assert len(failed) == 1 and failed[0].strategy == "short" and failed[0].param == 13.0
    assert np.isnan(failed[0].err_l2_pct) and "step 7" in failed[0].message
    assert fr.benchmark.run is real_run


def test_reference_cli_exit_code_on_bridged_divergence(fracgrid_ref, tmp_path, capsys):
    """cli.py:469-479: a DivergenceError from the rebound run exits with EXIT_DIVERGED (3)."""
    fr = fracgrid_ref

    def diverging_run(config, **kw):
        raise _engine.divergence(3, 1.5e300)

    undo = integrate.install(fr, run=diverging_run)
    try:
        rc = fr.cli.main(["simulate", "--out-dir", str(tmp_path), "--gamma", "0.5", "--memory", "full",
                          "--dt", "1.0", "--dx", "10.0", "--grid", "10x10", "--steps", "5"])
    finally:
        undo()
    assert rc == fr.cli.EXIT_DIVERGED
    assert "diverged at step 3" in capsys.readouterr().err
