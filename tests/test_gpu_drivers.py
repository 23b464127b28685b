"""The reference's drivers (benchmark.py:69-193) on the GPU stepper match the goldens."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_run_comparison_matches_reference(cuda_device, golden):
    import paper_1004_5128_b200 as fg
    from paper_1004_5128_b200.benchmark import run_comparison

    cfg = fg.SimulationConfig(gamma=0.75, alpha=1.0, beta=0.0, dt=1.0, dx=10.0, nx=20, ny=20, n_steps=300,
                              sources=((10, 10, 10.0),))
    recs = run_comparison(cfg, (0.5, 0.9), (10.0, 50.0), (3, 5))
    want = golden.meta["comparison"]
    assert len(recs) == len(want)
    for r, (strategy, param, gamma, l2, linf, msg) in zip(recs, want):
        assert (r.strategy, r.param, r.gamma, r.message) == (strategy, param, gamma, msg)
        assert r.err_l2_pct == pytest.approx(l2, rel=1e-8, abs=1e-12)
        assert r.err_linf_pct == pytest.approx(linf, rel=1e-8, abs=1e-12)
        assert r.elapsed_s >= 0.0


def test_gamma_sweep_matches_reference(cuda_device, golden):
    import paper_1004_5128_b200 as fg
    from paper_1004_5128_b200.benchmark import gamma_sweep

    cfg = fg.SimulationConfig(gamma=0.9, alpha=1.0, beta=0.0, dt=0.5, dx=5.0, nx=100, ny=100, n_steps=60,
                              sources=((50, 50, 0.1), (49, 50, 0.05), (51, 50, 0.05), (50, 49, 0.05),
                                       (50, 51, 0.05)), snapshot_every=10)
    for e in gamma_sweep(cfg, tuple(golden.meta["sweep_gammas"])):
        assert np.array_equal(e.trace_steps, golden[f"sweep_{e.gamma}_steps"])
        np.testing.assert_allclose(e.profile, golden[f"sweep_{e.gamma}_profile"], rtol=1e-10, atol=1e-16)
        np.testing.assert_allclose(e.trace_values, golden[f"sweep_{e.gamma}_values"], rtol=1e-10, atol=1e-16)


def test_comparison_records_divergence(cuda_device):
    import warnings

    import paper_1004_5128_b200 as fg
    from paper_1004_5128_b200.benchmark import run_comparison

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cfg = fg.SimulationConfig(gamma=1.0, alpha=1.0, beta=0.0, dt=1.0, dx=1.0, nx=8, ny=8, n_steps=500,
                                  sources=((4, 4, 10.0),))
    # the full-memory reference run itself diverges: like benchmark.py:94 the
    # driver does not swallow that (only candidate cells become NaN records)
    with pytest.raises(fg.DivergenceError):
        run_comparison(cfg, (1.0,), (3.0,), (2,))


def test_rebind_seam_reference_handler_catches_gpu_divergence(cuda_device, monkeypatch):
    """INTEGRATION.md §1 on the GPU: with a stand-in ``fracgrid`` loaded (the
    reference's exception classes, solver.py:38-46), ``integrate.install`` rebinds
    the driver's ``run`` and a diverging candidate run on the GPU is caught by the
    driver's ``except fracgrid.solver.DivergenceError`` — a NaN record, as
    benchmark.py:114-128 does (mirror of pkg/tests/test_benchmark.py:105-124)."""
    import math
    import sys
    import types
    import warnings

    import paper_1004_5128_b200 as fg
    from paper_1004_5128_b200 import integrate

    pkg = types.ModuleType("fracgrid")
    solver = types.ModuleType("fracgrid.solver")
    bench = types.ModuleType("fracgrid.benchmark")

    class DivergenceError(RuntimeError):
        def __init__(self, step, peak):
            super().__init__(f"solution diverged at step {step}: max |u| reached {peak!r}")
            self.step, self.peak = step, peak

    solver.DivergenceError = DivergenceError
    bench.run = None

    def cells(configs):  # the shape of benchmark.py:106-128: failures become NaN records
        out = []
        for cfg in configs:
            try:
                res = bench.run(cfg)
                out.append((float(np.abs(res.final.data).max()), ""))
            except solver.DivergenceError as exc:
                out.append((math.nan, str(exc)))
        return out

    pkg.solver, pkg.benchmark = solver, bench
    for name, mod in (("fracgrid", pkg), ("fracgrid.solver", solver), ("fracgrid.benchmark", bench)):
        monkeypatch.setitem(sys.modules, name, mod)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        bad = fg.SimulationConfig(gamma=1.0, alpha=1.0, beta=0.0, dt=1.0, dx=1.0, nx=8, ny=8, n_steps=500,
                                  sources=((4, 4, 10.0),))
    good = fg.SimulationConfig(gamma=0.5, alpha=1.0, beta=0.0, dt=1.0, dx=10.0, nx=10, ny=10, n_steps=40,
                               sources=((5, 5, 10.0),))
    undo = integrate.install(pkg)
    try:
        recs = cells([good, bad])
    finally:
        undo()
    assert bench.run is None
    assert recs[0][1] == "" and math.isfinite(recs[0][0])
    assert math.isnan(recs[1][0])
    with pytest.raises(fg.DivergenceError) as exc:  # the same error through the package's own class
        fg.run(bad)
    assert isinstance(exc.value, DivergenceError)
    assert recs[1][1] == str(exc.value) and f"step {exc.value.step}" in recs[1][1]
