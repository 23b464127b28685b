"""Host-side logic of the drop-in (CPU only): config validation, snapshot cadence,
strategy duck-typing, host scalars, extension configs, workloads, term counts."""

import math
import warnings

import numpy as np
import pytest

import paper_1004_5128_b200 as fg
from paper_1004_5128_b200 import _engine as E
from paper_1004_5128_b200 import workloads as W


def make_config(**kw):
    d = dict(gamma=0.5, alpha=1.0, beta=0.0, dt=1.0, dx=10.0, nx=8, ny=8, n_steps=10, sources=((4, 4, 10.0),))
    d.update(kw)
    return fg.SimulationConfig(**d)


# mirrors tests/test_solver.py:47-101 of the reference
@pytest.mark.parametrize("gamma", [0.0, -0.5, 1.5, 2.0])
def test_gamma_range(gamma):
    with pytest.raises(ValueError, match="gamma"):
        make_config(gamma=gamma)


def test_parameter_validation():
    for kw, pat in ((dict(alpha=-1.0), "alpha"), (dict(beta=-0.1), "beta"), (dict(dt=0.0), "dt"),
                    (dict(dx=-5.0), "dx"), (dict(nx=2), "3x3"), (dict(n_steps=-1), "n_steps"),
                    (dict(snapshot_every=0), "snapshot_every"), (dict(sources=((0, 4, 1.0),)), "interior"),
                    (dict(sources=((4, 4, 1.0), (4, 4, 2.0))), "duplicate"),
                    (dict(sources=((4, 4, math.nan),)), "non-finite")):
        with pytest.raises(ValueError, match=pat):
            make_config(**kw)


def test_stability_warning_and_ratio():
    with pytest.warns(fg.StabilityWarning):
        make_config(gamma=1.0, dt=1.0, dx=1.0, alpha=0.3)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        make_config(gamma=1.0, dt=1.0, dx=2.0, alpha=1.0)
    assert make_config(gamma=0.5, alpha=2.0, dt=4.0, dx=10.0).stability_ratio == pytest.approx(0.04)


def test_snapshot_cadence_and_steps():
    assert make_config(snapshot_every=7).snapshot_cadence == 7
    assert make_config(n_steps=200).snapshot_cadence == 2
    assert make_config(n_steps=1500).snapshot_cadence == 15
    assert make_config(n_steps=0).snapshot_cadence == 1
    assert E.snapshot_steps(5, 2) == [0, 2, 4, 5]
    assert E.snapshot_steps(0, 1) == [0]
    # identical to the reference loop (solver.py:251-256) for many (n, cadence)
    for n in range(0, 60):
        for cad in range(1, 12):
            ref = [0]
            for k in range(n):
                done = k + 1
                if (done % cad == 0 or done == n) and ref[-1] != done:
                    ref.append(done)
            assert E.snapshot_steps(n, cad) == ref


def test_strategy_duck_typing():
    assert E.strategy_spec(fg.FullMemory()) == ("full", 0)
    assert E.strategy_spec(fg.ShortMemory(12.5)) == ("short", 12.5)
    assert E.strategy_spec(fg.AdaptiveMemory(5)) == ("adaptive", 5)

    class Foreign:
        tag = "adaptive"
        base = 3

    assert E.strategy_spec(Foreign()) == ("adaptive", 3)
    with pytest.raises(TypeError):
        E.strategy_spec(object())
    with pytest.raises(ValueError):
        fg.AdaptiveMemory(3.0)
    with pytest.raises(ValueError):
        fg.ShortMemory(math.inf)
    assert fg.AdaptiveMemory(7).param == 7.0 and fg.ShortMemory(25.0).param == 25.0 and fg.FullMemory().param == 0.0


def test_host_scalars_match_reference_formula():
    for alpha, beta, gamma, dt, dx in ((1.0, 0.1, 0.8, 5.4e-8, 1 / 255), (1.0, 0.0, 0.6, 2e-12, 1 / 1023),
                                       (2.0, 0.07, 0.5, 4.0, 10.0)):
        decay, diffuse = E.host_scalars(alpha, beta, gamma, dt, dx)
        assert decay == 1.0 - beta * dt
        assert diffuse == alpha * dt**gamma / dx**2
    assert E.short_horizon(500 * 1.997e-12, 1.997e-12) == 500
    assert E.short_horizon(1.0, 1e-300) == 1 << 62


def test_memory_budget_checked_before_device():
    cfg = make_config(n_steps=10_000, history_byte_cap=100_000)
    with pytest.raises(fg.MemoryBudgetError, match="cap"):
        E.check_history_budget(fg.solver.problem_from_config(cfg))


def test_field_config_validation():
    u = np.zeros((5, 5))
    u[2, 2] = 1.0
    p = fg.FieldConfig(initial=u, dx=1.0, gamma=0.5, dt=1.0, n_steps=3).to_problem()
    assert p.batch == 1 and p.shape == (5, 5) and p.reaction == ("linear", 0.0)
    bad = u.copy()
    bad[0, 1] = 1.0
    with pytest.raises(ValueError, match="boundary"):
        fg.FieldConfig(initial=bad, dx=1.0, gamma=0.5, dt=1.0, n_steps=3).to_problem()
    with pytest.raises(ValueError, match="gamma"):
        fg.FieldConfig(initial=u, dx=1.0, gamma=1.2, dt=1.0, n_steps=3).to_problem()
    with pytest.raises(ValueError, match="dimensions"):
        fg.FieldConfig(initial=np.zeros((3, 3, 3, 3)), dx=1.0, gamma=0.5, dt=1.0, n_steps=3).to_problem()
    with pytest.raises(ValueError, match="km"):
        fg.FieldConfig(initial=u, dx=1.0, gamma=0.5, dt=1.0, n_steps=3, reaction=fg.Saturating(1.0, 0.0)).to_problem()
    ens = fg.FieldConfig(initial=np.zeros((4, 9)), dx=1.0, gamma=[0.3, 0.4, 0.5, 0.6], dt=1.0, n_steps=3,
                         batched=True).to_problem()
    assert ens.batch == 4 and ens.gamma.tolist() == [0.3, 0.4, 0.5, 0.6] and ens.dt.tolist() == [1.0] * 4


def test_workloads_match_baseline_json():
    c1 = W.c1()
    assert c1.initial.shape == (101,) and c1.snapshot_every == 100 and c1.n_steps == 2000
    assert E.host_scalars(1.0, 0.0, 0.5, c1.dt, c1.dx)[1] == pytest.approx(0.2, rel=1e-14)
    c2 = W.c2(n_steps=10)
    assert c2.initial.shape == (256, 256) and c2.strategy == fg.AdaptiveMemory(5)
    assert c2.reaction == fg.LinearDecay(0.1)
    assert E.host_scalars(1.0, 0.1, 0.8, c2.dt, c2.dx)[1] == pytest.approx(0.1, rel=1e-13)
    assert np.all(c2.initial[0] == 0) and c2.initial.max() <= 1.01
    c3 = W.c3("short", n_steps=10, n=64)
    assert math.floor(c3.strategy.length / c3.dt) == 500
    c5 = W.c5(n_steps=10, members=16, n=512)
    assert c5.initial.shape == (16, 512) and c5.batched
    g = np.asarray(c5.gamma)
    assert g.min() >= 0.3 and g.max() <= 0.9
    sub = W.subset_members(c5, [0, 5])
    assert sub.initial.shape == (2, 512) and np.asarray(sub.gamma).tolist() == [g[0], g[5]]


def test_term_counts_match_oracle():
    from oracle import fg_oracle as fo

    p = W.c2(n_steps=300).to_problem()
    assert p.terms() == fo.count_terms("adaptive", 300, 5) * 256 * 256
    c5 = W.c5(n_steps=50, members=3, n=512).to_problem()
    assert c5.terms() == fo.count_terms("adaptive", 50, 5) * 3 * 512
    short = W.c3("short", n_steps=600, n=32).to_problem()
    assert short.terms() == fo.count_terms("short", 600, short.param, float(short.dt[0])) * 32 * 32


def test_relative_error_matches_reference_formula():
    from paper_1004_5128_b200.benchmark import BenchmarkRecord, relative_error, source_cell

    ref = np.zeros((5, 5))
    ref[2, 2], ref[1, 2] = 2.0, 1.0
    app = ref.copy()
    app[2, 2] = 1.5
    l2, linf = relative_error(fg.Grid2D(app, 1.0), fg.Grid2D(ref, 1.0))
    assert l2 == pytest.approx(0.5 / math.sqrt(5.0) * 100.0)
    assert linf == pytest.approx(25.0)
    with pytest.raises(ValueError, match="zero"):
        relative_error(fg.Grid2D(app, 1.0), fg.Grid2D(np.zeros((5, 5)), 1.0))
    assert BenchmarkRecord("short", 1.0, 0.5, 0.1, 1.0, 1.0, message="x").failed
    assert source_cell(make_config(sources=((3, 3, 1.0), (4, 4, -2.0)))) == (4, 4)
    assert source_cell(make_config(sources=())) == (4, 4)
