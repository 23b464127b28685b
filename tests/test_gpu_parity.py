"""GPU parity: the sm_100a path against the reference goldens and the CPU oracle.

Bar (BASELINE.json north_star): ψ, schedules (history-index selection) and the
stencil bit-exact; fields within max|Δ|/max|ref| ≤ 1e-10 (the reduction order
differs: FMA, split partial sums).  Runs through the public API and the C ABI.
"""

import hashlib
import math
import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-10  # normwise relative, BASELINE.json north_star


def normwise(got, want):
    want = np.asarray(want)
    scale = float(np.abs(want).max())
    diff = float(np.abs(np.asarray(got) - want).max())
    return diff / scale if scale > 0 else diff


@pytest.fixture(scope="module")
def fg(cuda_device):
    import paper_1004_5128_b200 as fg

    return fg


# ------------------------------------------------------------------------- ψ --

@pytest.mark.parametrize("gamma", [0.1, 0.3, 0.35, 0.5, 0.6, 0.7, 0.75, 0.8, 0.9, 1.0, 1.5, 1.99])
def test_device_psi_bitwise(fg, golden, gamma):
    t = fg.build_table(gamma, 10000).values.cpu().numpy()
    assert np.array_equal(t[:65], golden[f"psi_{gamma}_64"])
    assert hashlib.sha256(t.astype("<f8").tobytes()).hexdigest() == golden.meta["psi"][str(gamma)]


def test_device_psi_batched_and_frozen(fg):
    from oracle import fg_oracle as fo

    gam = np.random.default_rng(4).uniform(0.3, 0.9, size=300)
    tabs = fg.build_tables(gam, 2000).cpu().numpy()
    for b in (0, 17, 299):
        assert np.array_equal(tabs[b], fo.build_table(gam[b], 2000))
    assert [fg.psi(0.5, m) for m in range(4)] == [1.0, -0.5, -0.125, -0.0625]
    assert fg.psi(1.0, 7) == 0.0


# ----------------------------------------------------------------- schedules --

def _device_hash(fg, kind, kmax, base=0, horizon=0, chunk=1000):
    from paper_1004_5128_b200.schedule import device_schedules

    h = hashlib.sha256()
    for k0 in range(0, kmax + 1, chunk):
        nk = min(chunk, kmax + 1 - k0)
        offs, wts, lens = device_schedules(kind, k0, nk, base=base, horizon=horizon)
        offs, wts, lens = offs.cpu().numpy(), wts.cpu().numpy(), lens.cpu().numpy()
        for i in range(nk):
            n = int(lens[i])
            h.update(np.int64(n).astype("<i8").tobytes())
            h.update(offs[i, :n].astype("<i8").tobytes())
            h.update(wts[i, :n].astype("<i8").tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("base", ["2", "3", "4", "5", "8", "12", "20", "40", "100", "1500"])
def test_device_adaptive_schedule_every_k(fg, golden, base):
    """History-index selection bit-exact for every k in 0..10000 (schedule.py:97-151)."""
    assert _device_hash(fg, "adaptive", 10000, base=int(base)) == golden.meta["sched_hash"][base]


def test_device_full_and_short_schedules(fg, golden):
    assert _device_hash(fg, "full", 2000) == golden.meta["sched_hash"]["full"]
    for key, digest in golden.meta["short_hash"].items():
        L, dt = map(float, key.split("/"))
        assert _device_hash(fg, "short", 3000, horizon=int(math.floor(L / dt))) == digest, key


def test_schedule_pairs_and_strategies(fg, golden):
    for key, pairs in golden.meta["sched_pairs"].items():
        a, k = map(int, key.split("/"))
        assert fg.adaptive_schedule(k, a).pairs() == [tuple(p) for p in pairs]
    assert fg.ShortMemory(4.0).schedule_at(20, 0.5).pairs() == fg.full_schedule(8).pairs()
    assert len(fg.short_schedule(1499, 10.5, 1.0)) == 11


# ------------------------------------------------------------------- stencil --

@pytest.mark.parametrize("shape", [(7,), (101,), (9, 9), (6, 7), (33, 70), (5, 6, 7), (14, 14, 14)])
def test_device_stencil_bitwise(fg, shape):
    from oracle import fg_oracle as fo

    rng = np.random.default_rng(len(shape) * 100 + shape[0])
    u = np.zeros(shape)
    inner = tuple(slice(1, -1) for _ in shape)
    u[inner] = rng.normal(size=tuple(s - 2 for s in shape))
    assert np.array_equal(fg.stencil(u), fo.stencil(u))


def test_stencil_known_answer(fg):
    d = np.zeros((5, 5))
    d[2, 2] = 10.0
    out = fg.stencil(d)
    assert out[2, 2] == -40.0 and out[1, 2] == 10.0 and out[1, 1] == 0.0


# --------------------------------------------------------------- history_sum --

def test_history_sum_matches_golden(fg, golden):
    import torch

    for fields_key, k, gamma, cases in (
        ("hs_fields", 30, 0.6, {"full": fg.full_schedule(30), "adaptive3": fg.adaptive_schedule(30, 3),
                                "short7": fg.short_schedule(30, 7.0, 1.0)}),
        ("hs2_fields", 700, 0.8, {"full": fg.full_schedule(700), "adaptive5": fg.adaptive_schedule(700, 5),
                                  "adaptive2": fg.adaptive_schedule(700, 2)}),
    ):
        fields = golden[fields_key]
        buf = fg.HistoryBuffer(k + 1, fields.shape[1:], byte_cap=None)
        for f in fields:
            buf.append(f)
        table = fg.build_table(gamma, k)
        prefix = "hs_out_" if fields_key == "hs_fields" else "hs2_out_"
        for name, sched in cases.items():
            got = fg.history_sum(buf, sched, table, k).cpu().numpy()
            np.testing.assert_allclose(got, golden[prefix + name], rtol=1e-12, atol=1e-14)
    # validation mirrors solver.py:177-189
    buf = fg.HistoryBuffer(4, (3, 3))
    for _ in range(3):
        buf.append(np.zeros((3, 3)))
    with pytest.raises(ValueError, match="beyond"):
        fg.history_sum(buf, fg.full_schedule(5), fg.build_table(0.5, 10), 2)
    with pytest.raises(ValueError, match="history"):
        fg.history_sum(buf, fg.full_schedule(2), fg.build_table(0.5, 10), 3)
    with pytest.raises(ValueError, match="table covers"):
        fg.history_sum(buf, fg.full_schedule(2), fg.build_table(0.5, 1), 2)
    assert torch.cuda.is_available()


# ------------------------------------------------------------- run (2D API) --

RUN_CASES = ["small", "small_decay", "ftcs_g1", "point_full", "point_short100", "point_adaptive3",
             "point_adaptive5", "point_g05_adaptive1500", "spread_g09_adaptive4", "c2_small", "c2_small_full",
             "c2_small_short"]


def _config_from_golden(fg, golden, name):
    c = golden.case(name)
    kind, param = c["strategy"]
    strat = {"full": lambda: fg.FullMemory(), "short": lambda: fg.ShortMemory(param),
             "adaptive": lambda: fg.AdaptiveMemory(int(param))}[kind]()
    if c["sources"] is not None:
        sources = tuple((int(j), int(l), float(v)) for j, l, v in c["sources"])
    else:
        u0 = golden.initial_field(name)[0]
        sources = tuple((int(j), int(l), float(u0[j, l])) for j, l in zip(*np.nonzero(u0)))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return fg.SimulationConfig(gamma=c["gamma"], alpha=c["alpha"], beta=c["beta"], dt=c["dt"], dx=c["dx"],
                                   nx=c["nx"], ny=c["ny"], n_steps=c["n_steps"], sources=sources, strategy=strat,
                                   snapshot_every=c["snapshot_every"])


@pytest.mark.parametrize("name", RUN_CASES)
def test_run_matches_reference_goldens(fg, golden, name):
    cfg = _config_from_golden(fg, golden, name)
    res = fg.run(cfg)
    steps, snaps = golden.expected(name)
    assert [s for s, _ in res.snapshots] == steps.tolist()
    for (s, g), want in zip(res.snapshots, snaps):
        err = normwise(g.data, want[0])
        assert err <= TOL, f"{name} step {s}: normwise rel err {err:.3e}"
    assert res.final is res.snapshots[-1][1]
    assert res.elapsed_seconds >= 0.0 and res.config is cfg


def test_first_step_exact_and_decay_exact(fg):
    # tests/test_solver.py:112-128,168-175: exact to the last bit
    base = dict(gamma=0.5, alpha=1.0, beta=0.0, dt=1.0, dx=10.0, nx=8, ny=8, n_steps=1, sources=((4, 4, 10.0),))
    cfg = fg.SimulationConfig(**base)
    u0 = cfg.initial_grid().data
    from oracle import fg_oracle as fo

    expected = u0 + 1.0 * 1.0**0.5 / 10.0**2 * fo.stencil(u0)
    assert np.array_equal(fg.run(cfg).final.data, expected)
    cfg = fg.SimulationConfig(**{**base, "alpha": 0.0, "beta": 0.07, "dt": 0.5, "n_steps": 30, "snapshot_every": 1})
    value, factor = 10.0, 1.0 - 0.07 * 0.5
    for _, grid in fg.run(cfg).snapshots:
        want = np.zeros((8, 8))
        want[4, 4] = value
        assert np.array_equal(grid.data, want)
        value = value * factor


@pytest.mark.parametrize("strategy", ["short40", "adaptive40", "adaptive1500"])
def test_covering_strategies_reproduce_full_bitwise(fg, strategy):
    from dataclasses import replace

    strat = {"short40": fg.ShortMemory(40.0), "adaptive40": fg.AdaptiveMemory(40),
             "adaptive1500": fg.AdaptiveMemory(1500)}[strategy]
    base = fg.SimulationConfig(gamma=0.5, alpha=1.0, beta=0.0, dt=1.0, dx=10.0, nx=8, ny=8, n_steps=40,
                               sources=((4, 4, 10.0),))
    assert np.array_equal(fg.run(base).final.data, fg.run(replace(base, strategy=strat)).final.data)


def test_divergence_reported(fg, golden):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        cfg = fg.SimulationConfig(gamma=1.0, alpha=1.0, beta=0.0, dt=1.0, dx=1.0, nx=8, ny=8, n_steps=500,
                                  sources=((4, 4, 10.0),))
    with pytest.raises(fg.DivergenceError, match="step") as exc:
        fg.run(cfg)
    want = golden.meta["divergence"]
    assert exc.value.step == want["step"]
    assert exc.value.peak == pytest.approx(want["peak"], rel=1e-10)


def test_memory_budget_enforced(fg):
    cfg = fg.SimulationConfig(gamma=0.5, alpha=1.0, beta=0.0, dt=1.0, dx=10.0, nx=8, ny=8, n_steps=10_000,
                              sources=((4, 4, 10.0),), history_byte_cap=100_000)
    with pytest.raises(fg.MemoryBudgetError):
        fg.run(cfg)


def test_device_memory_checked_before_allocation(fg):
    """A history larger than the device (1024² x 30000 steps = 252 GB, no byte
    cap) is refused with MemoryBudgetError before anything is allocated."""
    u0 = np.zeros((1024, 1024))
    cfg = fg.FieldConfig(initial=u0, dx=1.0, gamma=0.5, dt=1.0, n_steps=30_000, history_byte_cap=None)
    with pytest.raises(fg.MemoryBudgetError, match="free"):
        fg.run_field(cfg)


def test_progress_logging(fg, caplog):
    import logging

    cfg = fg.SimulationConfig(gamma=0.5, alpha=1.0, beta=0.0, dt=1.0, dx=10.0, nx=8, ny=8, n_steps=10,
                              sources=((4, 4, 10.0),))
    with caplog.at_level(logging.INFO, logger="fracgrid"):
        fg.run(cfg, progress_every=5)
    msgs = [r.getMessage() for r in caplog.records]
    assert "step 5/10" in msgs and "step 10/10" in msgs


def test_step_api_matches_oracle(fg):
    """solver.step on the device: same history contract, m = 0 term read from H[k]."""
    from oracle import fg_oracle as fo

    cfg = fg.SimulationConfig(gamma=0.6, alpha=1.0, beta=0.05, dt=1.0, dx=10.0, nx=9, ny=11, n_steps=40,
                              sources=((4, 5, 10.0), (3, 3, 2.0)), strategy=fg.AdaptiveMemory(3))
    table = fg.build_table(cfg.gamma, cfg.n_steps)
    hist = fg.HistoryBuffer(cfg.n_steps + 1, (9, 11))
    u = cfg.initial_grid().data.copy()
    hist.append(fg.stencil(u))
    for k in range(cfg.n_steps):
        u = fg.step(u, hist, k, cfg, table)
    assert len(hist) == cfg.n_steps + 1
    ref = fo.run(fo.OracleProblem(u0=cfg.initial_grid().data[None], gamma=np.array([0.6]), dt=np.array([1.0]),
                                  alpha=1.0, dx=10.0, reaction=("linear", 0.05), strategy=("adaptive", 3),
                                  n_steps=cfg.n_steps))
    assert normwise(u, ref["final"][0]) <= TOL


def test_reference_config_duck_typed(fg):
    """run() accepts any config/strategy with the reference's attributes."""
    from dataclasses import dataclass

    @dataclass(frozen=True)
    class Strat:
        base: int
        tag = "adaptive"

    cfg = fg.SimulationConfig(gamma=0.75, alpha=1.0, beta=0.0, dt=1.0, dx=10.0, nx=20, ny=20, n_steps=50,
                              sources=((10, 10, 10.0),), strategy=fg.AdaptiveMemory(3))
    from dataclasses import replace

    a = fg.run(cfg).final.data
    b = fg.run(replace(cfg, strategy=Strat(3))).final.data
    assert np.array_equal(a, b)


# ------------------------------------------------------------- n-D / batched --

ND_CASES = ["c1", "1d_adaptive", "3d_sat_full", "3d_sat_adaptive", "batch_adaptive", "batch_short"]


def _field_config_from_golden(fg, golden, name):
    p = golden.problem_params(name)
    kind, param = p["strategy"]
    strat = {"full": lambda: fg.FullMemory(), "short": lambda: fg.ShortMemory(param),
             "adaptive": lambda: fg.AdaptiveMemory(int(param))}[kind]()
    react = fg.LinearDecay(p["reaction"][1]) if p["reaction"][0] == "linear" else fg.Saturating(*p["reaction"][1:])
    return fg.FieldConfig(initial=p["u0"], dx=p["dx"], gamma=p["gamma"], dt=p["dt"], n_steps=p["n_steps"],
                          alpha=p["alpha"], reaction=react, strategy=strat, batched=True,
                          snapshot_every=p["snapshot_every"], history_byte_cap=None)


@pytest.mark.parametrize("name", ND_CASES)
@pytest.mark.parametrize("split", [0, 1, 8])
def test_run_field_matches_goldens(fg, golden, name, split):
    cfg = _field_config_from_golden(fg, golden, name)
    res = fg.run_field(cfg, split=split)
    steps, snaps = golden.expected(name)
    assert [s for s, _ in res.snapshots] == steps.tolist()
    for (s, got), want in zip(res.snapshots, snaps):
        for b in range(want.shape[0]):
            err = normwise(got[b], want[b])
            assert err <= TOL, f"{name} member {b} step {s}: {err:.3e}"


@pytest.mark.parametrize("flags", [0, 1, 2, 3, 4, 6])
@pytest.mark.parametrize("name", ["batch_adaptive", "c2_small", "3d_sat_adaptive"])
def test_launch_modes_bitwise_identical(fg, golden, flags, name):
    """Per-step launches, CUDA graph, PDL, graph+PDL and the persistent
    cooperative kernel give identical bits (same arithmetic in every mode)."""
    if golden.case(name)["kind"] == "nd":
        cfg = _field_config_from_golden(fg, golden, name)
    else:
        p = golden.problem_params(name)
        cfg = fg.FieldConfig(initial=p["u0"][0], dx=p["dx"], gamma=float(p["gamma"][0]), dt=float(p["dt"][0]),
                             n_steps=p["n_steps"], reaction=fg.LinearDecay(p["reaction"][1]),
                             strategy=fg.AdaptiveMemory(int(p["strategy"][1])), snapshot_every=p["snapshot_every"])
    ref = fg.run_field(cfg, flags=0, tblock=0)
    got = fg.run_field(cfg, flags=flags, tblock=0)
    for (s0, a0), (s1, a1) in zip(ref.snapshots, got.snapshots):
        assert s0 == s1 and np.array_equal(a0, a1)


def test_persistent_multi_pass_ensemble(fg):
    """More tiles than resident CTAs: the persistent kernel loops over tiles
    (passes > 1); bitwise equal to per-step launches, members match the oracle."""
    from oracle import fg_oracle as fo

    rng = np.random.default_rng(9)
    B, n, steps = 3000, 64, 120
    x = np.arange(n) / (n - 1)
    centres = rng.uniform(0.3, 0.7, size=B)
    u0 = np.exp(-((x[None, :] - centres[:, None]) ** 2) / (2 * 0.05**2))
    u0[:, 0] = u0[:, -1] = 0.0
    gam = rng.uniform(0.3, 0.9, size=B)
    dts = (0.2 * (1 / (n - 1)) ** 2) ** (1 / gam)
    cfg = fg.FieldConfig(initial=u0, dx=1 / (n - 1), gamma=gam, dt=dts, n_steps=steps,
                         strategy=fg.AdaptiveMemory(4), batched=True, snapshot_every=40)
    pers = fg.run_field(cfg, flags=4, tblock=0)
    plain = fg.run_field(cfg, flags=0, tblock=0)
    for (_, a), (_, b) in zip(pers.snapshots, plain.snapshots):
        assert np.array_equal(a, b)
    # with temporal blocking: one cooperative launch per block == per-step PDL launches
    pers_b = fg.run_field(cfg, flags=4, tblock=16)
    pdl_b = fg.run_field(cfg, flags=2, tblock=16)
    for (_, a), (_, b) in zip(pers_b.snapshots, pdl_b.snapshots):
        assert np.array_equal(a, b)
    idx = [0, 1, 1499, 2999]
    ref = fo.run(fo.OracleProblem(u0=u0[idx], gamma=gam[idx], dt=dts[idx], alpha=1.0, dx=1 / (n - 1),
                                  reaction=("linear", 0.0), strategy=("adaptive", 4), n_steps=steps,
                                  snapshot_every=40))
    for (_, got), (_, want) in zip(pers.snapshots, ref["snapshots"]):
        for i, b in enumerate(idx):
            assert normwise(got[b], want[i]) <= TOL


def test_progress_chunks_bitwise(fg, golden):
    """progress_every splits the loop into several launches; results unchanged."""
    cfg = _field_config_from_golden(fg, golden, "3d_sat_full")
    a = fg.run_field(cfg).final
    b = fg.run_field(cfg, progress_every=37).final
    assert np.array_equal(a, b)


def test_divergence_all_modes(fg, golden):
    u0 = np.zeros((8, 8))
    u0[4, 4] = 10.0
    cfg = fg.FieldConfig(initial=u0, dx=1.0, gamma=1.0, dt=1.0, n_steps=500)
    want = golden.meta["divergence"]
    for flags in (0, 2, 4):
        with pytest.raises(fg.DivergenceError) as exc:
            fg.run_field(cfg, flags=flags)
        assert exc.value.step == want["step"]
        assert exc.value.peak == pytest.approx(want["peak"], rel=1e-10)


# ------------------------------------------------------------ temporal blocking --

def _any_field_config(fg, golden, name):
    if golden.case(name)["kind"] == "nd":
        return _field_config_from_golden(fg, golden, name)
    p = golden.problem_params(name)
    kind, param = p["strategy"]
    strat = {"full": lambda: fg.FullMemory(), "short": lambda: fg.ShortMemory(param),
             "adaptive": lambda: fg.AdaptiveMemory(int(param))}[kind]()
    return fg.FieldConfig(initial=p["u0"][0], dx=p["dx"], gamma=float(p["gamma"][0]), dt=float(p["dt"][0]),
                          n_steps=p["n_steps"], alpha=p["alpha"], reaction=fg.LinearDecay(p["reaction"][1]),
                          strategy=strat, snapshot_every=p["snapshot_every"], history_byte_cap=None)


BLOCK_CASES = ["small", "point_full", "point_short100", "point_adaptive3", "point_adaptive5", "c2_small",
               "c2_small_full", "c2_small_short", "spread_g09_adaptive4"] + ND_CASES


@pytest.mark.parametrize("tblock", [8, 16, 24, 32])
@pytest.mark.parametrize("name", BLOCK_CASES)
def test_temporal_blocking_matches_goldens(fg, golden, name, tblock):
    """One history pass feeding `tblock` steps reproduces the reference (≤1e-10)."""
    cfg = _any_field_config(fg, golden, name)
    res = fg.run_field(cfg, tblock=tblock)
    steps, snaps = golden.expected(name)
    assert [s for s, _ in res.snapshots] == steps.tolist()
    batched = golden.case(name)["kind"] == "nd"
    for (s, got), want in zip(res.snapshots, snaps):
        g = got if batched else got[None]
        for b in range(want.shape[0]):
            err = normwise(g[b], want[b])
            assert err <= TOL, f"{name} tblock {tblock} member {b} step {s}: {err:.3e}"


ADAPTIVE_WIDE = ["point_adaptive3", "point_adaptive5", "c2_small", "spread_g09_adaptive4", "point_g05_adaptive1500",
                 "batch_adaptive", "1d_adaptive", "3d_sat_adaptive"]


@pytest.mark.parametrize("tblock", [48, 56, 64, 96, 112, 128])
@pytest.mark.parametrize("name", ADAPTIVE_WIDE)
def test_wide_temporal_blocking_matches_goldens(fg, golden, name, tblock):
    """Factors above 32 (itemized main and tail launches; adaptive, single
    member and ensembles with per-member ψ)."""
    test_temporal_blocking_matches_goldens(fg, golden, name, tblock)


@pytest.mark.parametrize("cols", ["8", "16"])
@pytest.mark.parametrize("name", ["c2_small", "point_adaptive3", "batch_adaptive", "3d_sat_adaptive"])
def test_item_widths_match_goldens(fg, golden, name, cols, monkeypatch):
    """Both item widths (8-column items on wide tiles, 16-column items on
    narrow tiles) for single fields and ensembles, at tblock 32 and 128."""
    monkeypatch.setenv("FGB200_ITEM_COLS", cols)
    for tb in (32, 128):
        test_temporal_blocking_matches_goldens(fg, golden, name, tb)


@pytest.mark.parametrize("sub,tb,cols,delay", [("8", 64, None, None), ("16", 128, None, None), ("32", 128, None, None),
                                               ("8", 32, None, None), ("4", 24, None, None), ("28", 112, "16", None),
                                               ("32", 128, "16", None), ("28", 112, "16", "28"), ("28", 112, "16", "1"),
                                               ("8", 32, None, "8"), ("8", 32, None, "1")])
@pytest.mark.parametrize("name", ["c2_small", "point_adaptive5", "batch_adaptive", "3d_sat_adaptive",
                                  "spread_g09_adaptive4", "c2_small_full", "c2_small_short", "point_full",
                                  "point_short100"])
def test_subblock_launches_match_goldens(fg, golden, name, sub, tb, cols, delay, monkeypatch):
    """Sub-block launches (finished sub-blocks streamed into the later steps'
    partial sums on a third stream) reproduce the reference (<= 1e-10); (28,
    112, 16-column items, delay 7) is the default of single large adaptive fields
    (c3, c4); delays 1 and S bracket the default S/4."""
    monkeypatch.setenv("FGB200_SUBBLOCK", sub)
    if delay:
        monkeypatch.setenv("FGB200_SUBDELAY", delay)
    if cols:
        monkeypatch.setenv("FGB200_ITEM_COLS", cols)
    dense = name.endswith("full") or "short" in name
    if dense and tb > 32:
        pytest.skip("factors above 32 are adaptive only")
    test_temporal_blocking_matches_goldens(fg, golden, name, tb)


@pytest.mark.parametrize("name", ["c2_small", "batch_adaptive", "c2_small_full", "c2_small_short"])
def test_subblock_launch_modes_bitwise(fg, golden, name, monkeypatch):
    """With sub-blocks: launch modes, graph capture and split runs are bitwise equal."""
    monkeypatch.setenv("FGB200_SUBBLOCK", "8")
    cfg = _any_field_config(fg, golden, name)
    tb = 32 if name.endswith(("_full", "_short")) else 64
    ref = fg.run_field(cfg, flags=0, tblock=tb)
    for kw in (dict(flags=2), dict(flags=3), dict(flags=1), dict(progress_every=7), dict(progress_every=29),
               dict(flags=2, overlap="0")):
        kw = dict(kw)
        monkeypatch.setenv("FGB200_BLOCK_OVERLAP", kw.pop("overlap", "1"))
        got = fg.run_field(cfg, tblock=tb, **kw)
        for (s0, a0), (s1, a1) in zip(ref.snapshots, got.snapshots):
            assert s0 == s1 and np.array_equal(a0, a1), kw


PAIR_CASES = ["c2_small", "small", "point_full", "point_adaptive3", "point_adaptive5", "c1", "1d_adaptive",
              "batch_adaptive", "spread_g09_adaptive4", "c2_small_full"]


@pytest.mark.parametrize("tblock", [16, 32, 64])
@pytest.mark.parametrize("name", PAIR_CASES)
def test_fused_pairs_bitwise(fg, golden, name, tblock, monkeypatch):
    kind = golden.case(name).get("strategy", [None])[0] if golden.case(name)["kind"] != "nd" else None
    if tblock > 32 and (kind in ("full", "short") or name in ("c1", "c2_small_full", "small", "point_full")):
        pytest.skip("factors above 32 are adaptive only")
    """Fused step pairs (two steps per launch, halo recomputed) equal single-step
    launches bit for bit, snapshots included; and match the reference."""
    cfg = _any_field_config(fg, golden, name)
    monkeypatch.setenv("FGB200_PAIRS", "0")
    ref = fg.run_field(cfg, tblock=tblock)
    monkeypatch.setenv("FGB200_PAIRS", "1")
    for kw in (dict(), dict(flags=0), dict(progress_every=7), dict(flags=3)):
        got = fg.run_field(cfg, tblock=tblock, **kw)
        assert len(got.snapshots) == len(ref.snapshots)
        for (s0, a0), (s1, a1) in zip(ref.snapshots, got.snapshots):
            assert s0 == s1 and np.array_equal(a0, a1), (kw, s0)
    test_temporal_blocking_matches_goldens(fg, golden, name, tblock)


def test_fused_pairs_divergence(fg, golden, monkeypatch):
    """A run that blows up reports the same first bad step and peak with and
    without fused pairs (the bad field may sit in the pairs' scratch buffer)."""
    u0 = np.zeros((8, 8))
    u0[4, 4] = 10.0
    results = set()
    for n_steps in (500, 37, 38):
        cfg = fg.FieldConfig(initial=u0, dx=1.0, gamma=1.0, dt=1.0, n_steps=n_steps)
        for pairs in ("0", "1"):
            monkeypatch.setenv("FGB200_PAIRS", pairs)
            for tb in (16, 32):
                try:
                    fg.run_field(cfg, tblock=tb)
                except fg.DivergenceError as exc:
                    results.add((n_steps, exc.step, exc.peak))
                else:
                    results.add((n_steps, None, None))
    by_n = {}
    for n_steps, step, peak in results:
        by_n.setdefault(n_steps, set()).add((step, peak))
    assert all(len(v) == 1 for v in by_n.values()), by_n
    assert next(iter(by_n[500]))[0] == golden.meta["divergence"]["step"]


def test_cached_graph_replay(fg, golden):
    """FG_RUN_GRAPH: the second identical run replays the cached graph and
    gives the per-step launches' bits; a different plan is re-captured."""
    import torch

    from paper_1004_5128_b200._engine import Stepper

    outs = []
    for name in ("c2_small", "point_adaptive5", "c2_small"):
        cfg = _any_field_config(fg, golden, name)
        ref = fg.run_field(cfg, flags=2, tblock=64).final
        st = Stepper(cfg.to_problem(), flags=3, tblock=64, snapshots=False)
        u0 = st.u[0].clone()
        for _ in range(3):
            st.reset(u0)
            st.advance(cfg.n_steps)
            torch.cuda.synchronize()
            got = st.u[cfg.n_steps & 1][: st.n_m].cpu().numpy().reshape(np.asarray(ref).shape)
            assert np.array_equal(got, ref), name
        outs.append(got)
    assert np.array_equal(outs[0], outs[2])


def test_wide_temporal_blocking_rejects_dense_plans(fg, golden):
    cfg = _any_field_config(fg, golden, "point_full")
    with pytest.raises(ValueError, match="tblock 64"):
        fg.run_field(cfg, tblock=64)


@pytest.mark.parametrize("name", ["c2_small", "batch_short", "3d_sat_full"])
def test_temporal_blocking_modes_bitwise(fg, golden, name, monkeypatch):
    """Blocked runs are identical across launch modes (side-stream pipeline on
    and off, persistent), across runs split into several launches (partial sums
    continued or recomputed), and reruns."""
    cfg = _any_field_config(fg, golden, name)
    ref = fg.run_field(cfg, flags=0, tblock=16)
    for kw in (dict(flags=1), dict(flags=2), dict(flags=3), dict(flags=4), dict(progress_every=7),
               dict(progress_every=16), dict(flags=2, overlap="0"), dict(flags=1, overlap="0"),
               dict(flags=3, overlap="0"), dict(flags=2, progress_every=7)):
        kw = dict(kw)
        monkeypatch.setenv("FGB200_BLOCK_OVERLAP", kw.pop("overlap", "1"))
        got = fg.run_field(cfg, tblock=16, **kw)
        assert len(got.snapshots) == len(ref.snapshots)
        for (s0, a0), (s1, a1) in zip(ref.snapshots, got.snapshots):
            assert s0 == s1 and np.array_equal(a0, a1), kw


@pytest.mark.parametrize("flags", [1, 2, 4])
def test_temporal_blocking_divergence(fg, golden, flags):
    u0 = np.zeros((8, 8))
    u0[4, 4] = 10.0
    cfg = fg.FieldConfig(initial=u0, dx=1.0, gamma=1.0, dt=1.0, n_steps=500)
    with pytest.raises(fg.DivergenceError) as exc:
        fg.run_field(cfg, tblock=16, flags=flags)
    assert exc.value.step == golden.meta["divergence"]["step"]


def test_graph_replay_after_a_larger_plan(fg, monkeypatch):
    """A cached run graph replays its own plan's buffers: graph run A, a run of
    a larger 1D field (fused pairs, their scratch owned by that plan), then
    graph run A again gives A's results bitwise (the pair scratch is part of
    the plan, so a graph never captures another run's buffers)."""
    monkeypatch.setenv("FGB200_PAIRS", "1")

    def cfg_of(n):
        x = np.linspace(0.0, 1.0, n)
        u0 = np.exp(-((x - 0.4) ** 2) / 0.01)
        u0[0] = u0[-1] = 0.0
        return fg.FieldConfig(initial=u0, dx=x[1], gamma=0.6, dt=(0.2 * x[1] ** 2) ** (1 / 0.6), n_steps=300,
                              strategy=fg.AdaptiveMemory(4), snapshot_every=50, history_byte_cap=None)

    a, big = cfg_of(700), cfg_of(5000)
    ref = fg.run_field(a, flags=2, tblock=32)
    first = fg.run_field(a, flags=1, tblock=32)
    fg.run_field(big, flags=1, tblock=32)
    again = fg.run_field(a, flags=1, tblock=32)
    for res in (first, again):
        for (s0, a0), (s1, a1) in zip(ref.snapshots, res.snapshots):
            assert s0 == s1 and np.array_equal(a0, a1), s0
