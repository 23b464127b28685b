"""The temporal-blocking kernel alone (fg_block_partials): partial sums over
history slices t < kb0 for a block of steps, against a NumPy restatement, on
random histories; TMA bulk-copy geometry (TP 128 / 256), chunk boundaries,
partial last stages and reruns (determinism)."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def expected_partials(H, kind, param, kb0, bt, table, dt=1.0):
    from oracle import fg_oracle as fo

    N = H.shape[1]
    P = np.zeros((bt, N))
    for b in range(bt):
        offs, wts = fo.schedule(kind, kb0 + b, param, dt)
        for m, w in zip(offs, wts):
            t = kb0 + b - m
            if t < kb0:
                P[b] += (w * table[m]) * H[t]
    return P


@pytest.mark.parametrize("shape,kind,param", [
    ((256, 256), "adaptive", 5), ((256, 256), "full", 0), ((48, 48), "adaptive", 3), ((4096,), "full", 0),
    ((300,), "adaptive", 2), ((64, 64), "short", 37.0)])
@pytest.mark.parametrize("kb0,bt", [(16, 16), (160, 16), (1030, 16), (2000, 7), (517, 8), (48, 24), (1200, 24),
                                    (999, 32), (64, 64), (1280, 64), (1000, 48), (1920, 96), (2048, 128)])
def test_block_partials_match_numpy(cuda_device, shape, kind, param, kb0, bt):
    import torch

    import paper_1004_5128_b200 as fg
    from paper_1004_5128_b200 import _lib
    from paper_1004_5128_b200._engine import Stepper

    tblock = {8: 8, 24: 24, 32: 32, 48: 48, 64: 64, 96: 96, 128: 128}.get(bt, 16)
    if tblock > 32 and kind != "adaptive":
        pytest.skip("factors above 32 are adaptive only")
    n_steps = kb0 + bt + 1
    u0 = np.zeros(shape)
    strat = {"full": lambda: fg.FullMemory(), "short": lambda: fg.ShortMemory(param),
             "adaptive": lambda: fg.AdaptiveMemory(param)}[kind]()
    cfg = fg.FieldConfig(initial=u0, dx=1.0, gamma=0.63, dt=1.0, n_steps=n_steps, strategy=strat,
                         history_byte_cap=None)
    st = Stepper(cfg.to_problem(), tblock=tblock)
    gen = torch.Generator(device=st.device).manual_seed(kb0 * 7 + bt)
    st.H.copy_(torch.randn(st.H.shape, generator=gen, device=st.device, dtype=torch.float64))
    L = _lib.load()
    _lib.check(L.fg_block_partials(C.byref(st.plan), kb0, bt, _lib.stream_handle()))
    torch.cuda.synchronize()
    P1 = st.block_partials(kb0)[:bt].clone()
    for rep in range(5):
        _lib.check(L.fg_block_partials(C.byref(st.plan), kb0, bt, _lib.stream_handle()))
        torch.cuda.synchronize()
        bad = (P1 != st.block_partials(kb0)[:bt]).nonzero()
        assert bad.numel() == 0, f"rerun {rep} differs at {bad.shape[0]} places, first {bad[:8].tolist()}"
    n = int(np.prod(shape))
    H = st.H[:kb0, :n].cpu().numpy()
    table = st.psi[0].cpu().numpy()
    want = expected_partials(H, kind, param, kb0, bt, table)
    got = P1[:, :n].cpu().numpy()
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= 1e-12 * max(scale, 1.0)


@pytest.mark.parametrize("kind,param", [("full", 0), ("short", 300.0)])
@pytest.mark.parametrize("kb0,bt", [(999, 32), (130, 32), (64, 32), (96, 32), (700, 17)])
def test_solo_main_launch_matches_numpy(cuda_device, kind, param, kb0, bt):
    """Large single fields at tblock 32 take the solo dense main launch (one CTA
    per SM, software-pipelined fragments, 4-stage ring): ragged last tile (801
    tiles of 256 points, several per CTA), fewer stages than the ring, partial
    last stages and a short last block, against NumPy; reruns bitwise equal."""
    import torch

    import paper_1004_5128_b200 as fg
    from paper_1004_5128_b200 import _lib
    from paper_1004_5128_b200._engine import Stepper

    shape = (401, 511)
    n = int(np.prod(shape))
    assert -(-n // 256) >= 4 * 148  # the library's solo threshold on a B200
    strat = fg.FullMemory() if kind == "full" else fg.ShortMemory(param)
    cfg = fg.FieldConfig(initial=np.zeros(shape), dx=1.0, gamma=0.63, dt=1.0, n_steps=kb0 + bt + 1, strategy=strat,
                         history_byte_cap=None)
    st = Stepper(cfg.to_problem(), tblock=32)
    gen = torch.Generator(device=st.device).manual_seed(kb0 + bt)
    st.H.copy_(torch.randn(st.H.shape, generator=gen, device=st.device, dtype=torch.float64))
    L = _lib.load()
    _lib.check(L.fg_block_partials(C.byref(st.plan), kb0, bt, _lib.stream_handle()))
    torch.cuda.synchronize()
    P1 = st.block_partials(kb0)[:bt].clone()
    for rep in range(3):
        _lib.check(L.fg_block_partials(C.byref(st.plan), kb0, bt, _lib.stream_handle()))
        torch.cuda.synchronize()
        assert torch.equal(P1, st.block_partials(kb0)[:bt]), f"rerun {rep} differs"
    H = st.H[:kb0, :n].cpu().numpy()
    want = expected_partials(H, kind, param, kb0, bt, st.psi[0].cpu().numpy())
    got = P1[:, :n].cpu().numpy()
    assert np.abs(got - want).max() <= 1e-12 * max(np.abs(want).max(), 1.0)


@pytest.mark.parametrize("n_pts,B", [(300, 5), (512, 3), (40, 9)])
@pytest.mark.parametrize("kb0,bt", [(16, 16), (160, 16), (1032, 24), (992, 32), (1008, 48), (1280, 64), (2000, 7), (1920, 128)])
def test_ensemble_block_partials_match_numpy(cuda_device, n_pts, B, kb0, bt):
    """Itemized ensembles: the adaptive schedule is shared, each member has its
    own ψ table (own γ) and its own coefficient rows; member rows are padded
    (ms > n_m for 300 and 40 points)."""
    import torch

    import paper_1004_5128_b200 as fg
    from paper_1004_5128_b200 import _lib
    from paper_1004_5128_b200._engine import Stepper

    tblock = {8: 8, 24: 24, 32: 32, 48: 48, 64: 64, 96: 96, 128: 128}.get(bt, 16)
    n_steps = kb0 + bt + 1
    gam = np.linspace(0.31, 0.89, B)
    cfg = fg.FieldConfig(initial=np.zeros((B, n_pts)), dx=1.0, gamma=gam.tolist(), dt=[1.0] * B,
                         n_steps=n_steps, strategy=fg.AdaptiveMemory(5), batched=True, history_byte_cap=None)
    st = Stepper(cfg.to_problem(), tblock=tblock)
    assert st.plan.blkcoef_dev, "ensemble adaptive plans carry per-member item coefficient rows"
    gen = torch.Generator(device=st.device).manual_seed(kb0 * 3 + bt)
    st.H.copy_(torch.randn(st.H.shape, generator=gen, device=st.device, dtype=torch.float64))
    L = _lib.load()
    _lib.check(L.fg_block_partials(C.byref(st.plan), kb0, bt, _lib.stream_handle()))
    torch.cuda.synchronize()
    P1 = st.block_partials(kb0)[:bt].clone()
    _lib.check(L.fg_block_partials(C.byref(st.plan), kb0, bt, _lib.stream_handle()))
    torch.cuda.synchronize()
    assert torch.equal(P1, st.block_partials(kb0)[:bt]), "rerun differs"
    ms = st.ms
    Hs = st.H[:kb0].cpu().numpy().reshape(kb0, B, ms)
    got = P1.cpu().numpy().reshape(bt, B, ms)
    for b in range(B):
        table = st.psi[b].cpu().numpy()
        want = expected_partials(Hs[:, b, :n_pts], "adaptive", 5, kb0, bt, table)
        scale = max(np.abs(want).max(), 1.0)
        assert np.abs(got[:, b, :n_pts] - want).max() <= 1e-12 * scale, f"member {b}"


def expected_sub_partials(H, param, kb0, bt, S, D, table):
    """Old part + what the sub-block launches add: launch i feeds the steps
    b >= (i+1)S + D with the slices [kb0 + iS, kb0 + (i+1)S) their schedules use."""
    from oracle import fg_oracle as fo

    P = expected_partials(H, "adaptive", param, kb0, bt, table)
    for b in range(bt):
        offs, wts = fo.schedule("adaptive", kb0 + b, param, 1.0)
        for m, w in zip(offs, wts):
            t = kb0 + b - m
            if t < kb0:
                continue
            i = (t - kb0) // S
            if (i + 1) * S + D <= b:
                P[b] += (w * table[m]) * H[t]
    return P


@pytest.mark.parametrize("shape", [(96, 96), (4100,)])
@pytest.mark.parametrize("kb0,tblock,S,D", [(224, 112, 28, 7), (1024, 128, 32, 8), (640, 64, 16, 16), (1120, 112, 28, 28)])
def test_subblock_partials_match_numpy(cuda_device, monkeypatch, shape, kb0, tblock, S, D):
    """fg_block_subpartials replays a block's sub-block launches over a resident
    history (bench.py's whole-stage replay): main + tail + sub-blocks against NumPy."""
    import torch

    import paper_1004_5128_b200 as fg
    from paper_1004_5128_b200 import _lib
    from paper_1004_5128_b200._engine import Stepper

    bt = tblock
    cfg = fg.FieldConfig(initial=np.zeros(shape), dx=1.0, gamma=0.58, dt=1.0, n_steps=kb0 + bt + 1,
                         strategy=fg.AdaptiveMemory(5), history_byte_cap=None)
    monkeypatch.setenv("FGB200_SUBBLOCK", str(S))
    monkeypatch.setenv("FGB200_SUBDELAY", str(D))
    st = Stepper(cfg.to_problem(), tblock=tblock)
    assert int(st.plan.subblock) == S and (int(st.plan.subdelay) or S) == D
    gen = torch.Generator(device=st.device).manual_seed(kb0 + S)
    st.H.copy_(torch.randn(st.H.shape, generator=gen, device=st.device, dtype=torch.float64))
    L = _lib.load()
    n_sub = C.c_int32(-1)
    for _ in range(2):  # rerun: the main launch overwrites P, so the result is the same
        _lib.check(L.fg_block_partials(C.byref(st.plan), kb0, bt, _lib.stream_handle()))
        _lib.check(L.fg_block_subpartials(C.byref(st.plan), kb0, bt, _lib.stream_handle(), C.byref(n_sub)))
    torch.cuda.synchronize()
    assert n_sub.value == len([i for i in range(bt // S) if (i + 1) * S + D < bt])
    n = int(np.prod(shape))
    H = st.H[: kb0 + bt, :n].cpu().numpy()
    want = expected_sub_partials(H, 5, kb0, bt, S, D, st.psi[0].cpu().numpy())
    got = st.block_partials(kb0)[:bt, :n].cpu().numpy()
    assert np.abs(got - want).max() <= 1e-12 * max(np.abs(want).max(), 1.0)
