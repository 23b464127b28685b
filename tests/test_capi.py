"""The C-ABI library loads and exports every symbol include/fgb200.h declares (CPU only).

No compute is launched: only host-side entry points (version, layout, schedule
lengths, argument validation) are called.
"""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1004_5128_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fgb200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fg_\w+)\s*\(", text)))


def test_library_exists_and_loads():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build() first"
    L = _lib.load()
    assert L.fg_abi_version() == _lib.ABI_VERSION == 7


def test_every_declared_symbol_is_exported():
    L = _lib.load()
    names = declared_functions()
    assert names, "no declarations parsed"
    assert set(names) == set(_lib.EXPORTS)
    for n in names:
        assert hasattr(L, n), n


def test_plan_layout_matches_binding():
    assert _lib.load().fg_plan_sizeof() == C.sizeof(_lib.FgPlan)


def test_schedule_len_host_matches_oracle():
    from oracle import fg_oracle as fo

    L = _lib.load()
    out = C.c_int64(0)
    for a in (2, 3, 5, 12, 1500):
        for k in list(range(0, 200)) + [999, 4095, 9999, 123456]:
            assert L.fg_schedule_len(2, k, a, 0, C.byref(out)) == 0
            assert out.value == sum(n for _, n, _ in fo.schedule_segments("adaptive", k, a)), (a, k)
    assert L.fg_schedule_len(0, 77, 0, 0, C.byref(out)) == 0 and out.value == 78
    assert L.fg_schedule_len(1, 77, 0, 10, C.byref(out)) == 0 and out.value == 11
    assert L.fg_schedule_len(2, 10, 1, 0, C.byref(out)) == _lib.FG_ERR_ARG
    assert b"invalid" in L.fg_last_error()


def test_invalid_plans_rejected_without_gpu():
    L = _lib.load()
    plan = _lib.FgPlan()
    assert L.fg_step(C.byref(plan), 0, None, None) == _lib.FG_ERR_UNSUPPORTED
    plan.ndim, plan.B, plan.n_m, plan.ms = 2, 1, 64, 48
    plan.shape[0], plan.shape[1] = 8, 8
    assert L.fg_step(C.byref(plan), 0, None, None) == _lib.FG_ERR_ARG  # ms not multiple of 32
    plan.ms = 64
    assert L.fg_run(C.byref(plan), 0, 1, None, 0, None, 0, None) == _lib.FG_ERR_ARG  # NULL buffers
    assert b"NULL" in L.fg_last_error()
    with pytest.raises(ValueError):
        _lib.check(L.fg_step(C.byref(plan), 0, None, None))


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1004_5128_b200 as fg

    with pytest.raises(fg.NativeLibraryError):
        fg.build_table(0.5, 10)
    cfg = fg.SimulationConfig(gamma=0.5, alpha=1.0, beta=0.0, dt=1.0, dx=10.0, nx=8, ny=8, n_steps=3,
                              sources=((4, 4, 1.0),))
    with pytest.raises(fg.NativeLibraryError):
        fg.run(cfg)


def test_sass_is_sm100a():
    """The shipped library carries sm_100a SASS with 128-bit global loads."""
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "LDG.E.ENL2.128" in out or "LDG.E.128" in out or re.search(r"LDG\.E[.\w]*\.128", out)
    arr = np.zeros(1)
    assert arr.size == 1


def _valid_looking_plan():
    """A plan whose pointers are non-NULL placeholders: validation only, never launched."""
    plan = _lib.FgPlan()
    plan.ndim, plan.B, plan.n_m, plan.ms = 2, 1, 64, 64
    plan.shape[0], plan.shape[1], plan.shape[2] = 8, 8, 1
    plan.kind, plan.base = 2, 5
    for name in ("psi_dev", "H_dev", "status_dev", "decay_dev", "diffuse_dev", "dt_dev", "horizon_dev", "P_dev"):
        setattr(plan, name, 8)
    plan.u_dev[0] = plan.u_dev[1] = 8
    plan.psi_stride = plan.h_slices = 201
    return plan


def test_blocking_fields_validated_without_gpu():
    """tblock / item_cols / subblock combinations are checked before any launch
    (a zero-step fg_run returns after validation)."""
    L = _lib.load()
    plan = _valid_looking_plan()
    run = lambda: L.fg_run(C.byref(plan), 5, 5, None, 0, None, 0, None)  # noqa: E731
    assert run() == _lib.FG_OK
    plan.tblock = 40  # multiple of 8 above 32: adaptive with blkcoef_dev only
    assert run() == _lib.FG_ERR_UNSUPPORTED
    plan.blkcoef_dev = 8
    assert run() == _lib.FG_OK
    plan.tblock = 12
    assert run() == _lib.FG_ERR_ARG
    plan.tblock = 136  # above kMaxTBlock
    assert run() == _lib.FG_ERR_ARG
    plan.tblock = 128
    plan.subblock = 48  # must divide tblock
    assert run() == _lib.FG_ERR_ARG
    plan.subblock = 4  # 32 sub-blocks > 16
    assert run() == _lib.FG_ERR_ARG
    plan.subblock = 32
    assert run() == _lib.FG_OK
    plan.subdelay = 33  # a sub-block launch feeds steps (i+1)S + D on, D <= S
    assert run() == _lib.FG_ERR_ARG
    plan.subdelay = 8
    assert run() == _lib.FG_OK
    plan.subdelay = 0
    plan.kind = 0  # dense memory: single member only
    plan.tblock, plan.subblock = 32, 8
    assert run() == _lib.FG_OK
    plan.B, plan.ms = 2, 64
    assert run() in (_lib.FG_ERR_ARG, _lib.FG_ERR_UNSUPPORTED)


def test_history_pad_host():
    """fg_history_pad: (box rows - 1) strides of the largest adaptive interval any step samples
    (schedule.py:120-133: interval i >= 2 has stride 2i - 1, first sampled at
    k = a^(i-1) + i); dense schedules read stride-1 boxes."""
    import ctypes as C

    from paper_1004_5128_b200 import _lib

    L = _lib.load()
    out = C.c_int64(0)

    def pad(kind, n, base):
        _lib.check(L.fg_history_pad(kind, n, base, C.byref(out)))
        return out.value

    extra = pad(0, 4000, 0)  # rows per TMA box - 1, times stride 1
    assert extra >= 7 and pad(1, 4000, 0) == extra
    # a = 5: i = 6 (stride 11) first at k = 5^5 + 6 = 3131 <= 3999; i = 7 needs k >= 15632
    assert pad(2, 4000, 5) == extra * 11 and pad(2, 10000, 5) == extra * 11
    assert pad(2, 3132, 5) == extra * 11 and pad(2, 3131, 5) == extra * 9
    assert pad(2, 10, 100) == extra  # base beyond the run: the full schedule
    assert L.fg_history_pad(2, 100, 1, C.byref(out)) == _lib.FG_ERR_ARG
