"""ctypes binding of the C ABI in ``include/fgb200.h`` (``_lib/libfgb200.so``).

There is no CPU fallback: if the shared library is missing or no CUDA device is
present, every entry point raises :class:`NativeLibraryError`.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FGB200_LIB") or os.path.join(HERE, "_lib", "libfgb200.so")

ABI_VERSION = 7  # FGB200_ABI_VERSION of include/fgb200.h this binding mirrors
FG_OK = 0
FG_ERR_ARG = -1
FG_ERR_CUDA = -2
FG_ERR_UNSUPPORTED = -3
FG_NO_BAD_STEP = (1 << 63) - 1
FG_RUN_GRAPH = 1
FG_RUN_PDL = 2
FG_RUN_PERSISTENT = 4
FG_RUN_NO_OVERLAP = 64
FG_RUN_NO_PAIRS = 128
FG_RUN_PAIRS = 256
FG_RUN_CONTINUE = 16
FG_STEP_M0_FROM_HISTORY = 1
FG_COEF_ROW = 36  # doubles per coefficient row of blkcoef_dev (include/fgb200.h)
FG_ITEM_PITCH = {8: 12, 16: 20}  # doubles per item coefficient row by item width (kItemPitch8 / kItemPitch)

MEM_KINDS = {"full": 0, "short": 1, "adaptive": 2}
REACTIONS = {"linear": 0, "saturating": 1}

# every symbol include/fgb200.h declares (checked by tests/test_capi.py)
EXPORTS = (
    "fg_abi_version", "fg_plan_sizeof", "fg_last_error", "fg_kernel_launches", "fg_device_info", "fg_psi_tables", "fg_schedule_len",
    "fg_schedule_expand", "fg_history_sum", "fg_stencil", "fg_step", "fg_run", "fg_run_ex", "fg_status",
    "fg_step_geometry", "fg_block_union", "fg_block_partials", "fg_block_subpartials", "fg_block_item_rows",
    "fg_block_item_table", "fg_history_pad",
)


class NativeLibraryError(RuntimeError):
    """The CUDA library is missing, failed to load, or a CUDA call failed."""


class FgPlan(C.Structure):
    """Mirror of ``struct fg_plan`` (include/fgb200.h)."""

    _fields_ = [
        ("B", C.c_int64),
        ("n_m", C.c_int64),
        ("ms", C.c_int64),
        ("ndim", C.c_int32),
        ("reaction", C.c_int32),
        ("shape", C.c_int64 * 3),
        ("kind", C.c_int32),
        ("split", C.c_int32),
        ("base", C.c_int64),
        ("horizon_dev", C.c_void_p),
        ("psi_dev", C.c_void_p),
        ("psi_stride", C.c_int64),
        ("decay_dev", C.c_void_p),
        ("diffuse_dev", C.c_void_p),
        ("dt_dev", C.c_void_p),
        ("vmax", C.c_double),
        ("km", C.c_double),
        ("H_dev", C.c_void_p),
        ("h_slices", C.c_int64),
        ("u_dev", C.c_void_p * 2),
        ("status_dev", C.c_void_p),
        ("step_flags", C.c_int32),
        ("item_cols", C.c_int32),
        ("snap_slot_dev", C.c_void_p),
        ("horizon_max", C.c_int64),
        ("tblock", C.c_int32),
        ("reserved2", C.c_int32),
        ("P_dev", C.c_void_p),
        ("blkcoef_dev", C.c_void_p),
        ("psi_host", C.c_void_p),
        ("subblock", C.c_int64),
        ("coef_rows", C.c_int64),
        ("h_alloc", C.c_int64),
        ("pair_dev", C.c_void_p),
        ("subdelay", C.c_int64),
    ]


_lib = None
_p64 = C.POINTER(C.c_int64)
_p32 = C.POINTER(C.c_int32)


def _declare(L):
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
    plan = C.POINTER(FgPlan)
    sig = {
        "fg_abi_version": (C.c_int, []),
        "fg_plan_sizeof": (C.c_int64, []),
        "fg_last_error": (C.c_char_p, []),
        "fg_kernel_launches": (C.c_int64, []),
        "fg_device_info": (C.c_int, [_p32, _p32, _p32]),
        "fg_psi_tables": (C.c_int, [vp, i64, i64, i64, vp, vp]),
        "fg_schedule_len": (C.c_int, [i32, i64, i64, i64, _p64]),
        "fg_schedule_expand": (C.c_int, [i32, i64, i64, i64, i64, vp, vp, i64, vp, vp]),
        "fg_history_sum": (C.c_int, [vp, i64, i64, vp, vp, i64, vp, i64, i64, vp, vp]),
        "fg_stencil": (C.c_int, [plan, vp, vp, vp]),
        "fg_step": (C.c_int, [plan, i64, vp, vp]),
        "fg_run": (C.c_int, [plan, i64, i64, _p64, i64, vp, i32, vp]),
        "fg_run_ex": (C.c_int, [plan, i64, i64, _p64, i64, vp, vp, i32, vp]),
        "fg_status": (C.c_int, [plan, _p64, vp]),
        "fg_step_geometry": (C.c_int, [plan, _p64, _p32, _p32]),
        "fg_block_union": (C.c_int, [i32, i64, i32, i64, i64, _p64]),
        "fg_block_partials": (C.c_int, [plan, i64, i32, vp]),
        "fg_block_subpartials": (C.c_int, [plan, i64, i32, vp, C.POINTER(C.c_int32)]),
        "fg_block_item_rows": (C.c_int, [i32, i64, i32, i64, i64, i32, _p64]),
        "fg_block_item_table": (C.c_int, [i32, i64, i32, i64, i64, i64, i64, i32, i32, _p64, i32, _p32]),
        "fg_history_pad": (C.c_int, [i32, i64, i64, _p64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def load(path: str = LIB_PATH):
    """Load (once) and return the library; raise loudly if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        try:
            L = C.CDLL(path)
        except OSError as exc:  # pragma: no cover - environment specific
            raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
        _declare(L)
        if L.fg_abi_version() != ABI_VERSION:
            raise NativeLibraryError(f"{path} has ABI {L.fg_abi_version()}, this binding expects {ABI_VERSION}: rebuild it")
        _lib = L
    return _lib


def check(rc: int, what: str = "fgb200") -> None:
    if rc == FG_OK:
        return
    msg = load().fg_last_error().decode(errors="replace")
    if rc in (FG_ERR_ARG, FG_ERR_UNSUPPORTED):
        raise ValueError(f"{what}: {msg}")
    raise NativeLibraryError(f"{what}: {msg} (code {rc})")


def require_cuda():
    """Return the current CUDA device, failing loudly without one."""
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryError("paper_1004_5128_b200 needs a CUDA device (B200, sm_100a); none is visible")
    load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
