"""Build ``_lib/libfgb200.so`` in-tree with nvcc for sm_100a (no JIT cache).

    python -m paper_1004_5128_b200.build

The C ABI library links the CUDA runtime statically so it does not depend on
which libcudart torch happened to load; device pointers and streams are shared
through the driver's primary context.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "libfgb200.so")
SOURCES = [os.path.join(CSRC, "fg_kernels.cu")]
HEADERS = ("fg_common.cuh", "fg_schedule.cuh", "fg_step.cuh", "fg_block_dense.cuh", "fg_block_items.cuh",
           "fg_support.cuh")
DEPS = SOURCES + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "fgb200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str = OUT, defines: tuple[str, ...] = ()) -> str:
    """Compile the library; ``defines`` builds an experimental variant into ``out``."""
    if not force and out == OUT and not defines and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(out), exist_ok=True)
    tmp = out + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-o", tmp,
           *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stderr[-4000:]}")
    if verbose:
        sys.stderr.write(res.stderr)
    with open(out[: -len(".so")] + ".ptxas.log", "w") as fh:
        fh.write(res.stderr)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
