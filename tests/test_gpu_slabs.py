"""Slab-sharded single-field runs on the GPU.

World size 1 runs the per-step slab driver (one advance per step, halo exchange
a no-op) and must reproduce the engine's own run bit for bit.  Two ranks with
real halos run on the one GPU over gloo (edge rows staged through the host).
The 2-rank NCCL run needs two GPUs: it is launched with torchrun when they are
present and skipped otherwise (the host logic is also proven with gloo and the
oracle's arithmetic in tests/test_dist.py).
"""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cfg():
    from paper_1004_5128_b200 import workloads as W

    from dataclasses import replace

    return replace(W.c3("adaptive", n_steps=300, n=96), snapshot_every=100)


def test_slab_driver_world1_bitwise(cuda_device):
    import paper_1004_5128_b200 as fg
    from paper_1004_5128_b200.sharding import run_slabs

    cfg = _cfg()
    snaps, bad = run_slabs(cfg, device=cuda_device)
    ref = fg.run_field(cfg)
    assert bad is None
    assert [s for s, _ in snaps] == [s for s, _ in ref.snapshots]
    for (_, got), (_, want) in zip(snaps, ref.snapshots):
        assert np.array_equal(got[0], want)


def _worker_main():
    import torch
    import torch.distributed as dist

    import paper_1004_5128_b200 as fg
    from paper_1004_5128_b200.sharding import run_slabs

    rank = int(os.environ["RANK"])
    if os.environ.get("FGB200_SLAB_TEST_BACKEND") == "gloo":
        # both ranks on cuda:0, halos staged through the host: the ranks' kernels
        # never wait on one another (each exchange is host-synchronised)
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", device_id=dev)
    cfg = _cfg()
    snaps, bad = run_slabs(cfg, device=dev)
    if rank == 0:
        ref = fg.run_field(cfg)
        worst = max(float(np.abs(g[0] - w).max() / np.abs(w).max()) for (_, g), (_, w) in zip(snaps, ref.snapshots))
        assert bad is None and worst <= 1e-10, worst
        print("slab parity ok", worst)
    dist.destroy_process_group()


def test_slab_two_ranks_one_gpu_gloo(cuda_device):
    """The 2-rank slab path with real halos on ONE GPU: two processes share
    cuda:0, every rank runs the engine on its slab, edge rows travel over gloo
    through the host.  Same layout, plan and gather as the NCCL run."""
    env = dict(os.environ, FGB200_SLAB_TEST_BACKEND="gloo")
    env.setdefault("GLOO_SOCKET_IFNAME", "lo")  # both ranks are local; the box's hostname may not resolve
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29534", os.path.abspath(__file__)]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    assert "slab parity ok" in res.stdout


def test_slab_two_ranks_nccl(cuda_device):
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (host logic is covered by the gloo test)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.abspath(__file__)]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    assert "slab parity ok" in res.stdout


if __name__ == "__main__":
    sys.path.insert(0, ROOT)
    _worker_main()
