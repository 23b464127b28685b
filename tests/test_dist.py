"""Multi-process host logic on CPU (gloo, world_size 2): member sharding of an
ensemble and the max-over-ranks timing reduction used by bench.py."""

import os
import socket

import numpy as np
import pytest

from paper_1004_5128_b200.sharding import member_range, shard_config


def test_member_ranges_partition():
    for n in (1, 2, 7, 2048, 2049):
        for world in (1, 2, 3, 8):
            if n < world:
                continue
            spans = [member_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        member_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1004_5128_b200 import workloads as W
    from paper_1004_5128_b200.sharding import max_over_ranks, sum_over_ranks

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = W.c5(n_steps=10, members=9, n=512)
    mine = shard_config(cfg, rank, world)
    t = max_over_ranks(1.5 + rank)
    total = sum_over_ranks(float(mine.members()))
    q.put((rank, mine.members(), np.asarray(mine.gamma).tolist(), t, total))
    dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_reduce():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_1004_5128_b200 import workloads as W

    gam = np.asarray(W.c5(n_steps=10, members=9, n=512).gamma).tolist()
    assert out[0][1] + out[1][1] == 9
    assert out[0][2] + out[1][2] == gam          # contiguous blocks, nothing lost or duplicated
    assert out[0][3] == out[1][3] == 2.5          # max over ranks
    assert out[0][4] == out[1][4] == 9.0
