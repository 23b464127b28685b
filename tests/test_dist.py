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


# ------------------------------------------------------------- slab sharding --

def test_slab_layout_partition_and_plan():
    from paper_1004_5128_b200.sharding import SlabLayout

    for n, world in ((10, 2), (128, 4), (1024, 8), (9, 3)):
        lays = [SlabLayout(n, r, world) for r in range(world)]
        assert lays[0].lo == 0 and lays[-1].hi == n
        assert all(a.hi == b.lo for a, b in zip(lays, lays[1:]))
        assert lays[0].halo_lo == 0 and lays[-1].halo_hi == 0
        for lay in lays:
            assert lay.local_rows == (lay.hi - lay.lo) + lay.halo_lo + lay.halo_hi
            own = lay.own
            assert own.stop - own.start == lay.hi - lay.lo
        # every send is matched by the neighbour's receive with the same tag, and
        # lands in a halo row; every halo row is filled by exactly one receive
        for lay in lays:
            for op, peer, row, tag in lay.exchange_plan():
                other = lays[peer]
                if op == "send":
                    assert any(o == "recv" and q == lay.rank and t == tag for o, q, _, t in other.exchange_plan())
                    assert lay.own.start <= row < lay.own.stop
                else:
                    assert row in (0, lay.local_rows - 1) and not (lay.own.start <= row < lay.own.stop)
    with pytest.raises(ValueError):
        SlabLayout(5, 0, 2)


def _slab_worker(rank, world, port, q, shape, kind, param, n_steps, reaction):
    """The slab driver's host logic (layout, per-step halo exchange, gather) over
    gloo, with the oracle's arithmetic standing in for the GPU engine: each rank
    steps only its slab (own rows + halos) exactly as solver.py:200-226 does."""
    import torch
    import torch.distributed as dist

    from oracle import fg_oracle as fo
    from paper_1004_5128_b200.sharding import SlabLayout, exchange_halos, gather_rows

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    u0, gamma, dt = _slab_problem(shape)
    lay = SlabLayout(shape[0], rank, world)
    u = np.ascontiguousarray(lay.local(u0))
    table = fo.build_table(gamma, n_steps)
    beta = reaction[1] if reaction[0] == "linear" else 0.0
    decay, diffuse = fo.host_scalars(1.0, beta, gamma, dt, 1.0)
    H = np.empty((n_steps + 1,) + u.shape)
    H[0] = fo.stencil(u)
    rows = u.shape[0]
    for k in range(n_steps):
        offs, wts = fo.schedule(kind, k, param, dt)
        acc = fo.history_sum(H[: k + 1], offs, wts, table, k)
        nxt = fo._update(u, acc, reaction, dt, decay, diffuse)
        fo.zero_ring(nxt)                                 # global ring + (harmless) halo rows
        t = torch.from_numpy(nxt).view(rows, -1)
        exchange_halos(t, lay)                            # neighbours' edge rows into the halos
        H[k + 1] = fo.stencil(nxt)
        u = nxt
    full = gather_rows(torch.from_numpy(np.ascontiguousarray(u[lay.own])).view(lay.hi - lay.lo, -1), lay)
    q.put((rank, full.numpy().reshape(shape)))
    dist.destroy_process_group()


def _slab_problem(shape):
    rng = np.random.default_rng(11)
    u0 = rng.uniform(0.0, 1.0, size=shape)
    for ax in range(len(shape)):
        idx = [slice(None)] * len(shape)
        idx[ax] = 0
        u0[tuple(idx)] = 0.0
        idx[ax] = -1
        u0[tuple(idx)] = 0.0
    return u0, 0.6, 0.05


@pytest.mark.parametrize("shape,kind,param,reaction", [
    ((14, 11), "adaptive", 3, ("linear", 0.2)),
    ((9, 6, 5), "full", 0, ("saturating", 0.5, 0.2)),
])
def test_gloo_slab_run_bitwise_equals_single_process(shape, kind, param, reaction):
    """World size 2 over gloo: the slab-sharded run (own rows + one halo row per
    neighbour, per-step exchange) gathers to exactly the single-process oracle run."""
    import torch.multiprocessing as mp

    from oracle import fg_oracle as fo

    n_steps = 40
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, 2, port, q, shape, kind, param, n_steps, reaction))
             for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    u0, gamma, dt = _slab_problem(shape)
    ref = fo.run(fo.OracleProblem(u0=u0[None], gamma=np.array([gamma]), dt=np.array([dt]), alpha=1.0, dx=1.0,
                                  reaction=reaction, strategy=(kind, param), n_steps=n_steps))
    assert np.array_equal(out[0], ref["final"][0]) and np.array_equal(out[1], ref["final"][0])


def test_bench_multi_gpu_c5_is_member_sharded():
    """bench.py --gpus N --config c5 splits ONE seeded ensemble by member (strong
    scaling): the ranks' shards are disjoint, cover all 2048 members, and keep
    each member's γ, Δt and initial field; other workloads run replicas."""
    import bench
    from paper_1004_5128_b200.sharding import shard_config

    assert bench.sharded("c5", 2) and not bench.sharded("c5", 1) and not bench.sharded("c4", 8)
    cfg, _ = bench.workload("c5", 0)
    parts = [shard_config(cfg, r, 3) for r in range(3)]
    assert sum(p.members() for p in parts) == cfg.members()
    np.testing.assert_array_equal(np.concatenate([np.asarray(p.gamma) for p in parts]), np.asarray(cfg.gamma))
    np.testing.assert_array_equal(np.concatenate([np.asarray(p.initial) for p in parts]), np.asarray(cfg.initial))
