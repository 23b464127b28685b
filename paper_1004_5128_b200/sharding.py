"""Multi-GPU layout: one process per GPU.

The GL history sum is pointwise in space (/root/reference/pkg/src/fracgrid/
solver.py:162-197: each point reads only its own history) and only the stencil
couples neighbouring points (grid.py:88-106, a one-cell reach), SURVEY.md §8e:

* Ensembles (BASELINE c5) shard by member with no data-path collective at all:
  rank r owns a contiguous block of members and streams only its own history.
* One large field (c3 2D, c4 3D) shards into slabs along its first (slowest)
  axis: rank r owns rows [lo, hi) plus a one-row halo towards each neighbour,
  stores and streams only its own rows of every history slice (capacity and
  bandwidth both scale), and after every step exchanges its edge rows of u^{k+1}
  with its neighbours (2D 1024²: 8 KB per neighbour; 3D 128³: 128 KB) — the one
  real exchange of the path.  The engine treats a slab's first/last local row as
  boundary ring (δ = 0 there, u pinned to 0), which is exactly right for the
  global boundary and harmless for a halo row: its u is overwritten by the
  exchange before the next step's stencil reads it, and its δ/history belong to
  the neighbour.  Every owned point therefore sees the same operands in the same
  order as the single-GPU run: the sharded result is bitwise identical
  (tests/test_dist.py proves it on CPU with gloo and the oracle's arithmetic).
"""

from __future__ import annotations

import os
from dataclasses import replace

import numpy as np


def dist_env() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults 0, 1, 0)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def member_range(n_members: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced block of members owned by ``rank`` (sizes differ by ≤ 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(int(n_members), world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def shard_config(cfg, rank: int, world: int):
    """This rank's share of a ``FieldConfig``: a member block of an ensemble."""
    if world == 1:
        return cfg
    if not cfg.batched:
        raise ValueError("only batched (ensemble) configs shard by member; use replica_config")
    lo, hi = member_range(cfg.members(), rank, world)
    idx = np.arange(lo, hi)
    return replace(cfg, initial=np.asarray(cfg.initial)[idx],
                   gamma=np.broadcast_to(np.asarray(cfg.gamma, dtype=np.float64), (cfg.members(),))[idx],
                   dt=np.broadcast_to(np.asarray(cfg.dt, dtype=np.float64), (cfg.members(),))[idx])


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (loop time) over the process group, if any."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------ slab sharding --

class SlabLayout:
    """Rows of axis 0 owned by one rank and its local array (own rows + halos)."""

    def __init__(self, n_rows: int, rank: int, world: int):
        if n_rows < 3 * world:
            raise ValueError(f"{n_rows} rows are too few for {world} slabs (at least 3 per rank)")
        self.n_rows, self.rank, self.world = int(n_rows), int(rank), int(world)
        self.lo, self.hi = member_range(n_rows, rank, world)          # owned rows [lo, hi)
        self.halo_lo = 1 if rank > 0 else 0                            # a halo row below lo
        self.halo_hi = 1 if rank < world - 1 else 0                    # a halo row at hi
        self.local_lo, self.local_hi = self.lo - self.halo_lo, self.hi + self.halo_hi

    @property
    def local_rows(self) -> int:
        return self.local_hi - self.local_lo

    @property
    def own(self) -> slice:
        """Owned rows inside the local array."""
        return slice(self.halo_lo, self.halo_lo + (self.hi - self.lo))

    def local(self, field):
        """This rank's local array (own rows + halos) of a global field (rows first)."""
        return field[self.local_lo:self.local_hi]

    def exchange_plan(self) -> list[tuple[str, int, int, int]]:
        """(op, peer, local row, tag): send my edge rows, receive the neighbours' into my halos.
        Tags: 0 = travelling towards higher ranks, 1 = towards lower ranks."""
        ops = []
        r = self.rank
        if self.halo_hi:
            ops.append(("send", r + 1, self.local_rows - 2, 0))   # my last own row → rank+1's low halo
            ops.append(("recv", r + 1, self.local_rows - 1, 1))   # rank+1's first own row → my high halo
        if self.halo_lo:
            ops.append(("send", r - 1, 1, 1))                     # my first own row → rank-1's high halo
            ops.append(("recv", r - 1, 0, 0))                     # rank-1's last own row → my low halo
        return ops


def exchange_halos(rows, layout: SlabLayout) -> None:
    """Per-step halo exchange of a local field laid out rows-first (a torch tensor
    of shape (local_rows, row_elems); CUDA tensors go over NCCL, CPU ones over
    gloo).  Edge rows are sent as contiguous row views; all four point-to-point
    operations are posted at once (batch_isend_irecv) and waited on."""
    import torch.distributed as dist

    if layout.world == 1:
        return
    plan = layout.exchange_plan()
    if rows.is_cuda and dist.get_backend() == "gloo":
        # gloo moves host memory only: stage the edge rows through the host (the
        # one-GPU test of the slab path; ranks on real GPUs use NCCL below)
        bufs = {(op, peer, tag): (rows[row].cpu() if op == "send" else rows[row].new_empty(rows[row].shape, device="cpu"))
                for op, peer, row, tag in plan}
        ops = [dist.P2POp(dist.isend if op == "send" else dist.irecv, bufs[(op, peer, tag)], peer, tag=tag)
               for op, peer, _, tag in plan]
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for op, peer, row, tag in plan:
            if op == "recv":
                rows[row].copy_(bufs[(op, peer, tag)])
        return
    ops = []
    for op, peer, row, tag in plan:
        fn = dist.isend if op == "send" else dist.irecv
        ops.append(dist.P2POp(fn, rows[row], peer, tag=tag))
    for req in dist.batch_isend_irecv(ops):
        req.wait()


def gather_rows(own, layout: SlabLayout, device=None):
    """All ranks' owned rows (rows-first tensors) concatenated on every rank."""
    import torch
    import torch.distributed as dist

    if layout.world == 1:
        return own
    counts = [member_range(layout.n_rows, r, layout.world) for r in range(layout.world)]
    width = own.shape[1:]
    parts = [torch.empty((hi - lo,) + tuple(width), dtype=own.dtype, device=own.device) for lo, hi in counts]
    # rows differ by at most one between ranks: gather padded blocks of the largest size
    big = max(hi - lo for lo, hi in counts)
    pad = torch.zeros((big,) + tuple(width), dtype=own.dtype, device=own.device)
    pad[: own.shape[0]] = own
    if pad.is_cuda and dist.get_backend() == "gloo":  # host-staged (see exchange_halos)
        hb = [torch.empty_like(pad, device="cpu") for _ in counts]
        dist.all_gather(hb, pad.cpu())
        bufs = [b.to(pad.device) for b in hb]
    else:
        bufs = [torch.empty_like(pad) for _ in counts]
        dist.all_gather(bufs, pad)
    for i, (lo, hi) in enumerate(counts):
        parts[i].copy_(bufs[i][: hi - lo])
    return torch.cat(parts, 0)


def run_slabs(cfg, device=None):
    """One field run split into row slabs over the process group.

    Every rank steps its slab on its GPU with the same engine (one launch chain
    per step, ``Stepper.advance``) and exchanges u's edge rows with its
    neighbours after each step (NCCL send/recv of one row = one plane of the
    field).  Returns ``(snapshots, first_bad_step)`` on every rank, snapshots as
    ``[(step, (B, *shape) array)]`` gathered from all ranks.  The slab plans
    use the global field's temporal blocking factor, so results agree with the
    single-GPU run within the parity bound (bitwise when the slab's tile split
    and item width equal the global plan's).
    """
    import torch
    import torch.distributed as dist

    from ._engine import Problem, Stepper, default_tblock

    p = cfg.to_problem()
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    if p.batch != 1 or len(p.shape) < 2:
        raise ValueError("slab sharding splits one 2D or 3D field (ensembles shard by member)")
    lay = SlabLayout(p.shape[0], rank, world)
    local_shape = (lay.local_rows,) + p.shape[1:]
    u0 = np.ascontiguousarray(lay.local(np.asarray(p.u0[0])))[None]
    local = Problem(u0=u0, gamma=p.gamma, dt=p.dt, alpha=p.alpha, dx=p.dx, reaction=p.reaction, kind=p.kind,
                    param=p.param, n_steps=p.n_steps, cadence=p.cadence, history_byte_cap=None)
    st = Stepper(local, device=device, tblock=default_tblock(p))
    row = int(np.prod(local_shape[1:]))
    n_local = lay.local_rows * row
    snaps = {}
    for k in range(p.n_steps):
        st.advance(k + 1)
        rows = st.u[(k + 1) & 1][:n_local].view(lay.local_rows, row)
        exchange_halos(rows, lay)  # the next step's stencil reads the neighbours' edge rows
        if (k + 1) in st.snap_steps:
            snaps[k + 1] = rows[lay.own].clone()
    torch.cuda.synchronize(device)
    bad = torch.tensor([st.first_bad_step() or (1 << 62)], dtype=torch.int64, device=st.device)
    if world > 1:
        if dist.get_backend() == "gloo":
            bad = bad.cpu()
        dist.all_reduce(bad, op=dist.ReduceOp.MIN)
    out = [(0, np.asarray(p.u0))]
    for s in sorted(snaps):
        full = gather_rows(snaps[s], lay).cpu().numpy()
        out.append((s, full.reshape((1,) + p.shape)))
    first_bad = int(bad.item())
    return out, (None if first_bad == 1 << 62 else first_bad)
