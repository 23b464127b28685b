"""Benchmark: GL history terms/s of the fused B200 stepper (and the CPU reference arm).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4]

Workload (default ``c4``, the largest single-GPU configuration of BASELINE.json,
configs[3]): 3D 128³ fractional reaction-diffusion (2.1M points, fp64), γ=0.7,
r=0.05, saturating consumption f(u) = -0.5u/(0.2+u), seeded smoothed initial
field, 4000 steps, run with full memory AND with adaptive memory (a=5) — the
config names both.  One benchmark *step* = one complete 4000-step run of each
(1.68e13 + 2.15e12 history terms).  ``--config`` also takes c1, c2, c3 (full,
short and adaptive runs), c5 or a single run (c3-adaptive, c4-full, …).

Metric: GL history terms/s = Σ_k len_k · N / time, whole job over
all ranks.  ``value`` times the runs with inputs resident in HBM (CUDA events on
the launching stream, barrier + synchronise on both sides, max over ranks);
``e2e`` times the public API ``run_field`` from host arrays (H2D of u0, D2H of
the snapshots inside the timed region).  ``roofline`` reports the dominant
kernel (the block stage of the run with the most block-stage time: the dense
fp64-tensor block kernel for full memory, the TMA item kernel for adaptive
memory) against its measured peak; ``runs`` carries every run's own numbers.
``cpu_baseline`` is the C restatement of the reference (oracle/, OpenMP over the
host's cores) on exact prefixes of the same runs.  ``other_configs`` (default
workload, one GPU) adds a short device-timed line for every other BASELINE
config (c1, c2, c3, c5: one warm + two timed complete runs each).

``--impl reference`` times that CPU reference arm alone (rank 0; other ranks exit).
Under torchrun (N > 1) every rank runs an independently seeded replica of the
workload (weak scaling; the spatial slab split of one field is
``paper_1004_5128_b200.sharding``); ``--config c5`` instead splits
one ensemble by member across the ranks (strong scaling, no collective).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GL history terms/s (grid pts × memory terms)"
UNIT = "terms/s"
# workloads made of several runs of one BASELINE config (a bench step runs each once)
GROUPS = {
    "c4": ("c4-full", "c4-adaptive"),
    "c3": ("c3-full", "c3-short", "c3-adaptive"),
}
# CPU arms: exact prefixes (steps) of each run, sized to a few seconds of
# 16-thread C-port time per bench step; single-core figure on shorter prefixes
REF_PREFIX = {"c1": 2000, "c2": 1000, "c3-full": 250, "c3-short": 700, "c3-adaptive": 700,
              "c4-full": 120, "c4-adaptive": 240, "c5": 1000}
SINGLE_PREFIX = {"c1": 500, "c2": 300, "c3-full": 80, "c3-short": 150, "c3-adaptive": 200,
                 "c4-full": 40, "c4-adaptive": 80, "c5": 200}
REF_WARM_STEPS = 50
FP64_TENSOR_PEAK = 37.0e12  # DMMA m8n8k4, measured on this pool (scripts/micro/fp64_rates.cu, profiles/fp64_rates.txt)


def runs_of(name: str) -> tuple[str, ...]:
    return GROUPS.get(name, (name,))


def sharded(name: str, world: int) -> bool:
    """Multi-GPU c5: one 2048-member ensemble split by member across the ranks
    (sharding.shard_config, no data-path collective); every other workload runs
    one seeded replica per rank."""
    return world > 1 and name == "c5"


def workload(name: str, rank: int = 0):
    from paper_1004_5128_b200 import workloads as W

    if name == "c2":
        cfg = W.c2(seed=1 + rank)
        desc = "c2: 2D 256x256 fractional reaction-diffusion, gamma=0.8, r=0.1, f(u)=-0.1u, adaptive memory a=5, 5000 steps"
    elif name == "c1":
        cfg, desc = W.c1(), "c1: 1D 101 points, gamma=0.5, r=0.2, full memory, 2000 steps"
    elif name.startswith("c3-"):
        cfg = W.c3(name[3:], seed=2 + rank)
        desc = f"c3: 2D 1024x1024, gamma=0.6, r=0.1, {name[3:]} memory, 4000 steps"
    elif name.startswith("c4-"):
        cfg = W.c4(name[3:], seed=3 + rank)
        desc = f"c4: 3D 128^3, gamma=0.7, r=0.05, saturating f(u), {name[3:]} memory, 4000 steps"
    elif name == "c5":
        cfg, desc = W.c5(seed=4 + rank), "c5: 2048 x 1D 512-point ensemble, per-member gamma, adaptive a=5, 10000 steps"
    else:
        raise SystemExit(f"unknown config {name}")
    return cfg, desc


def group_desc(name: str) -> str:
    if name == "c4":
        return ("c4: 3D 128^3 (2.1M points, fp64), gamma=0.7, r=0.05, saturating f(u)=-0.5u/(0.2+u), "
                "4000 steps, full memory + adaptive memory a=5 (one run of each per step)")
    if name == "c3":
        return "c3: 2D 1024x1024, gamma=0.6, r=0.1, 4000 steps, full + short L=500 steps + adaptive a=5"
    return workload(name)[1]


def load_peaks() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(config_name: str):
    """Per-launch DRAM traffic from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            data = json.load(fh)
        return data.get(config_name)
    except (OSError, ValueError):
        return None


# ------------------------------------------------------------------ clocks --

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.rows: list[list[str]] = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return self
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self) -> dict:
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if self.thread is not None:
                self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            if len(r) < 7:
                continue
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, r[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def gpu_id_for(device_index: int) -> str:
    import torch

    try:
        uuid = str(torch.cuda.get_device_properties(device_index).uuid)
        return uuid if uuid.startswith("GPU-") else "GPU-" + uuid
    except Exception:
        return str(device_index)


# ---------------------------------------------------------- CPU reference --

def oracle_problem(cfg):
    from oracle import fg_oracle as fo
    from paper_1004_5128_b200._engine import strategy_spec

    p = cfg.to_problem()
    return fo.OracleProblem(u0=p.u0, gamma=p.gamma, dt=p.dt, alpha=p.alpha, dx=p.dx, reaction=p.reaction,
                            strategy=strategy_spec(cfg.strategy), n_steps=p.n_steps, snapshot_every=p.cadence)


def cpu_reference(cfg, steps: int, nthreads: int = 0):
    """Time the C restatement of the reference on a prefix of the run (exact prefix, §8c)."""
    from oracle import fg_oracle as fo
    from oracle import fg_oracle_c as foc

    prob = oracle_problem(cfg)
    kind, param = prob.strategy
    res = foc.run(prob, nthreads=nthreads, max_steps=steps, snapshots=False)
    n = res["steps_run"]
    per_member = fo.count_terms(kind, n, param, float(prob.dt[0]))
    terms = per_member * int(np.prod(prob.u0.shape))
    return terms, res["elapsed_seconds"], n


def cpu_group(name: str, prefixes: dict, nthreads: int = 0):
    """(terms, seconds, description) of the C port over an exact prefix of every run."""
    terms, secs, parts = 0, 0.0, []
    for run in runs_of(name):
        cfg, _ = workload(run)
        t, el, n = cpu_reference(cfg, prefixes[run], nthreads)
        terms += t
        secs += el
        parts.append(f"{run} steps 0..{n - 1} of {cfg.n_steps}")
    return terms, secs, "; ".join(parts)


def cpu_cores() -> int:
    from oracle import fg_oracle_c as foc

    return foc.max_threads()


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def single_core(name: str) -> dict:
    t, el, what = cpu_group(name, SINGLE_PREFIX, nthreads=1)
    return {"value": t / el, "unit": UNIT, "cores": 1, "sample": f"exact prefixes ({what}), 1 thread"}


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # torchrun pins OMP_NUM_THREADS=1 for every rank; only rank 0 works here, so it
        # takes every host core it may run on (set before the oracle library loads libgomp)
        os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    for run in runs_of(args.config):  # warm (page cache, OpenMP pool)
        cpu_reference(workload(run)[0], REF_WARM_STEPS)
    tot_terms, tot_time, what = 0, 0.0, ""
    for _ in range(args.steps):
        t, el, what = cpu_group(args.config, REF_PREFIX)
        tot_terms += t
        tot_time += el
    value = tot_terms / tot_time
    cores = cpu_cores()
    sample = (f"exact prefixes of the same runs per bench step ({what}), C restatement of the reference "
              f"(oracle/fg_oracle.c), {cores} OpenMP threads on {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_time / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": group_desc(args.config), "runs": list(runs_of(args.config)), "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                         "single_core": single_core(args.config)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm --

def sub_launch_bytes(st, prob, bt: int) -> int:
    """Algorithmic bytes of one block's sub-block launches: launch i reads its
    S slices once and adds into the P rows of the steps b >= (i+1)S + D (a
    read-modify-write of each row)."""
    S = int(st.plan.subblock)
    D = int(st.plan.subdelay) or S
    rows = 0
    i = 0
    while (i + 1) * S + D < bt:
        rows += S + 2 * (bt - ((i + 1) * S + D))
        i += 1
    return rows * prob.batch * prob.n_m * 8


def time_block_stage(st, prob, stream, with_sub: bool = False) -> dict:
    """Every block-stage launch pair (main + tail) of one run, replayed over the
    resident history (left by the timed runs) between CUDA events on the
    launching stream; ``with_sub`` also replays each block's sub-block launches
    (slices inside the block, fg_block_subpartials) and counts their bytes."""
    import ctypes as C

    import torch

    from paper_1004_5128_b200 import _lib
    from paper_1004_5128_b200._engine import block_launch_bytes

    L = _lib.load()
    blocks = block_launch_bytes(prob, st.tblock, with_flops=True)
    if not blocks:
        return None
    h = C.c_void_p(_lib.stream_handle(stream))
    plan = C.byref(st.plan)
    n_sub = C.c_int32(0)
    sub_launches = 0

    def stage(kb0, bt):
        nonlocal sub_launches
        _lib.check(L.fg_block_partials(plan, kb0, bt, h), "fg_block_partials")
        if with_sub:
            _lib.check(L.fg_block_subpartials(plan, kb0, bt, h, C.byref(n_sub)), "fg_block_subpartials")
            sub_launches += n_sub.value

    for kb0, bt, _, _ in blocks[-4:]:  # warm (code, smem config)
        stage(kb0, bt)
    sub_launches = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for kb0, bt, _, _ in blocks:
        stage(kb0, bt)
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    nbytes = sum(b[2] for b in blocks)
    flops = sum(b[3] for b in blocks)
    if with_sub:
        nbytes += sum(sub_launch_bytes(st, prob, b[1]) for b in blocks)
        return {"launches": len(blocks), "sub_block_launches": sub_launches, "total_ms": ms,
                "alg_bytes_total": nbytes, "hbm_gbs": nbytes / (ms * 1e-3) / 1e9}
    return {"launches": len(blocks), "total_ms": ms, "avg_launch_us": ms * 1e3 / len(blocks),
            "alg_bytes_per_launch": nbytes / len(blocks), "alg_bytes_total": nbytes,
            "alg_flops_per_launch": flops / len(blocks), "alg_flops_total": flops,
            "hbm_gbs": nbytes / (ms * 1e-3) / 1e9, "fp64_tflops": flops / (ms * 1e-3) / 1e12,
            "fp64_frac": flops / (ms * 1e-3) / FP64_TENSOR_PEAK, "share_of_run": None}


class Run:
    """One run of the workload: its stepper, resident u0 and accounting."""

    def __init__(self, name, rank, dev, args, world=1):
        from paper_1004_5128_b200._engine import Stepper, execution_bytes
        from paper_1004_5128_b200.sharding import shard_config

        self.name = name
        if sharded(name, world):  # one ensemble, members split across the ranks
            cfg, self.desc = workload(name, 0)
            self.cfg = shard_config(cfg, rank, world)
        else:  # one seeded replica per rank
            self.cfg, self.desc = workload(name, rank)
        self.prob = self.cfg.to_problem()
        flags = None if args.flags is None else int(args.flags)
        self.st = Stepper(self.prob, device=dev, split=args.split, flags=flags, tblock=args.tblock)
        self.u0 = self.st.u[0].clone()
        self.terms = self.prob.terms()
        self.single_bytes, self.exec_bytes = execution_bytes(self.prob, self.st.tblock)
        self.ms: list[float] = []

    def run(self):
        self.st.reset(self.u0)
        self.st.advance(self.prob.n_steps)

    def roofline(self, stream, peak_gbs) -> dict:
        st, prob = self.st, self.prob
        run_s = statistics.mean(self.ms) / 1e3
        out = {"run": self.name, "ms_per_run": run_s * 1e3, "terms_per_run": self.terms,
               "terms_per_s": self.terms / run_s, "temporal_block": st.tblock,
               "algorithmic_bytes_per_run": self.exec_bytes, "single_pass_bytes_per_run": self.single_bytes,
               "run_achieved_gbs": self.exec_bytes / run_s / 1e9,
               "run_frac_hbm": self.exec_bytes / run_s / 1e9 / peak_gbs,
               "single_pass_equivalent_gbs": self.single_bytes / run_s / 1e9}
        blk = time_block_stage(st, prob, stream) if st.tblock else None
        if blk:
            blk["share_of_run"] = blk["total_ms"] / (run_s * 1e3)
            item = "fg_block_item8_kernel" if int(st.plan.item_cols) == 8 else "fg_block_item_kernel"
            if prob.kind == "adaptive":
                blk["kernel"] = f"fg_item_coef_kernel + {item} (main + tail)"
                blk["bound"] = "hbm"
            else:
                big = st.tblock == 32 and prob.batch == 1 and -(-prob.n_m // 256) >= 4 * 148
                blk["kernel"] = ("fg_block_coef_kernel + fg_block_tma_solo_kernel (main, one CTA per SM) + "
                                 "fg_block_tma_kernel (tail)" if big
                                 else "fg_block_coef_kernel + fg_block_tma_kernel (main + tail)")
                # at tblock >= 24 a dense block does 2·tblock flops per 8 history bytes:
                # past the fp64 tensor ridge (37 TF/s ÷ 6.45 TB/s ≈ 5.7 flop/B)
                blk["bound"] = "tensor" if st.tblock * 2 / 8 > FP64_TENSOR_PEAK / (peak_gbs * 1e9) else "hbm"
            blk["hbm_frac"] = blk["hbm_gbs"] / peak_gbs
            if int(st.plan.subblock) > 0 and prob.kind == "adaptive":
                # the same item kernel also runs the block's sub-block launches: the
                # whole stage (main + tail + sub-blocks) replayed serially
                sub = time_block_stage(st, prob, stream, with_sub=True)
                sub["hbm_frac"] = sub["hbm_gbs"] / peak_gbs
                blk["with_sub_blocks"] = sub
        out["block_stage"] = blk
        return out


OTHER_CONFIGS = ("c1", "c2", "c3", "c5")  # every other BASELINE config, a short line each


def quick_line(name: str, rank: int, dev, args, stream, reps: int = 2) -> dict:
    """Device-timed runs of another BASELINE config (same method as the headline:
    inputs resident, CUDA events on the launching stream, one untimed warm run)."""
    import torch

    runs = [Run(r, rank, dev, args) for r in runs_of(name)]
    for r in runs:
        r.run()
    torch.cuda.synchronize(dev)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(runs) + 1)] for _ in range(reps)]
    for i in range(reps):
        evs[i][0].record(stream)
        for j, r in enumerate(runs):
            r.run()
            evs[i][j + 1].record(stream)
    torch.cuda.synchronize(dev)
    for r in runs:
        r.st.raise_if_diverged()
    out = {"workload": group_desc(name), "reps": reps, "runs": {}}
    tot_ms = 0.0
    for j, r in enumerate(runs):
        ms = statistics.mean(evs[i][j].elapsed_time(evs[i][j + 1]) for i in range(reps))
        tot_ms += ms
        out["runs"][r.name] = {"ms_per_run": ms, "terms_per_run": r.terms, "terms_per_s": r.terms / (ms * 1e-3),
                               "temporal_block": r.st.tblock, "history_gb": (r.prob.n_steps + 1) * r.prob.batch * r.prob.n_m * 8 / 1e9}
    out["value"] = sum(r.terms for r in runs) / (tot_ms * 1e-3)
    out["unit"] = UNIT
    out["ms_per_step"] = tot_ms
    return out


def single_pass_step(dev, stream, peak_gbs: float, k_first: int = 1500, n_timed: int = 5) -> dict:
    """The unblocked fused step kernel alone (tblock 0: ONE fg_step_kernel launch per
    step streams every slice of the step's schedule from HBM, then stencil, reaction
    and update in the same pass — the single-pass algorithm of the reference and of
    BASELINE.json's north star): c4-full steps k_first .. k_first+n_timed-1, each timed
    with CUDA events on the launching stream after an unblocked prefix has written the
    history.  Algorithmic bytes of step k: its k+1 history slices, the field read and
    the field and stencil slice written."""
    import torch
    from dataclasses import replace

    from paper_1004_5128_b200._engine import Stepper

    cfg = replace(workload("c4-full")[0], n_steps=k_first + n_timed)
    st = Stepper(cfg.to_problem(), tblock=0)
    st.advance(k_first)
    torch.cuda.synchronize(dev)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n_timed + 1)]
    evs[0].record(stream)
    for i in range(n_timed):
        st.advance(k_first + i + 1)
        evs[i + 1].record(stream)
    torch.cuda.synchronize(dev)
    st.raise_if_diverged()
    us = [evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(n_timed)]
    n = int(np.prod(cfg.to_problem().shape))
    by = [(k_first + i + 1 + 3) * n * 8 for i in range(n_timed)]
    gbs = sum(by) / (sum(us) * 1e-6) / 1e9
    return {"kernel": "fg_step_kernel<3, saturating, 1, unblocked> (one launch per step, whole schedule streamed)",
            "workload": f"c4-full steps {k_first}..{k_first + n_timed - 1} with temporal blocking off",
            "us_per_step": us, "algorithmic_bytes_per_step": by, "bound": "hbm", "achieved": gbs, "peak": peak_gbs,
            "unit": "GB/s", "frac": gbs / peak_gbs,
            "ncu": "profiles/r02n_unblocked_c4f_step_ncu_full.txt (DRAM bytes 1.00x algorithmic)"}


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_1004_5128_b200 import _lib
    from paper_1004_5128_b200.problem import run_field
    from paper_1004_5128_b200.sharding import dist_env, max_over_ranks, sum_over_ranks

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    runs = [Run(name, rank, dev, args, world) for name in runs_of(args.config)]
    stream = torch.cuda.current_stream(dev)
    L = _lib.load()
    terms = sum(r.terms for r in runs)

    for _ in range(args.warmup):
        for r in runs:
            r.run()
    torch.cuda.synchronize(dev)
    for r in runs:
        r.st.raise_if_diverged()

    sampler = ClockSampler(gpu_id_for(local)).start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(len(runs) + 1)] for _ in range(args.steps)]
    n0 = L.fg_kernel_launches()  # the library counts every kernel it launches
    for i in range(args.steps):
        evs[i][0].record(stream)
        for j, r in enumerate(runs):
            r.run()
            evs[i][j + 1].record(stream)
    torch.cuda.synchronize(dev)
    total_launches = L.fg_kernel_launches() - n0
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    per_step_ms = []
    for i in range(args.steps):
        for j, r in enumerate(runs):
            r.ms.append(evs[i][j].elapsed_time(evs[i][j + 1]))
        per_step_ms.append(evs[i][0].elapsed_time(evs[i][-1]))
    t_local = sum(per_step_ms) / 1e3
    for r in runs:
        r.st.raise_if_diverged()
    t_max = max_over_ranks(t_local, dev)
    all_terms = sum_over_ranks(float(terms) * args.steps, dev)
    value = all_terms / t_max
    ms_per_step = t_max / args.steps * 1e3

    # roofline of the dominant kernel: the block stage of the run that spends the
    # most time in it, replayed between CUDA events on the launching stream
    peak, peak_src = load_peaks()
    per_run = [r.roofline(stream, peak) for r in runs]
    dom = max((x for x in per_run if x["block_stage"]), key=lambda x: x["block_stage"]["total_ms"], default=None)
    if dom:
        blk = dom["block_stage"]
        tr = load_traffic(dom["run"])
        traffic = None
        if tr and tr.get("algorithmic_bytes_per_launch"):
            # ncu DRAM bytes of the captured launch, scaled to the average launch
            traffic = tr["dram_bytes_per_launch"][0] * blk["alg_bytes_per_launch"] / tr["algorithmic_bytes_per_launch"][0]
        if blk["bound"] == "tensor":
            achieved = blk["alg_flops_per_launch"] / (blk["avg_launch_us"] * 1e-6) / 1e12
            roofline = {"bound": "tensor", "achieved": achieved, "peak": FP64_TENSOR_PEAK / 1e12, "unit": "TFLOP/s",
                        "frac": achieved * 1e12 / FP64_TENSOR_PEAK, "traffic": traffic,
                        "peak_source": "measured fp64 DMMA m8n8k4 rate on this pool (profiles/fp64_rates.txt; "
                                       "MEASURED_PEAKS.json has no fp64 figure)",
                        "hbm_frac": blk["hbm_frac"], "hbm_peak_gbs": peak}
        else:
            achieved = blk["alg_bytes_per_launch"] / (blk["avg_launch_us"] * 1e-6) / 1e9
            roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                        "traffic": traffic, "peak_source": peak_src}
        roofline.update({"kernel": f"{dom['run']}: {blk['kernel']}", "traffic_detail": tr, "runs": per_run,
                         "note": ("achieved = algorithmic bytes (or flops) per block-stage launch pair of the "
                                  "dominant run / its average duration (CUDA events on the launching stream); "
                                  "traffic = ncu DRAM bytes of a captured launch scaled by its algorithmic-byte "
                                  "ratio.  With temporal blocking one history pass serves temporal_block steps, "
                                  "so single_pass_equivalent_gbs exceeds the HBM peak")})
    else:
        run_s = t_local / args.steps
        ex = sum(r.exec_bytes for r in runs)
        roofline = {"bound": "hbm", "achieved": ex / run_s / 1e9, "peak": peak, "unit": "GB/s",
                    "frac": ex / run_s / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                    "kernel": "fg_step_kernel (whole run)", "runs": per_run}

    launch_geo = [dict(zip(("ctas", "threads", "split"), r.st.geometry()), flags=r.st.flags) for r in runs]
    h2d = sum(r.st.h2d_bytes for r in runs)
    d2h = sum(8 * r.prob.batch * r.st.ms * len([s for s in r.st.snap_steps if s > 0]) for r in runs)
    info = [{"run": r.name, "grid": list(r.prob.shape), "members": r.prob.batch, "n_steps": r.prob.n_steps,
             "memory": f"{r.prob.kind}:{r.prob.param}" if r.prob.kind != "full" else "full",
             "history_gb": (r.prob.n_steps + 1) * r.prob.batch * r.prob.n_m * 8 / 1e9, "terms_per_run": r.terms}
            for r in runs]
    cfgs = [r.cfg for r in runs]
    flags = None if args.flags is None else int(args.flags)
    # free the resident histories before the public-API runs allocate theirs (the
    # loops above leave `r` bound to the last run: c5 cannot hold two histories)
    del runs, r
    torch.cuda.empty_cache()

    # end to end through the public API, host arrays in and out (one untimed pass
    # first, like the device arm's warm-up: allocator pools and pinned staging)
    for cfg in cfgs:
        run_field(cfg, split=args.split, flags=flags, tblock=args.tblock)
    e2e_times = []
    for _ in range(max(1, min(args.steps, 5))):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for cfg in cfgs:
            res = run_field(cfg, split=args.split, flags=flags, tblock=args.tblock)
            del res
        e2e_times.append(time.perf_counter() - t0)
    e2e_local = statistics.mean(e2e_times)
    e2e_max = max_over_ranks(e2e_local, dev)
    e2e_value = sum_over_ranks(float(terms), dev) / e2e_max

    # the other BASELINE configs, a short device-timed line each (default workload only)
    others = None
    if world == 1 and args.config == "c4" and not args.no_other_configs and args.tblock is None:
        others = {}
        for name in OTHER_CONFIGS:
            torch.cuda.empty_cache()
            try:
                others[name] = quick_line(name, rank, dev, args, stream)
            except Exception as exc:  # the headline line must survive a failed side measurement
                others[name] = {"error": f"{type(exc).__name__}: {exc}"}
        torch.cuda.empty_cache()
    single = None
    if others is not None:
        try:
            single = single_pass_step(dev, stream, peak)
        except Exception as exc:
            single = {"error": f"{type(exc).__name__}: {exc}"}
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        t, el, what = cpu_group(args.config, REF_PREFIX)
        cpu = {"value": t / el, "unit": UNIT, "cores": cpu_cores(), "kind": "port",
               "sample": f"exact prefixes of the same runs ({what}), C restatement of the reference path "
                         f"(oracle/fg_oracle.c), OpenMP on {cpu_model()}",
               "single_core": single_core(args.config)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if sharded(args.config, world) else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": group_desc(args.config), "runs": info, "terms_per_step": terms,
                       "l2": "inputs larger than L2 (history > 126 MB L2; not flushed)",
                       "parallelism": ("single GPU" if world == 1 else
                                       f"ensemble members sharded x{world} (strong scaling, no collective)"
                                       if sharded(args.config, world) else
                                       f"independent replicas x{world} (weak scaling)"),
                       "launch": launch_geo},
            "gpu_launches": total_launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "seconds_per_step": e2e_max},
            "clocks": clocks,
            "other_configs": others,
            "single_pass_step": single,
            "per_step_ms": per_step_ms,
            "device": torch.cuda.get_device_name(dev),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="c4")
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--flags", type=int, default=None)
    ap.add_argument("--tblock", type=int, default=None, help="temporal blocking factor (0 = off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the short lines of the other BASELINE configs (default workload only)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
