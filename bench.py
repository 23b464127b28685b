"""Benchmark: GL history terms/s of the fused B200 stepper (and the CPU reference arm).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Workload (BASELINE.json configs[1], the metric's configuration): c2 — 2D 256x256
fractional reaction-diffusion, γ=0.8, r=0.1, f(u)=-0.1u, adaptive memory a=5,
5000 GL steps, seeded synthetic initial field.  One benchmark *step* = one
complete 5000-step run (every fused step kernel of the simulation).

Metric: GL history terms/s = Σ_k len_k · N / time, whole job over
all ranks.  ``value`` times the run with inputs resident in HBM (CUDA events on
the launching stream, barrier + synchronise on both sides, max over ranks);
``e2e`` times the public API ``run_field`` from host arrays (H2D of u0, D2H of
the snapshots inside the timed region).  ``roofline`` reports the fused step
kernel against the measured HBM copy peak; ``cpu_baseline`` the C restatement of
the reference (oracle/, OpenMP over the host's cores) on a bounded prefix sample.

``--impl reference`` times that CPU reference arm alone (rank 0; other ranks exit).
Under torchrun (N > 1) each rank runs an independently seeded member of the
workload (weak scaling, member sharding, no data-path collective).
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
REF_SAMPLE_STEPS = 1000       # CPU reference arm: prefix of the c2 run per timed step
REF_WARM_STEPS = 100
CPU_BASELINE_STEPS = 1000     # cpu_baseline sample inside our own line (rank 0, N=1)


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


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    cfg, desc = workload(args.config)
    for _ in range(args.warmup):
        cpu_reference(cfg, REF_WARM_STEPS)
    tot_terms, tot_time, n = 0, 0.0, 0
    for _ in range(args.steps):
        t, el, n = cpu_reference(cfg, REF_SAMPLE_STEPS)
        tot_terms += t
        tot_time += el
    value = tot_terms / tot_time
    cores = cpu_cores()
    sample = (f"prefix of the first {n} of {cfg.n_steps} steps of the same workload per bench step "
              f"(exact prefix), C restatement of the reference, {cores} OpenMP threads on {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_time / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "parallelism": "cpu"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm --

def time_block_stage(st, prob, stream) -> dict:
    """Every block-kernel launch of one run, replayed over the resident history
    (left by the timed runs) between CUDA events on the launching stream."""
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
    for kb0, bt, _, _ in blocks[-4:]:  # warm (code, smem config)
        _lib.check(L.fg_block_partials(plan, kb0, bt, h), "fg_block_partials")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for kb0, bt, _, _ in blocks:
        _lib.check(L.fg_block_partials(plan, kb0, bt, h), "fg_block_partials")
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    nbytes = sum(b[2] for b in blocks)
    flops = sum(b[3] for b in blocks)
    fp64_peak = 37.0e12  # measured DMMA m8n8k4 rate, profiles/fp64_rates.txt
    return {"launches": len(blocks), "total_ms": ms, "avg_launch_us": ms * 1e3 / len(blocks),
            "alg_bytes_per_launch": nbytes / len(blocks), "alg_bytes_total": nbytes,
            "alg_flops_total": flops, "fp64_tflops": flops / (ms * 1e-3) / 1e12,
            "fp64_frac": flops / (ms * 1e-3) / fp64_peak, "fp64_peak_tflops": fp64_peak / 1e12,
            "share_of_run": None}


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_1004_5128_b200 import _lib
    from paper_1004_5128_b200._engine import Stepper, execution_bytes
    from paper_1004_5128_b200.problem import run_field
    from paper_1004_5128_b200.sharding import dist_env, max_over_ranks, sum_over_ranks

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg, desc = workload(args.config, rank)
    prob = cfg.to_problem()
    n_steps = prob.n_steps
    flags = None if args.flags is None else int(args.flags)
    st = Stepper(prob, device=dev, split=args.split, flags=flags, tblock=args.tblock)
    u0_dev = st.u[0].clone()
    terms = prob.terms()
    # algorithmic bytes per run.  Single pass: history reads
    # 8·N·len_k plus u^k read, u^{k+1} write and δ^k write (8·N each) per step.
    # With temporal blocking (st.tblock) the algorithm as executed reads each
    # block's union of old slices once, plus partial sums and recent slices.
    n_pts = prob.batch * prob.n_m
    hist_bytes = 8 * terms
    single_bytes, exec_bytes = execution_bytes(prob, st.tblock)
    stream = torch.cuda.current_stream(dev)
    L = _lib.load()

    def one_run():
        st.reset(u0_dev)
        st.advance(n_steps)

    for _ in range(args.warmup):
        one_run()
    torch.cuda.synchronize(dev)
    st.raise_if_diverged()

    sampler = ClockSampler(gpu_id_for(local)).start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    n0 = L.fg_kernel_launches()  # the library counts every kernel it launches
    evs[0].record(stream)
    for i in range(args.steps):
        one_run()
        evs[i + 1].record(stream)
    torch.cuda.synchronize(dev)
    total_launches = L.fg_kernel_launches() - n0
    launches = total_launches // args.steps
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    per_run_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    t_local = sum(per_run_ms) / 1e3
    st.raise_if_diverged()
    t_max = max_over_ranks(t_local, dev)
    all_terms = sum_over_ranks(float(terms) * args.steps, dev)
    value = all_terms / t_max
    ms_per_step = t_max / args.steps * 1e3

    # roofline.  Whole run: bytes of the algorithm as executed ÷ device time per
    # run (gaps between launches count).  Dominant kernel: with temporal blocking
    # the block stage (fg_block_coef_kernel + fg_block_tma_kernel, >50% of the
    # launch list) timed live below; without it the step kernel, i.e. the run.
    peak, peak_src = load_peaks()
    run_s = t_local / args.steps
    run_achieved = exec_bytes / run_s / 1e9
    tr = load_traffic(args.config)
    blk = time_block_stage(st, prob, stream) if st.tblock else None
    if blk:
        blk["share_of_run"] = blk["total_ms"] / (run_s * 1e3)
        achieved = blk["alg_bytes_per_launch"] / (blk["avg_launch_us"] * 1e-6) / 1e9
        item = "fg_block_item8_kernel" if int(st.plan.item_cols) == 8 else "fg_block_item_kernel"
        sub = f" + sub-block launches (S={int(st.plan.subblock)})" if int(st.plan.subblock) else ""
        kernel = (f"block stage (per block: fg_item_coef_kernel + {item} main + tail{sub})"
                  if prob.kind == "adaptive" else
                  "block stage (per block: coefficient kernels + fg_block_tma_kernel main + tail)")
        traffic = tr["dram_bytes_per_launch"][0] * blk["alg_bytes_per_launch"] / tr["algorithmic_bytes_per_launch"][0] \
            if tr and tr.get("algorithmic_bytes_per_launch") else None
    else:
        achieved = run_achieved
        kernel = "fg_step_kernel"
        traffic = tr["dram_bytes_per_launch"][0] if tr else None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_detail": tr, "kernel": kernel, "block_stage": blk,
                "run_achieved": run_achieved, "run_frac": run_achieved / peak,
                "peak_source": peak_src,
                "algorithmic_bytes_per_run": exec_bytes,
                "single_pass_bytes_per_run": single_bytes,
                "single_pass_equivalent_gbs": single_bytes / run_s / 1e9,
                "history_bytes_per_run": hist_bytes,
                "launches_per_run": launches,
                "avg_launch_us": run_s / launches * 1e6,
                "temporal_block": st.tblock,
                "note": ("achieved = algorithmic bytes per launch of the dominant kernel / its average launch "
                         "time (CUDA events on the launching stream); traffic = ncu DRAM bytes of the captured "
                         "launch scaled to the average launch by its algorithmic-byte ratio; run_achieved = "
                         "executed algorithmic bytes per run / run time.  With temporal blocking one history "
                         "pass serves temporal_block steps, so the single-pass-equivalent rate exceeds HBM peak")}

    ctas, threads, split = st.geometry()
    h2d = st.h2d_bytes
    d2h = 8 * prob.batch * st.ms * len([s for s in st.snap_steps if s > 0])
    st_flags = st.flags
    del st, u0_dev  # free the resident history before the public-API runs allocate theirs
    torch.cuda.empty_cache()

    # end to end through the public API, host arrays in and out (one untimed call
    # first, like the device arm's warm-up: allocator pools and pinned staging)
    run_field(cfg, split=args.split, flags=flags, tblock=args.tblock)
    e2e_times = []
    for i in range(max(1, min(args.steps, 5))):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        res = run_field(cfg, split=args.split, flags=flags, tblock=args.tblock)
        t1 = time.perf_counter()
        e2e_times.append(t1 - t0)
        del res
    e2e_local = statistics.mean(e2e_times)
    e2e_max = max_over_ranks(e2e_local, dev)
    e2e_value = sum_over_ranks(float(terms), dev) / e2e_max

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        t, el, n = cpu_reference(cfg, CPU_BASELINE_STEPS)
        cpu = {"value": t / el, "unit": UNIT, "cores": cpu_cores(), "kind": "port",
               "sample": f"first {n} of {n_steps} steps of the same workload (exact prefix), C restatement of "
                         f"the reference path, OpenMP on {cpu_model()}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "grid": list(prob.shape), "members_per_rank": prob.batch,
                       "n_steps": n_steps, "memory": f"{prob.kind}:{prob.param}" if prob.kind != "full" else "full",
                       "history_gb": (n_steps + 1) * n_pts * 8 / 1e9, "terms_per_run": terms,
                       "l2": "inputs larger than L2 (history > 126 MB L2; not flushed)",
                       "parallelism": f"member-sharded x{world}" if world > 1 else "single GPU",
                       "launch": {"ctas": ctas, "threads": threads, "split": split, "flags": st_flags}},
            "gpu_launches": total_launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "seconds_per_step": e2e_max},
            "clocks": clocks,
            "per_run_ms": per_run_ms,
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
    ap.add_argument("--config", default="c2")
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--flags", type=int, default=None)
    ap.add_argument("--tblock", type=int, default=None, help="temporal blocking factor (0 = off)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
