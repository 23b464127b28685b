"""Summarise ncu output from gpurun_out/ into profiles/ (run in the build container).

    python scripts/ncu_summary.py --launches gpurun_out/launches.csv \
        --rep gpurun_out/prof_c2.ncu-rep --tag r01_c2 --config c2

Writes profiles/<tag>_launches.json (per-kernel share of the launch list),
profiles/<tag>_ncu_full.txt (key metrics of the captured launches) and updates
profiles/traffic.json (DRAM bytes per launch vs the algorithmic bytes of that
launch) which bench.py reports as roofline.traffic.
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "sm__maximum_warps_per_active_cycle_pct",
    "launch__grid_size",
    "lts__t_sector_hit_rate.pct",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
]


def launches(path: str) -> dict:
    rows = []
    with open(path) as fh:
        text = fh.read()
    start = text.find('"ID"')
    reader = csv.DictReader(io.StringIO(text[start:]))
    for r in reader:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")), r.get("Metric Unit", "")))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    unit = rows[0][2] if rows else ""
    for name, v, _ in rows:
        short = name.replace("void ", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        short = short.split("(")[0].split("<")[0]
        tot[short] += v
        cnt[short] += 1
    total = sum(tot.values())
    return {"unit": unit, "launches": len(rows), "total": total,
            "kernels": {k: {"count": cnt[k], "total": tot[k], "share": tot[k] / total if total else 0.0}
                        for k in sorted(tot, key=lambda k: -tot[k])}}


def raw_metrics(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    header, units, data = rows[0], rows[1], rows[2:]
    res = []
    for d in data:
        rec = {}
        for h, u, v in zip(header, units, d):
            if h in KEYS or h in ("Kernel Name", "ID", "Grid Size", "Block Size"):
                rec[h] = (v, u)
        res.append(rec)
    return res


def to_bytes(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    return x * scale


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--alg-bytes", type=float, nargs="*", default=None,
                    help="algorithmic bytes of each captured launch, in capture order")
    args = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if args.launches:
        summ = launches(args.launches)
        with open(os.path.join(PROF, f"{args.tag}_launches.json"), "w") as fh:
            json.dump(summ, fh, indent=1)
        print(json.dumps(summ, indent=1)[:2000])
    if args.rep:
        recs = raw_metrics(args.rep)
        lines = []
        traffic = []
        for i, r in enumerate(recs):
            lines.append(f"--- launch {i}: {r.get('Kernel Name', ('?',))[0][:90]}")
            for k in KEYS:
                if k in r:
                    lines.append(f"  {k:70s} {r[k][0]:>16s} {r[k][1]}")
            if "dram__bytes_read.sum" in r and "dram__bytes_write.sum" in r:
                rd = to_bytes(*r["dram__bytes_read.sum"])
                wr = to_bytes(*r["dram__bytes_write.sum"])
                traffic.append(rd + wr)
        with open(os.path.join(PROF, f"{args.tag}_ncu_full.txt"), "w") as fh:
            fh.write("\n".join(lines) + "\n")
        print("\n".join(lines))
        if traffic:
            path = os.path.join(PROF, "traffic.json")
            data = {}
            if os.path.exists(path):
                with open(path) as fh:
                    data = json.load(fh)
            entry = {"dram_bytes_per_launch": traffic, "source": f"profiles/{args.tag}_ncu_full.txt"}
            if args.alg_bytes:
                entry["algorithmic_bytes_per_launch"] = args.alg_bytes
                entry["ratio"] = [t / a for t, a in zip(traffic, args.alg_bytes)]
            data[args.config] = entry
            with open(path, "w") as fh:
                json.dump(data, fh, indent=1)


if __name__ == "__main__":
    sys.exit(main())
