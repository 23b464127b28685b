"""Turn the final round-1 captures (gpurun_out/r01s/, scripts/r01s_measure.sh) into
profiles/: launch-list summaries, per-launch DRAM traffic of the c2 main item
launches against their algorithmic bytes, key metrics of the full captures and
the bench lines (run in the build container; reads no reference code)."""

from __future__ import annotations

import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import ncu_summary as NS  # noqa: E402

SRC = os.path.join(ROOT, "gpurun_out", "r01s")
PROF = os.path.join(ROOT, "profiles")


def launch_rows(path):
    text = open(path).read()
    reader = csv.DictReader(io.StringIO(text[text.find('"ID"'):]))
    rows = {}
    for r in reader:
        rid = int(r["ID"])
        rec = rows.setdefault(rid, {"name": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", ""))
        rec[r["Metric Name"]] = NS.to_bytes(r["Metric Value"], r["Metric Unit"]) if "bytes" in r["Metric Name"] else v
    return [rows[k] for k in sorted(rows)]


def main_alg_bytes(kb0, bt, tb, base, n_pts):
    """Union of the slices t < kb0 - tb the steps kb0..kb0+bt-1 read, plus bt P rows."""
    from oracle import fg_oracle as fo

    used = set()
    for b in range(bt):
        k = kb0 + b
        for m0, cnt, st in fo.schedule_segments("adaptive", k, base):
            for c in range(cnt):
                t = k - (m0 + c * st)
                if t < kb0 - tb:
                    used.add(t)
    return 8 * n_pts * (len(used) + bt)


def main():
    os.makedirs(os.path.join(PROF, "r01s"), exist_ok=True)
    for f in os.listdir(SRC):
        if f.startswith("bench_") and f.endswith(".log"):
            lines = [x for x in open(os.path.join(SRC, f)) if x.startswith("{")]
            if lines:
                open(os.path.join(PROF, "r01s", f.replace(".log", ".json")), "w").write(lines[-1])
    shutil.copy(os.path.join(SRC, "smoke.log"), os.path.join(PROF, "r01s", "smoke.log"))
    for cfg in ("c2", "c5"):
        summ = NS.launches(os.path.join(SRC, f"{cfg}_launches.csv"))
        json.dump(summ, open(os.path.join(PROF, f"r01s_{cfg}_launches.json"), "w"), indent=1)
        print(cfg, {k: (v["count"], round(v["share"], 3)) for k, v in summ["kernels"].items()})
    # c2: main item launches of the launch list vs their algorithmic bytes.  Issue
    # order per block kb (fg_run_ex): main(kb + tb) on the side stream, then
    # tail(kb); main(tb) and tail(0) launch no item kernel.
    tb = int(json.load(open(os.path.join(PROF, "r01s", "bench_default.json")))["roofline"]["temporal_block"])
    n, base, n_pts = 5000, 5, 256 * 256
    rows = [r for r in launch_rows(os.path.join(SRC, "c2_launches.csv")) if "fg_block_item8_kernel" in r["name"]]
    seq = []
    for kb in range(0, n, tb):
        if kb + tb < n and kb > 0:
            seq.append(("main", kb + tb))
        if kb > 0:
            seq.append(("tail", kb))
    assert len(seq) == len(rows), (len(seq), len(rows))
    mains = []
    for (role, kb0), r in zip(seq, rows):
        if role == "main":
            bt = min(tb, n - kb0)
            alg = main_alg_bytes(kb0, bt, tb, base, n_pts)
            dram = r["dram__bytes_read.sum"] + r["dram__bytes_write.sum"]
            mains.append({"kb0": kb0, "us": r["gpu__time_duration.sum"] / 1e3 if r["gpu__time_duration.sum"] > 1e4
                          else r["gpu__time_duration.sum"], "dram_bytes": dram, "alg_bytes": alg})
    tot_d = sum(m["dram_bytes"] for m in mains)
    tot_a = sum(m["alg_bytes"] for m in mains)
    json.dump({"c2_main_item_launches": mains, "dram_over_algorithmic": tot_d / tot_a},
              open(os.path.join(PROF, "r01s_c2_main_traffic.json"), "w"), indent=1)
    print("c2 main launches", len(mains), "DRAM / algorithmic bytes", round(tot_d / tot_a, 4))
    # full capture of item8 launch index 140 = main((140 // 2 + 2) * tb)
    kb_cap = (140 // 2 + 2) * tb
    alg_cap = main_alg_bytes(kb_cap, min(tb, n - kb_cap), tb, base, n_pts)
    subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), "--rep",
                    os.path.join(SRC, "c2_item8.ncu-rep"), "--tag", "r01s_c2_item8", "--config", "c2",
                    "--alg-bytes", str(alg_cap)], check=True)
    tr = json.load(open(os.path.join(PROF, "traffic.json")))
    tr["c2"]["capture"] = (f"ncu --set full --clock-control none -k regex:fg_block_item8_kernel -s 140 -c 1 python "
                           f"scripts/profile_run.py --config c2 (tblock {tb}): main item launch of block kb0={kb_cap}")
    tr["c2"]["kernel"] = "fg_block_item8_kernel<224, 6, false> (main)"
    tr["c2"]["launch_list_dram_over_algorithmic"] = tot_d / tot_a
    json.dump(tr, open(os.path.join(PROF, "traffic.json"), "w"), indent=1)
    subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), "--rep",
                    os.path.join(SRC, "c2_step.ncu-rep"), "--tag", "r01s_c2_step", "--config", "c2_step"], check=True)
    subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), "--rep",
                    os.path.join(SRC, "c5_item16.ncu-rep"), "--tag", "r01s_c5_item16", "--config", "c5"], check=True)


if __name__ == "__main__":
    main()
