"""Wall-time breakdown of one public-API run (run_field): setup, stepping, fetch.

    python scripts/e2e_breakdown.py --config c2 [--reps 3]
"""

from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch

    import bench
    from paper_1004_5128_b200._engine import Stepper
    from paper_1004_5128_b200.problem import run_field

    cfg, _ = bench.workload(args.config)
    run_field(cfg)  # warm
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prob = cfg.to_problem()
        t1 = time.perf_counter()
        st = Stepper(prob)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        st.run()
        t3 = time.perf_counter()
        st.fetch_snapshots()
        t4 = time.perf_counter()
        del st
        t5 = time.perf_counter()
        res = run_field(cfg)
        t6 = time.perf_counter()
        print(f"to_problem {1e3 * (t1 - t0):.2f} ms  Stepper() {1e3 * (t2 - t1):.2f} ms  run {1e3 * (t3 - t2):.2f} ms  "
              f"fetch {1e3 * (t4 - t3):.2f} ms  free {1e3 * (t5 - t4):.2f} ms  | run_field {1e3 * (t6 - t5):.2f} ms "
              f"({len(res.snapshots)} snapshots)")


if __name__ == "__main__":
    main()
