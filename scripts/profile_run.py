"""One run of a workload with no warm-up, for ncu captures (few launches to skip).

    ncu ... python scripts/profile_run.py --config c2 [--flags 2] [--steps N]
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
    ap.add_argument("--flags", type=int, default=None)
    ap.add_argument("--steps", type=int, default=None, help="truncate the run (prefix)")
    ap.add_argument("--split", type=int, default=0)
    args = ap.parse_args()
    import torch
    from dataclasses import replace

    import bench
    from paper_1004_5128_b200._engine import Stepper

    cfg, _ = bench.workload(args.config)
    if args.steps:
        cfg = replace(cfg, n_steps=args.steps)
    st = Stepper(cfg.to_problem(), split=args.split, flags=args.flags)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.advance(cfg.n_steps)
    torch.cuda.synchronize()
    print(f"{args.config}: {cfg.n_steps} steps in {time.perf_counter() - t0:.4f} s, geometry {st.geometry()}")
    st.raise_if_diverged()


if __name__ == "__main__":
    main()
