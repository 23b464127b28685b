"""Algorithmic bytes of one MAIN block-stage launch (slices t < kb0 - tblock):
the distinct old slices its steps' schedules use, read once, plus the tblock
partial-sum rows it writes.  Used to annotate ncu captures.

    python scripts/main_alg_bytes.py --config c4-adaptive --kb0 1904
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main_bytes(cfg_name: str, kb0: int) -> tuple[int, int]:
    import bench
    from oracle import fg_oracle as fo  # schedules (checker restatement, host-side accounting only)
    from paper_1004_5128_b200._engine import default_tblock

    cfg, _ = bench.workload(cfg_name)
    p = cfg.to_problem()
    tb = default_tblock(p)
    kind = p.kind
    used = set()
    for b in range(tb):
        k = kb0 + b
        offs, _ = fo.schedule(kind, k, float(p.param) if kind != "full" else 0.0)
        for m in offs:
            t = k - int(m)
            if t < kb0 - tb:
                used.add(t)
    slice_bytes = p.batch * p.n_m * 8
    return (len(used) + tb) * slice_bytes, tb


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", required=True)
    ap.add_argument("--kb0", type=int, required=True)
    a = ap.parse_args()
    print(*main_bytes(a.config, a.kb0))
