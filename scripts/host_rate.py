"""Host enqueue time vs device time of one c2 run (is the per-step launch loop host-bound?)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1004_5128_b200._engine import Stepper

cfg, _ = bench.workload(os.environ.get("CFG", "c2"))
st = Stepper(cfg.to_problem(), snapshots=False)
u0 = st.u[0].clone()
for i in range(4):
    st.reset(u0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    st.advance(cfg.n_steps)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"run {i}: host enqueue {1e3 * (t1 - t0):.2f} ms, device {e0.elapsed_time(e1):.2f} ms, wall {1e3 * (t2 - t0):.2f} ms",
          flush=True)
