"""Debug: first step where a blocked ensemble run departs from the unblocked one."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1004_5128_b200 as fg

B, n = int(os.environ.get("DBG_B", 6)), int(os.environ.get("DBG_N", 64))
rng = np.random.default_rng(4)
dx = 1.0 / (n - 1)
x = np.arange(n) * dx
gam = rng.uniform(0.3, 0.9, size=B)
u0 = np.stack([np.exp(-((x - c) ** 2) / (2 * 0.03**2)) for c in rng.uniform(0.2, 0.8, size=B)])
u0[:, 0] = u0[:, -1] = 0
dts = [(0.2 * dx**2) ** (1 / g) for g in gam]
steps = int(os.environ.get("DBG_STEPS", 260))
cfg = fg.FieldConfig(initial=u0, dx=dx, gamma=gam.tolist(), dt=dts, n_steps=steps, strategy=fg.AdaptiveMemory(5),
                     batched=True, snapshot_every=1, history_byte_cap=None)
ref = fg.run_field(cfg, tblock=0)
for tb in [int(t) for t in os.environ.get("DBG_TB", "16,24,32,48").split(",")]:
    for flags in (0, 2):
        got = fg.run_field(cfg, tblock=tb, flags=flags)
        bad = None
        for (s, a), (_, b) in zip(ref.snapshots, got.snapshots):
            err = np.abs(a - b).max() / np.abs(a).max()
            if err > 1e-10:
                bad = (s, err, np.argwhere(np.abs(a - b) > 1e-10 * np.abs(a).max())[:4].tolist())
                break
        print("tb", tb, "flags", flags, "items", os.environ.get("FGB200_BLOCK_ITEMS", "1"), "first bad", bad, flush=True)
