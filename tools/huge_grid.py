"""One engine at the edge of device memory: a side x side hanging cloth
built on the device (Engine.from_grid), stepped, checked finite, timed.

    python tools/huge_grid.py [side, default 23170] [frames, default 16]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2507_11794_b200 as P
from paper_2507_11794_b200.scenes import CONTACT_DT, NODE_MASS, stable_coefficients

side = int(sys.argv[1]) if len(sys.argv) > 1 else 23170
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 16
k, c = stable_coefficients(NODE_MASS, CONTACT_DT)
t0 = time.perf_counter()
e = P.Engine.from_grid(side, side, P.SimParams(dt=CONTACT_DT, stiffness=k, damping=c),
                       total_mass=NODE_MASS * side * side, pinned_rows="first")
e.synchronize()
setup = time.perf_counter() - t0
free, total = torch.cuda.mem_get_info()
e.step_frames(8)
e.synchronize()
t0 = time.perf_counter()
e.step_frames(frames)
e.synchronize()
dt = (time.perf_counter() - t0) / frames
n = side * side
pos = e.read_positions()
print(f"{side}^2 = {n / 1e6:.0f}M nodes: setup {setup:.2f} s, device memory used "
      f"{(total - free) / 1e9:.1f} of {total / 1e9:.0f} GB, frame {dt * 1e3:.2f} ms "
      f"({n * 60 / dt / 1e12:.2f} TB/s at 60 B/node), finite {bool(np.isfinite(pos[::9973]).all())}, "
      f"lowest y {pos[:, 1].min():.4f}", flush=True)
