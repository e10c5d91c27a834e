"""C3 stability / contact statistics over a long run, both precisions."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2507_11794_b200 as P

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
sc = P.baseline_scene(sys.argv[2] if len(sys.argv) > 2 else "C3")
for prec in ("fixed", "fast"):
    eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, precision=prec)
    out, t0, last = [], time.time(), 0
    for blk in range(frames // 100):
        eng.step_frames(100)
        pos, vel = eng.read_positions(), eng.read_velocities()
        hc = eng.stats()["hit_counter"]
        out.append(f"{(blk + 1) * 100}:{np.abs(pos).max():.3g}/{np.abs(vel).max():.3g}/h{(hc - last) // 100}")
        last = hc
        if not np.isfinite(pos).all():
            break
    print(prec, f"{time.time() - t0:.1f}s", " ".join(out), flush=True)
