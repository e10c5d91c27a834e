"""Diagnostics: stability of the drop scenes per precision mode."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_11794_b200 as P

for cfg in ("C4", "C3"):
    sc = P.baseline_scene(cfg)
    for prec in ("fixed", "fast"):
        for graph in (True, False):
            eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, precision=prec, graph=graph)
            line = []
            for f in range(1, 301):
                r = eng.step()
                if f % 25 == 0 or f < 4:
                    p = eng.read_positions(); v = eng.read_velocities()
                    line.append(f"{f}:{np.nanmax(np.abs(p)):.3g}/{np.nanmax(np.abs(v)):.3g}/h{r.hits}")
                    if not np.isfinite(p).all():
                        break
            print(cfg, prec, "graph" if graph else "eager", " ".join(line), flush=True)
sc = P.baseline_scene("C2")
eng = P.Engine(sc.mesh, params=sc.params)
eng.step_frames(300)
p = eng.read_positions()
print("C2 fast 300 frames finite", np.isfinite(p).all(), np.abs(p).max())
