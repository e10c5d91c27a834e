"""Which C3 parameterisation drapes stably?  Fixed mode = the reference
engine's own arithmetic, so the verdict applies to the reference too."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2507_11794_b200 as P
from paper_2507_11794_b200.mesh import SimParams

base = P.baseline_scene("C3")
variants = [("margin1e-3", {}), ("margin3e-4", dict(response_margin=3e-4)),
            ("margin1e-4", dict(response_margin=1e-4)), ("margin0", dict(response_margin=0.0)),
            ("dt2e-3", dict(dt=0.002)), ("sub4", dict(substeps=4))]
for name, kw in variants:
    p = base.params
    d = dict(dt=p.dt, stiffness=p.stiffness, damping=p.damping, response_margin=p.response_margin)
    d.update(kw)
    params = SimParams(**d)
    for prec in ("fixed", "fast"):
        eng = P.Engine(base.mesh, base.obstacle, params, pair_budget=10**13, precision=prec)
        out = []
        t0 = time.time()
        for blk in range(12):
            eng.step_frames(50)
            pos, vel = eng.read_positions(), eng.read_velocities()
            st = eng.stats()
            out.append(f"{(blk+1)*50}:{np.nanmax(np.abs(pos)):.3g}/{np.nanmax(np.abs(vel)):.3g}/h{st['hits']}")
            if not np.isfinite(pos).all() or np.abs(pos).max() > 100:
                break
        print(name, prec, f"{time.time()-t0:.1f}s", " ".join(out), flush=True)
