"""Small end-to-end workload touching every kernel family (a smoke for new
kernels; compute-sanitizer is not available on the GPU pool):
fast / fixed / fp64 steps, collision (batched narrow phase), debug passes,
single-process p2p row bands, record."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2507_11794_b200 as P
from paper_2507_11794_b200 import _native as N
from paper_2507_11794_b200.bands import BandedEngine, link_local

sc = P.build_scene(P.ScenarioConfig("drop", (20, 17), obstacle="icosphere:2"))
for precision in ("fast", "fixed", "fp64"):
    eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, precision=precision)
    eng.step_frames(30)
    for pid in (N.PASS_FORCE_INTEGRATE, N.PASS_DETECT, N.PASS_RESPOND, N.PASS_NORMALS):
        N.check(eng._lib.cs_run_pass(eng._handle, pid))
    if precision != "fp64":
        eng.simulate(3)
    eng.read_normals()
    eng.close()
h = P.build_scene(P.ScenarioConfig("hanging", (61, 37), dt=0.004))
for kernel in ("pair", "strip", "tile"):
    e = P.Engine(h.mesh, params=h.params, kernel=kernel)
    e.step_frames(5)
    e.read_normals()
    e.close()
k, c = P.scenes.stable_coefficients(0.05, 0.004)
params = P.SimParams(dt=0.004, stiffness=k, damping=c)
bands = [BandedEngine(45, 45, params, r, 3, exchange="p2p") for r in range(3)]
link_local(bands)
for _ in range(4):
    for b in bands:
        b.step(1)
    for b in bands:
        b.engine.synchronize()
print("sanitize workload ok", [np.isfinite(b.owned_positions()).all() for b in bands])
