"""Small end-to-end workload touching every kernel family (a smoke for new
kernels; compute-sanitizer is closed on this GPU pool -- it refuses to run,
"runs under it have left GPUs needing a reset" -- so this runs plain, with
the kernels' own bounds and the oracle comparisons of tests/ as the checks):
fast / fixed / fp64 steps, collision (fused, batched and warp narrow
phases), debug passes, forces readback, the tensor boundary, the device grid
generator, single-process p2p row bands (both seam handshakes), record."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2507_11794_b200 as P
from paper_2507_11794_b200 import _native as N
from paper_2507_11794_b200.bands import BandedEngine, link_local

sc = P.build_scene(P.ScenarioConfig("drop", (20, 17), obstacle="icosphere:2"))
for narrow in ("batch", "warp"):
    eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, narrow=narrow)
    eng.step_frames(30)
    eng.close()
for precision in ("fast", "fixed", "fp64"):
    eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, precision=precision)
    eng.step_frames(30)
    for pid in (N.PASS_FORCE_INTEGRATE, N.PASS_DETECT, N.PASS_RESPOND, N.PASS_NORMALS):
        N.check(eng._lib.cs_run_pass(eng._handle, pid))
    if precision != "fp64":
        eng.simulate(3)
        eng.read_forces_raw()
        eng.broadphase_dump()
    eng.read_normals()
    eng.close()
import torch  # noqa: E402  (the tensor boundary)

e = P.Engine.from_grid(40, 33, P.SimParams(dt=0.004))
t = torch.empty((e.num_nodes, 3), dtype=torch.float32, device="cuda")
e.step_frames(3)
e.read_positions(out=t)
e.write_velocities(torch.zeros_like(t))
e.step_frames(2)
e.close()
for precision in ("fast", "fixed"):
    e = P.Engine.from_grid(40, 33, P.SimParams(dt=0.004), precision=precision, orientation="xz")
    e.step_frames(3)
    e.read_normals()
    e.close()
topo = torch.empty((sum(P.spring_count_formula(9, 7)), 2), dtype=torch.int32, device="cuda")
N.check(N.load().cs_grid_topology(9, 7, 0, 7, 1.0, 1.0, topo.data_ptr(), None, None, None, None,
                                  None))
torch.cuda.synchronize()
h = P.build_scene(P.ScenarioConfig("hanging", (61, 37), dt=0.004))
for kernel in ("pair", "strip", "tile"):
    e = P.Engine(h.mesh, params=h.params, kernel=kernel)
    e.step_frames(5)
    e.read_normals()
    e.close()
k, c = P.scenes.stable_coefficients(0.05, 0.004)
params = P.SimParams(dt=0.004, stiffness=k, damping=c)
ok = []
for seam in ("kernel", "stream"):
    bands = [BandedEngine(45, 45, params, r, 3, exchange="p2p", seam=seam) for r in range(3)]
    link_local(bands)
    for _ in range(4):
        for b in bands:
            b.step(1)
        for b in bands:
            b.engine.synchronize()
    ok += [bool(np.isfinite(b.owned_positions()).all()) for b in bands]
    for b in bands:
        b.close()
print("sanitize workload ok", ok)
