"""Per-pass CUDA-event timing of the collision config (C3 by default).

    python tools/prof_c3.py [C3|C4] [frames]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2507_11794_b200 as P
from paper_2507_11794_b200 import _native as N

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
narrow = os.environ.get("CS_NARROW", "tri")
sc = P.baseline_scene(cfg)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, stream=stream.cuda_stream,
               narrow=narrow, cell_size=float(os.environ["CS_CELL"]) if "CS_CELL" in os.environ else None)
eng.step_frames(200)
torch.cuda.synchronize()


def ev():
    return torch.cuda.Event(enable_timing=True)


names = [("force", N.PASS_FORCE_INTEGRATE), ("detect", N.PASS_DETECT), ("respond", N.PASS_RESPOND),
         ("normals", N.PASS_NORMALS)]
acc = {k: [] for k, _ in names}
for _ in range(reps):
    evs = []
    for name, pid in names:
        a, b = ev(), ev()
        a.record(stream)
        N.check(eng._lib.cs_run_pass(eng._handle, pid))
        b.record(stream)
        evs.append((name, a, b))
    torch.cuda.synchronize()
    for name, a, b in evs:
        acc[name].append(a.elapsed_time(b) * 1e3)
for name, _ in names:
    print(f"{cfg} {name:8s} median {np.median(acc[name]):8.1f} us")
a, b = ev(), ev()
a.record(stream)
eng.step_frames(reps)
b.record(stream)
torch.cuda.synchronize()
print(f"{cfg} frame (graph) {a.elapsed_time(b) * 1e3 / reps:8.1f} us  -> {1e3 / (a.elapsed_time(b) / reps):.0f} steps/s")
print("broadphase", eng.broadphase_stats(), "hits/frame", eng.stats()["hits"])
