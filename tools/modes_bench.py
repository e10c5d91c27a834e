"""Steps/s of each arithmetic mode at a config (graph replays, L2 not flushed).

    python tools/modes_bench.py C2 [frames]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2507_11794_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 50
sc = P.baseline_scene(cfg)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
for prec in os.environ.get("CS_MODES", "fast,fixed,fp64").split(","):
    eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, precision=prec,
                   stream=stream.cuda_stream, normals=os.environ.get("CS_NORMALS", "auto"))
    eng.step_frames(5 if sc.obstacle is None else 200)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(k):
        eng.step()
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / k
    print(f"{cfg} {prec:5s}: {ms * 1e3:8.1f} us/frame  {1000 / ms:9.0f} steps/s  "
          f"({eng.kernels_per_frame} kernels/frame)", flush=True)
    # the passes alone (force + integrate, normals)
    from paper_2507_11794_b200 import _native as N
    for name, pid in (("force+integrate", N.PASS_FORCE_INTEGRATE), ("normals", N.PASS_NORMALS)):
        N.check(eng._lib.cs_run_pass(eng._handle, pid))
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(k):
            N.check(eng._lib.cs_run_pass(eng._handle, pid))
        b.record(stream)
        torch.cuda.synchronize()
        print(f"    {name:16s} {a.elapsed_time(b) / k * 1e3:8.1f} us", flush=True)
    eng.close()
