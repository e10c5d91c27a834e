"""Per-pass CUDA-event timing (L2 flushed between launches) for a config.

    python tools/prof_kernels.py C5 [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2507_11794_b200 as P
from paper_2507_11794_b200 import _native as N

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
t0 = time.time()
sc = P.baseline_scene(cfg)
t1 = time.time()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, stream=stream.cuda_stream,
               kernel=os.environ.get("CS_KERNEL", "pair"),
               normals=os.environ.get("CS_NORMALS", "auto"))
t2 = time.time()
print(f"{cfg}: scene {t1 - t0:.1f}s engine {t2 - t1:.1f}s nodes {sc.mesh.num_nodes}", flush=True)
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
peak = 6558.1
n = sc.mesh.num_nodes


def timed(fn, k, do_flush=True):
    out = []
    for _ in range(k):
        if do_flush:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        out.append((a, b))
    torch.cuda.synchronize()
    return np.array([a.elapsed_time(b) for a, b in out])


def run_pass(pid):
    return lambda: N.check(eng._lib.cs_run_pass(eng._handle, pid))


eng.step_frames(5)
torch.cuda.synchronize()
for name, pid, alg in (("force+integrate", N.PASS_FORCE_INTEGRATE, 48), ("normals", N.PASS_NORMALS, 24)):
    for fl in (True, False):
        t = timed(run_pass(pid), reps, fl)
        ms = np.median(t)
        print(f"  {name:16s} flush={fl!s:5s} median {ms * 1e3:8.1f} us  min {t.min() * 1e3:8.1f}  "
              f"alg {alg} B/node -> {alg * n / ms / 1e6:8.1f} GB/s = {alg * n / ms / 1e6 / peak:.3f} of {peak}",
              flush=True)
t = timed(lambda: eng.step(), reps, True)
print(f"  full step flush  median {np.median(t) * 1e3:8.1f} us  -> {1000 / np.median(t):.0f} steps/s", flush=True)
t = timed(lambda: eng.step(), reps, False)
print(f"  full step warm   median {np.median(t) * 1e3:8.1f} us  -> {1000 / np.median(t):.0f} steps/s", flush=True)
pos = eng.read_positions()
print("  finite", bool(np.isfinite(pos).all()), "max|x|", float(np.abs(pos).max()))
