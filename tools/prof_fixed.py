"""Reference-exact (fixed) mode passes at a config, for ncu captures.
    python tools/prof_fixed.py C2 [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2507_11794_b200 as P
from paper_2507_11794_b200 import _native as N

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sc = P.baseline_scene(cfg)
eng = P.Engine(sc.mesh, params=sc.params, precision="fixed")
eng.step_frames(3)
for _ in range(reps):
    N.check(eng._lib.cs_run_pass(eng._handle, N.PASS_FORCE_INTEGRATE))
    N.check(eng._lib.cs_run_pass(eng._handle, N.PASS_NORMALS))
eng.synchronize()
print("ok")
