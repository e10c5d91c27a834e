"""Run a few frames of a baseline config with a chosen kernel variant
(for ncu captures):  python tools/run_frames.py C5 strip 3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_11794_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
kernel = sys.argv[2] if len(sys.argv) > 2 else "strip"
frames = int(sys.argv[3]) if len(sys.argv) > 3 else 3
precision = sys.argv[4] if len(sys.argv) > 4 else "fast"
sc = P.baseline_scene(cfg)
eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, kernel=kernel,
               precision=precision, graph=False)
eng.step_frames(frames)
eng.synchronize()
print("ok", cfg, kernel, frames, eng.read_positions()[:1])
