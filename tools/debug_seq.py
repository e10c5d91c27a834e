"""Reproduce bench.py's engine sequence with a sync after every phase."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2507_11794_b200 as P

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
kernel = sys.argv[1] if len(sys.argv) > 1 else "pair"
for cfg in sys.argv[2:] or ["C2", "C5"]:
    sc = P.baseline_scene(cfg)
    eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, stream=stream.cuda_stream,
                   kernel=kernel)
    for f in range(5):
        eng.step()
        torch.cuda.synchronize()
        print(cfg, "frame", f, "ok", flush=True)
    eng.step_frames(20)
    torch.cuda.synchronize()
    print(cfg, "20 frames ok", np.isfinite(eng.read_positions()).all(), flush=True)
