"""C2 per-step time (L2 flushed between steps): graph replay vs eager launch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2507_11794_b200 as P

sc = P.baseline_scene(sys.argv[1] if len(sys.argv) > 1 else "C2")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
for graph in (True, False):
    eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, stream=stream.cuda_stream,
                   graph=graph)
    eng.step_frames(10)
    ts = []
    for _ in range(100):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.step()
        b.record(stream)
        ts.append((a, b))
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) for a, b in ts]) * 1e3
    print(f"graph={graph}: median {np.median(t):.1f} us  min {t.min():.1f}")
    eng.close()
