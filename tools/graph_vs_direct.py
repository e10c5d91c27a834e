"""C2 frame time, L2 flushed between steps: CUDA-graph replay vs direct
launches of the same one-kernel frame (Engine(graph=False)).

    python tools/graph_vs_direct.py [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2507_11794_b200 as P

k = int(sys.argv[1]) if len(sys.argv) > 1 else 200
sc = P.baseline_scene("C2")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
flush = torch.empty(128 * 1024 * 1024, dtype=torch.float32, device="cuda")
for graph in (True, False, True, False):
    eng = P.Engine(sc.mesh, params=sc.params, stream=stream.cuda_stream, graph=graph)
    eng.step_frames(20)
    evs = []
    for _ in range(k):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.step_frames(1)
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    t = np.array([a.elapsed_time(b) for a, b in evs]) * 1e3
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    eng.step_frames(k)
    b.record(stream)
    torch.cuda.synchronize()
    print(f"graph={graph!s:5s} flushed mean {t.mean():6.2f} us median {np.median(t):6.2f}  "
          f"back-to-back {a.elapsed_time(b) * 1e3 / k:6.2f} us", flush=True)
    eng.close()
