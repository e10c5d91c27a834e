"""C3 frame time vs broad-phase cell size and narrow-phase mapping
(drape 200 frames, time 200)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2507_11794_b200 as P

sc = P.baseline_scene(sys.argv[1] if len(sys.argv) > 1 else "C3")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
for narrow in ("warp", "thread"):
    for cs in [0.0, 0.003, 0.0045, 0.006, 0.009]:
        eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13,
                       stream=stream.cuda_stream, cell_size=cs or None, narrow=narrow)
        eng.step_frames(200)
        torch.cuda.synchronize()
        h0 = eng.stats()["hit_counter"]
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.step_frames(200)
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 200
        bp = eng.broadphase_stats()
        print(f"{narrow:6s} cell={cs or 'auto'} {ms * 1000:.1f} us/frame ({1000 / ms:.0f} steps/s) "
              f"cells={bp['cells']} refs={bp['refs']} "
              f"hits/frame={(eng.stats()['hit_counter'] - h0) / 200:.0f}", flush=True)
        eng.close()
