"""One row band of config 5 (4096 x (4096/N + 4) rows) timed alone: the
compute part of an N-GPU frame (bench.py band_projection).

    CS_STRIP_ROWS=h python tools/band_sweep.py [N] [frames]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2507_11794_b200 as P
from paper_2507_11794_b200.mesh import grid_band

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
k = int(sys.argv[2]) if len(sys.argv) > 2 else 50
sc = P.baseline_scene("C1")  # params only (dt 0.004 stable coefficients)
rows = 4096 // n + 4
band = grid_band(4096, 4096, 0, rows, total_mass=0.05 * 4096 * 4096, pinned_rows="first")
band.positions = np.stack([band.positions[:, 0], -band.positions[:, 2],
                           np.zeros(len(band.positions))], axis=1)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng = P.Engine(band, params=sc.params, stream=stream.cuda_stream)
eng.step_frames(5)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record(stream)
eng.step_frames(k)
b.record(stream)
torch.cuda.synchronize()
print(f"N={n} rows={rows} h={os.environ.get('CS_STRIP_ROWS', 'model')}: "
      f"{a.elapsed_time(b) / k * 1e3:.1f} us/frame")
