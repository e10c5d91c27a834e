"""Split vs fused frame pieces on a plain middle band of C5 (no links):
the fused frame (k_pair3<NORMALS=1>), the force pass alone (k_pair3<0>)
and the stand-alone normals pass (k_pair_normals), each timed back to back.

    python tools/band_split.py [world, default 8] [reps, default 200]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2507_11794_b200 as P
from paper_2507_11794_b200 import _native as N
from paper_2507_11794_b200.bands import BandedEngine
from paper_2507_11794_b200.scenes import CONTACT_DT, NODE_MASS, stable_coefficients

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
k = int(sys.argv[2]) if len(sys.argv) > 2 else 200
kk, cc = stable_coefficients(NODE_MASS, CONTACT_DT)
params = P.SimParams(dt=CONTACT_DT, stiffness=kk, damping=cc)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng = BandedEngine(4096, 4096, params, 1, world, exchange="p2p", stream=stream.cuda_stream).engine


def timed(fn):
    fn(5)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    fn(k)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k * 1e3


def passes(pid):
    def run(n):
        for _ in range(n):
            N.check(eng._lib.cs_run_pass(eng._handle, pid))
    return run


print(f"world {world}: fused frame {timed(lambda n: eng.step_frames(n)):.1f} us, "
      f"force pass {timed(passes(N.PASS_FORCE_INTEGRATE)):.1f} us, "
      f"normals pass {timed(passes(N.PASS_NORMALS)):.1f} us")
