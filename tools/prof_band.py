"""A self-linked middle band of C5 (in-kernel seam handshake, peer stores to
a dummy neighbour; tools/band_overhead.py) stepped a few frames, for ncu
captures of the BAND kernel.

    python tools/prof_band.py [world, default 8] [frames, default 4]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_11794_b200 as P
from paper_2507_11794_b200.bands import BandedEngine, HaloPlan
from paper_2507_11794_b200.scenes import CONTACT_DT, NODE_MASS, stable_coefficients

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4
kk, cc = stable_coefficients(NODE_MASS, CONTACT_DT)
params = P.SimParams(dt=CONTACT_DT, stiffness=kk, damping=cc)
me = BandedEngine(4096, 4096, params, 1, world, exchange="p2p", seam="kernel")
dummy = BandedEngine(4096, 4096, params, 1, world, exchange="p2p", seam="kernel")
mine, info = me.buffers(), dummy.buffers()
up = (dict(info, flags=mine["flags"] - 4), HaloPlan(4096, world, 0))
down = (dict(info, flags=mine["flags"] + 4), HaloPlan(4096, world, 2)) if world > 2 else None
me.link(up, down)
me.step(frames)
me.engine.synchronize()
print("ok")
