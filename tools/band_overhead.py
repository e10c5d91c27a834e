"""Per-frame cost of the row-band seam handshake, measured on ONE GPU.

A middle band of config 5 (rank 1 of N: both neighbours) is linked to a
dummy neighbour engine on the same device (its peer stores land there) with
its remote flag words pointing at its OWN flag words, so every stream wait
is satisfied by its own previous signal: the frame then pays the full
handshake machinery (stream memops, peer stores of the boundary rows,
system fences, no graph) but no cross-GPU latency and no neighbour skew.
Compared with the same band stepped as a plain engine (one graph replay per
frame).

    python tools/band_overhead.py [frames] [worlds, e.g. 2,4,8]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2507_11794_b200 as P
from paper_2507_11794_b200.bands import BandedEngine, HaloPlan
from paper_2507_11794_b200.scenes import CONTACT_DT, NODE_MASS, stable_coefficients

k = int(sys.argv[1]) if len(sys.argv) > 1 else 100
worlds = [int(w) for w in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 4, 8]
kk, cc = stable_coefficients(NODE_MASS, CONTACT_DT)
params = P.SimParams(dt=CONTACT_DT, stiffness=kk, damping=cc)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)


def timed(fn):
    fn(5)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    fn(k)
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k * 1e3


def self_linked(world, seam):
    """A middle band linked to a dummy neighbour; its remote flag words are
    its own, so every wait is satisfied by its own previous pass."""
    me = BandedEngine(4096, 4096, params, 1, world, stream=stream.cuda_stream, exchange="p2p",
                      seam=seam)
    dummy = BandedEngine(4096, 4096, params, 1, world, stream=stream.cuda_stream, exchange="p2p",
                         seam=seam)
    mine, info = me.buffers(), dummy.buffers()
    # link() aims the up signal at up.flags + 4 (the neighbour's from_dn) and
    # the down signal at down.flags + 0 (its from_up); shift both so they land
    # on my own block: up -> my word 0 (from_up), down -> my word 1 (from_dn)
    up = (dict(info, flags=mine["flags"] - 4), HaloPlan(4096, world, 0))
    down = (dict(info, flags=mine["flags"] + 4), HaloPlan(4096, world, 2)) if world > 2 else None
    me.link(up, down)
    return me, dummy


out = []
for world in worlds:
    rec = {"gpus": world}
    me = BandedEngine(4096, 4096, params, 1, world, stream=stream.cuda_stream, exchange="p2p")
    rec["local_rows"] = me.local_rows
    rec["plain_us"] = timed(lambda f: me.engine.step_frames(f))
    me.close()
    for seam in ("stream", "kernel"):
        me, dummy = self_linked(world, seam)
        rec[f"linked_{seam}_us"] = timed(lambda f: me.step(f))
        assert np.isfinite(me.owned_positions()).all()
        me.close()
        dummy.close()
    print(json.dumps(rec), flush=True)
    out.append(rec)
