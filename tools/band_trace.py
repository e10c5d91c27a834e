"""Per-warp timeline of one k_pair3 launch (diagnostic build with
-DCS_PAIR3_TRACE: tools/ab_build.py trace -DCS_PAIR3_TRACE, then
CLOTHSIM_LIB=.../var_trace.so): start / end spread, per-SM load and the
share of the launch that is ramp-up and tail.

    python tools/band_trace.py [world, default 8]  (a plain middle band of C5)
    python tools/band_trace.py 1                   (the whole sheet)
    python tools/band_trace.py 8 linked            (self-linked, in-kernel seam)
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2507_11794_b200 as P
from paper_2507_11794_b200 import _native as N
from paper_2507_11794_b200.bands import BandedEngine
from paper_2507_11794_b200.scenes import CONTACT_DT, NODE_MASS, stable_coefficients

world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
linked = len(sys.argv) > 2 and sys.argv[2] == "linked"
kk, cc = stable_coefficients(NODE_MASS, CONTACT_DT)
params = P.SimParams(dt=CONTACT_DT, stiffness=kk, damping=cc)
if world > 1 and linked:
    # the self-linked middle band of tools/band_overhead.py (in-kernel seam)
    from paper_2507_11794_b200.bands import HaloPlan
    me = BandedEngine(4096, 4096, params, 1, world, exchange="p2p", seam="kernel")
    dummy = BandedEngine(4096, 4096, params, 1, world, exchange="p2p", seam="kernel")
    mine, info = me.buffers(), dummy.buffers()
    up = (dict(info, flags=mine["flags"] - 4), HaloPlan(4096, world, 0))
    down = (dict(info, flags=mine["flags"] + 4), HaloPlan(4096, world, 2)) if world > 2 else None
    me.link(up, down)
    eng = me.engine
    me.step(20)
elif world > 1:
    eng = BandedEngine(4096, 4096, params, 1, world, exchange="p2p").engine
    eng.step_frames(20)
else:
    eng = P.Engine.from_grid(4096, 4096, params)
    eng.step_frames(20)
eng.synchronize()
lib = N.load()
raw = np.zeros((1 << 16) * 7, dtype=np.uint64)
lib.cs_debug_pair3_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
assert lib.cs_debug_pair3_trace(raw.ctypes.data, 1 << 16) == 0
buf = raw[: 3 << 16].reshape(-1, 3)
stamps = raw[3 << 16:].reshape(-1, 4)
t = buf[buf[:, 1] > 0]
t0 = t[:, 0].min()
start, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
sm, slot = t[:, 2] // 256, t[:, 2] % 256
dur = end - start
print(f"world {world}: {len(t)} warps, launch span {end.max():.2f} us")
print(f"  start: median {np.median(start):.2f}  p99 {np.percentile(start, 99):.2f}  max {start.max():.2f} us")
print(f"  end:   min {end.min():.2f}  median {np.median(end):.2f}  p99 {np.percentile(end, 99):.2f}  max {end.max():.2f} us")
print(f"  warp duration: min {dur.min():.2f}  median {np.median(dur):.2f}  max {dur.max():.2f} us")
per_sm = np.bincount(sm.astype(int))
print(f"  warps per SM: min {per_sm[per_sm > 0].min()}  max {per_sm.max()}  SMs used {np.count_nonzero(per_sm)}")
# per sub-partition (SMSP = warp slot % 4): warps sharing it and their end times
part = sm.astype(int) * 4 + (slot.astype(int) % 4)
load = np.bincount(part, minlength=int(part.max()) + 1)
print("  warps per SMSP:", dict(zip(*np.unique(load[load > 0], return_counts=True))))
for k in sorted(set(load[part])):
    sel = load[part] == k
    print(f"    SMSP with {k} warps: {sel.sum()} warps, end median {np.median(end[sel]):.2f} max {end[sel].max():.2f} us,"
          f" duration median {np.median(dur[sel]):.2f}")
strips = (4096 + 59) // 60
sy = np.nonzero(buf[:, 1] > 0)[0] // strips
for name, sel in (("seam chunk rows (sy 0, 1)", sy <= 1), ("interior", sy > 1)):
    if sel.any():
        print(f"  {name}: {sel.sum()} warps, duration median {np.median(dur[sel]):.2f} max {dur[sel].max():.2f},"
              f" end median {np.median(end[sel]):.2f} max {end[sel].max():.2f} us")
if linked:
    st = stamps[np.nonzero(buf[:, 1] > 0)[0]].astype(np.int64)
    rel = lambda a: (a - t[:, 0].astype(np.int64)) / 1e3
    w0, lp, ep, sg = rel(st[:, 0]), rel(st[:, 1]), rel(st[:, 2]), rel(st[:, 3])
    for name, sel in (("seam warps", sy <= 1), ("interior warps", sy > 1)):
        print(f"  {name} ({sel.sum()}), medians after their start: wait done {np.median(w0[sel]):.2f},"
              f" row loop done {np.median(lp[sel]):.2f}"
              + (f", epilogue done {np.median(ep[sel]):.2f}" if (st[sel, 2] > 0).all() else "")
              + f", signal done {np.median(sg[sel]):.2f} us")
# does the finish order on a sub-partition follow warp (block) order?
wid = np.nonzero(buf[:, 1] > 0)[0]
groups = {}
for w_, pi, e in zip(wid, part, end):
    groups.setdefault(int(pi), []).append((int(w_), float(e)))
same = total = 0
for g in groups.values():
    if len(g) == 3:
        total += 1
        by_id = [x[0] for x in sorted(g)]
        by_end = [x[0] for x in sorted(g, key=lambda x: x[1])]
        same += by_id == by_end
if total:
    print(f"  3-warp sub-partitions finishing in warp-id order: {same} of {total}")
    for rank in range(3):
        ids = [sorted(g)[rank][0] for g in groups.values() if len(g) == 3]
        ends_r = [sorted(g)[rank][1] for g in groups.values() if len(g) == 3]
        print(f"    id rank {rank}: mean warp id {np.mean(ids):7.1f}, mean end {np.mean(ends_r):6.2f} us")
ends = {}
for pi, e in zip(part, end):
    ends.setdefault(int(pi), []).append(float(e))
for k in (2, 3, 4, 5, 6):
    grp = [sorted(v) for v in ends.values() if len(v) == k]
    if grp:
        m = np.mean(np.array(grp), axis=0)
        print(f"    SMSPs with {k} warps ({len(grp)}): mean k-th end times " + ", ".join(f"{x:.2f}" for x in m))
busy = np.zeros(int(end.max() * 10) + 2)
for s_, e_ in zip(start, end):
    busy[int(s_ * 10):int(e_ * 10)] += 1
cap = busy.max()
print(f"  resident warps over time (0.1 us bins): peak {cap:.0f}; mean/peak {busy.mean() / cap:.3f}")
for q in (0.1, 0.25, 0.5, 0.75, 0.9, 1.0):
    i = int(q * (len(busy) - 1))
    print(f"    t={i / 10:6.2f} us  resident {busy[i]:.0f}")
