"""Row-band partition of one cloth across ranks (BASELINE config 5).

The grid's flat index j*nx+i makes a band of rows contiguous.  Rank r owns
rows [j0, j1) and keeps a 2-row halo on each side, because bend springs reach
two rows (mesh.py:284-289) and damping reads neighbour velocities
(solver.py:117-119) -- the halo carries positions AND velocities (SURVEY.md
finding 3).  Per frame:

  1. every rank steps its local sheet (owned rows + halos) on its GPU;
  2. owned boundary rows are exchanged: rows [j0, j0+2) go to rank-1's
     bottom halo, rows [j1-2, j1) to rank+1's top halo (torch.distributed
     point-to-point: NCCL over NVLink on GPUs, gloo on CPU tensors).

Two exchange mechanisms:

* ``exchange="p2p"`` (default on GPUs): step 2 disappears into step 1.  The
  step kernel stores each boundary row straight into the neighbour's halo
  (peer memory over NVLink; CUDA IPC handles are swapped once through
  torch.distributed), and a stream-ordered handshake (cuStreamWaitValue32 /
  cuStreamWriteValue32 on per-neighbour flag words) orders the passes -- no
  NCCL call, no packing kernel, no host synchronisation per frame
  (cs_set_halo_peers in include/clothsim_b200.h).
* ``exchange="nccl"``: torch.distributed point-to-point after each step
  (``exchange_halos``), the plain baseline; also what the CPU gloo tests run.

Because each node's force sums the same springs in the same program order
whatever band it sits in, a banded run is bit-identical to the single-GPU
run (tests/test_bands_gloo.py checks the exchange plans on CPU; the GPU
tests link several bands in one process).  The obstacle (if any) would be
replicated per rank.  Every band detects over its local sheet (owned rows +
halo), but accumulates contacts only into its owned nodes and counts a hit
only when the primitive's minimum node is owned, so positions stay
bit-identical and the bands' hit counts sum to one engine's.
"""

from __future__ import annotations

import ctypes
import json
import os
import time

import numpy as np

HALO = 2  # rows


def band_rows(ny: int, world: int, rank: int):
    """Owned rows [j0, j1) of `rank` -- contiguous, as even as possible."""
    base, extra = divmod(ny, world)
    j0 = rank * base + min(rank, extra)
    j1 = j0 + base + (1 if rank < extra else 0)
    return j0, j1


def local_rows(ny: int, world: int, rank: int, halo: int = HALO):
    """Rows [l0, l1) held locally (owned + halo, clipped to the grid)."""
    j0, j1 = band_rows(ny, world, rank)
    return max(0, j0 - halo), min(ny, j1 + halo)


class HaloPlan:
    """Which local rows are sent to / received from each neighbour."""

    def __init__(self, ny: int, world: int, rank: int, halo: int = HALO):
        self.rank, self.world, self.halo = rank, world, halo
        self.j0, self.j1 = band_rows(ny, world, rank)
        self.l0, self.l1 = local_rows(ny, world, rank, halo)
        # local row indices (relative to l0)
        self.up = rank - 1 if rank > 0 else None
        self.down = rank + 1 if rank + 1 < world else None
        self.send_up = (self.j0 - self.l0, self.j0 - self.l0 + halo)           # my first owned rows
        self.recv_up = (0, self.j0 - self.l0)                                  # my top halo
        self.send_down = (self.j1 - self.l0 - halo, self.j1 - self.l0)         # my last owned rows
        self.recv_down = (self.j1 - self.l0, self.l1 - self.l0)                # my bottom halo


def peer_rows(me: HaloPlan, nbr: HaloPlan, direction: str):
    """(src_row0, dst_row0, rows): my local rows stored into neighbour `nbr`'s
    halo -- `direction` "up" for rank-1 (my first owned rows -> its bottom
    halo), "down" for rank+1 (my last owned rows -> its top halo)."""
    if direction == "up":
        src, dst = me.send_up, nbr.recv_down
    elif direction == "down":
        src, dst = me.send_down, nbr.recv_up
    else:
        raise ValueError(direction)
    if src[1] - src[0] != dst[1] - dst[0]:
        raise ValueError("halo plans of neighbouring bands disagree")
    return src[0], dst[0], src[1] - src[0]


def exchange_halos(planes, plan: HaloPlan, group=None):
    """Swap halo rows with the neighbouring ranks.

    `planes` is a list of 2-D tensors (rows x pitch), one per state component
    (x, y, z, vx, vy, vz), on any device torch.distributed supports for the
    active backend.  Rows are packed into one contiguous buffer per
    direction so each neighbour pair needs a single send and a single recv.
    """
    import torch
    import torch.distributed as dist

    ops, recvs = [], []

    def pack(rows):
        return torch.cat([p[rows[0]:rows[1]].reshape(-1) for p in planes])

    if plan.up is not None:
        ops.append(dist.P2POp(dist.isend, pack(plan.send_up).contiguous(), plan.up, group))
        buf = torch.empty((plan.recv_up[1] - plan.recv_up[0]) * planes[0].shape[1] * len(planes),
                          dtype=planes[0].dtype, device=planes[0].device)
        ops.append(dist.P2POp(dist.irecv, buf, plan.up, group))
        recvs.append((plan.recv_up, buf))
    if plan.down is not None:
        ops.append(dist.P2POp(dist.isend, pack(plan.send_down).contiguous(), plan.down, group))
        buf = torch.empty((plan.recv_down[1] - plan.recv_down[0]) * planes[0].shape[1] * len(planes),
                          dtype=planes[0].dtype, device=planes[0].device)
        ops.append(dist.P2POp(dist.irecv, buf, plan.down, group))
        recvs.append((plan.recv_down, buf))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for rows, buf in recvs:
        nrow = rows[1] - rows[0]
        chunks = buf.view(len(planes), nrow, planes[0].shape[1])
        for q, p in enumerate(planes):
            p[rows[0]:rows[1]].copy_(chunks[q])


class _CudaPlane:
    """__cuda_array_interface__ wrapper for one engine state plane."""

    def __init__(self, ptr, rows, pitch):
        self.__cuda_array_interface__ = {
            "shape": (rows, pitch), "typestr": "<f4", "data": (ptr, False), "version": 3,
            "strides": None,
        }


class BandedEngine:
    """One rank's band of a hanging cloth (scenes.baseline_scene('C5') split
    in rows), stepped on this rank's GPU, halos exchanged over NCCL."""

    def __init__(self, nx, ny, params, rank, world, group=None, stream=None, width=1.0,
                 height=1.0, node_mass=0.05, pinned_rows="first", exchange="nccl",
                 precision="fast", mesh=None, obstacle=None, **engine_kw):
        """A band of the hanging nx x ny cloth (BASELINE config 5), or -- with
        `mesh` -- of any grid ClothMesh (e.g. a drop scene) with the static
        `obstacle` replicated on every band."""
        from .engine import Engine, _grid_stencil_rest
        from .mesh import band_of_mesh, grid_band

        if exchange not in ("nccl", "p2p"):
            raise ValueError("exchange must be 'nccl' or 'p2p'")
        self.exchange = exchange
        self.linked = False
        self._opened = []
        self.plan = HaloPlan(ny, world, rank)
        self.nx, self.ny = nx, ny
        if mesh is None and obstacle is None and precision in ("fast", "fixed"):
            # the hanging cloth's band generated on the device (cs_create_grid):
            # no per-node or per-spring host array, even at 4096^2
            self.engine = Engine.from_grid(nx, ny, params, width=width, height=height,
                                           total_mass=node_mass * nx * ny,
                                           pinned_rows=pinned_rows, orientation="hanging",
                                           row_lo=self.plan.l0, row_hi=self.plan.l1,
                                           stream=stream, precision=precision, **engine_kw)
            self.mesh = self.engine.mesh
        else:
            if mesh is not None:
                stencil = _grid_stencil_rest(mesh)
                if stencil is None or (stencil[0], stencil[1]) != (nx, ny):
                    raise ValueError("row bands need an nx x ny grid mesh with uniform spring "
                                     "families")
                band = band_of_mesh(mesh, nx, ny, stencil[2], self.plan.l0, self.plan.l1)
            else:
                band = grid_band(nx, ny, self.plan.l0, self.plan.l1, width, height,
                                 total_mass=node_mass * nx * ny, pinned_rows=pinned_rows)
                rot = np.zeros_like(band.positions)  # scenes._rotate_xz_to_xy
                rot[:, 0] = band.positions[:, 0]
                rot[:, 1] = -band.positions[:, 2]
                band.positions = rot
            self.mesh = band
            self.engine = Engine(band, obstacle, params=params, stream=stream,
                                 precision=precision, **engine_kw)
        self.group = group
        self.local_rows = self.plan.l1 - self.plan.l0

    # ---- p2p linking ---------------------------------------------------------
    def buffers(self):
        """Device pointers of this band's state buffers and flag words."""
        from . import _native as N

        s0, s1, fl = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        plane, pitch = ctypes.c_int64(), ctypes.c_int64()
        N.check(self.engine._lib.cs_state_buffers(self.engine._handle, ctypes.byref(s0),
                                                  ctypes.byref(s1), ctypes.byref(fl),
                                                  ctypes.byref(plane), ctypes.byref(pitch)))
        return {"state": (s0.value, s1.value), "flags": fl.value, "plane": plane.value,
                "pitch": pitch.value}

    def link(self, up=None, down=None):
        """Make the step kernel store boundary rows into the neighbours.

        `up` / `down` are ``(buffers_dict, HaloPlan)`` of rank-1 / rank+1 with
        pointers valid in this process (same device, or opened IPC handles)."""
        from . import _native as N

        def peer(nb, direction):
            if nb is None:
                return None
            info, nplan = nb
            src, dst, rows = peer_rows(self.plan, nplan, direction)
            p = N.CsHaloPeer()
            p.state[0], p.state[1] = info["state"]
            p.plane, p.src_row0, p.dst_row0, p.rows = info["plane"], src, dst, rows
            # the neighbour's flag word 1 is written by its lower neighbour
            # (me, when it is above me), word 0 by its upper neighbour
            p.remote_flag = info["flags"] + 4 * (1 if direction == "up" else 0)
            return p

        pu, pd = peer(up, "up"), peer(down, "down")
        lo, hi = self.plan.j0 - self.plan.l0, self.plan.j1 - self.plan.l0
        N.check(self.engine._lib.cs_set_halo_peers(
            self.engine._handle, lo, hi, ctypes.byref(pu) if pu else None,
            ctypes.byref(pd) if pd else None))
        self.linked = True

    def link_ipc(self):
        """Multi-process linking: swap CUDA IPC handles of the state buffers and
        flag words with the neighbouring ranks over torch.distributed."""
        import torch.distributed as dist

        from . import _native as N

        lib = self.engine._lib
        info = self.buffers()

        def export(ptr):
            buf = ctypes.create_string_buffer(64)
            N.check(lib.cs_ipc_export(ptr, buf))
            return buf.raw

        mine = {"rank": self.plan.rank, "plane": info["plane"], "ny": self.plan.l1,
                "h": [export(info["state"][0]), export(info["state"][1]), export(info["flags"])]}
        allinfo = [None] * self.plan.world
        dist.all_gather_object(allinfo, mine, group=self.group)

        def open_nbr(r):
            if r is None:
                return None
            ptrs = []
            for hbytes in allinfo[r]["h"]:
                p = ctypes.c_void_p()
                N.check(lib.cs_ipc_open(hbytes, ctypes.byref(p)))
                self._opened.append(p.value)
                ptrs.append(p.value)
            nplan = HaloPlan(self.ny, self.plan.world, r)
            return ({"state": (ptrs[0], ptrs[1]), "flags": ptrs[2],
                     "plane": allinfo[r]["plane"]}, nplan)

        self.link(open_nbr(self.plan.up), open_nbr(self.plan.down))
        dist.barrier(group=self.group)  # every band linked before anyone steps

    def close(self):
        from . import _native as N

        self.engine.synchronize()
        for p in self._opened:
            N.check(self.engine._lib.cs_ipc_close(p))
        self._opened = []
        self.engine.close()

    def planes(self):
        import torch

        out = []
        for q in range(6):
            ptr, pitch = self.engine.state_plane(q)
            out.append(torch.as_tensor(_CudaPlane(ptr, self.local_rows, pitch), device="cuda"))
        return out

    def step(self, frames=1):
        if self.exchange == "p2p":
            if not self.linked:
                raise RuntimeError("p2p bands must be linked (link / link_ipc) before stepping")
            self.engine.step_frames(frames)  # halos travel inside the step kernels
            return
        for _ in range(frames):
            self.engine.step()
            exchange_halos(self.planes(), self.plan, self.group)

    def _owned(self, arr):
        a = (self.plan.j0 - self.plan.l0) * self.nx
        b = (self.plan.j1 - self.plan.l0) * self.nx
        return arr[a:b]

    def owned_positions(self):
        return self._owned(self.engine.read_positions())

    def owned_velocities(self):
        return self._owned(self.engine.read_velocities())

    def owned_normals(self):
        return self._owned(self.engine.read_normals())


def link_local(bands):
    """Link the bands of one process (one device) for p2p stepping."""
    info = [b.buffers() for b in bands]
    for r, b in enumerate(bands):
        up = (info[r - 1], bands[r - 1].plan) if r > 0 else None
        down = (info[r + 1], bands[r + 1].plan) if r + 1 < len(bands) else None
        b.link(up, down)


def run_banded_bench(args, metric, clock_sampler=None, peak=None):
    """bench.py for N > 1 (torchrun): config 5 split in row bands, one per GPU;
    value = whole-job steps/s, timed with CUDA events, max over ranks; e2e =
    the same through Engine.write_* + Engine.simulate with host buffers."""
    import contextlib

    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    exchange = os.environ.get("CLOTHSIM_BAND_EXCHANGE", "p2p")
    # one GPU per rank; with fewer devices than ranks (a functional run on a
    # single-GPU box) ranks share devices -- each rank is its own process and
    # CUDA context, which the flag handshake requires
    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev
    torch.cuda.set_device(dev)
    if exchange == "p2p" and ndev > 1:
        # peer stores need load/store access to the neighbours' GPUs (NVLink /
        # NVSwitch); without it the bands exchange halos over NCCL instead
        # (every rank evaluates the same machine-wide condition, so all pick
        # the same mode)
        pairs = [(r % ndev, (r + 1) % ndev) for r in range(world - 1)]
        if not all(a == b or torch.cuda.can_device_access_peer(a, b) for a, b in pairs):
            exchange = "nccl"
    if exchange == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    else:  # the data path is peer stores: the process group only swaps IPC handles
        dist.init_process_group("gloo")
    red_dev = "cuda" if exchange == "nccl" else "cpu"
    from .engine import pinned_empty
    from .mesh import SimParams
    from .scenes import CONTACT_DT, NODE_MASS, stable_coefficients

    n = 4096
    k, c = stable_coefficients(NODE_MASS, CONTACT_DT)
    params = SimParams(dt=CONTACT_DT, stiffness=k, damping=c)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    band = BandedEngine(n, n, params, rank, world, stream=stream.cuda_stream, exchange=exchange)
    if exchange == "p2p":
        band.link_ipc()
    band.step(args.warmup)
    torch.cuda.synchronize()
    dist.barrier()
    slowdowns = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    attempts = []
    for attempt in range(2):  # a throttled timed region is measured once more
        sampler = clock_sampler(dev) if (clock_sampler and rank == 0) else contextlib.nullcontext()
        with sampler as clk:
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            band.step(args.steps)
            b.record(stream)
            torch.cuda.synchronize()
        dist.barrier()
        again = torch.zeros(1, dtype=torch.float64, device=red_dev)
        if clock_sampler and rank == 0:
            attempts.append({"rank0_ms_per_step": a.elapsed_time(b) / args.steps,
                             "clocks": clk.summary()})
            if set(clk.summary()["reasons"]) & slowdowns:
                again[0] = 1.0
        dist.broadcast(again, src=0)
        if attempt == 1 or not again.item():
            break
    finite = bool(np.isfinite(band.owned_positions()).all())

    def max_over_ranks(v):
        t = torch.tensor([v], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = max_over_ranks(a.elapsed_time(b) / args.steps)

    # end to end with host buffers: upload this band's state from pinned
    # memory, then Engine.simulate streams every frame's positions back
    nloc = band.mesh.num_nodes
    k_e2e = max(3, min(args.steps, 10))
    host_pos = pinned_empty((nloc, 3))
    host_vel = pinned_empty((nloc, 3))
    host_pos[...] = band.engine.read_positions()
    host_vel[...] = band.engine.read_velocities()
    traj = pinned_empty((k_e2e, nloc, 3))
    dist.barrier()
    t0 = time.perf_counter()
    band.engine.write_positions(host_pos)
    band.engine.write_velocities(host_vel)
    if exchange == "p2p":
        # the halo exchange travels inside the step kernels: simulate()
        # streams every frame's positions while the next frame computes
        band.engine.simulate(k_e2e, out=traj)
    else:
        # NCCL exchange: the engine alone would step stale halos, so each
        # frame is the band's step + halo swap, then its positions D2H
        for f in range(k_e2e):
            band.step(1)
            band.engine.read_positions(out=traj[f])
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    del traj

    owned = (band.plan.j1 - band.plan.j0) * n
    frame_bytes = 60 * owned  # fused k_pair3: 24 B read + 24 B + 12 B normals written per node
    achieved = frame_bytes / (ms * 1e-3) / 1e9  # rank 0's band kernel (all ranks equal size)
    if rank == 0:
        line = {
            "metric": metric, "value": 1000.0 / ms, "unit": "steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (hanging 4096^2, dt 0.004)",
            "config": {"workload": "C5: 4096x4096 hanging cloth, row bands with 2-row halos",
                       "nodes": n * n, "parallelism": f"rowband{world}",
                       "halo_exchange": ("peer stores inside the step kernel + stream-ordered "
                                         "flag handshake (CUDA IPC over NVLink)"
                                         if exchange == "p2p" else
                                         "torch.distributed NCCL send/recv after each step"),
                       "l2": "inputs (16.8M nodes, 805 MB/step) larger than L2",
                       "scaling_baseline": ("the same C5 workload on 1 GPU is roofline_c5."
                                            "steps_per_s in the N=1 line, whose headline "
                                            "value is C2 (the metric's named config)")},
            "node_updates_per_s": 1000.0 / ms * n * n,
            "roofline": {"bound": "hbm", "kernel": "k_pair3<NORMALS=1> on rank 0's band",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if peak else None, "traffic": None,
                         "bytes_per_launch": frame_bytes, "bytes_per_node": 60,
                         "launch_ms": ms},
            "e2e": {"value": k_e2e / e2e_s, "unit": "steps/s",
                    "h2d_bytes_per_step": int(24 * n * n / k_e2e), "d2h_bytes_per_step": 12 * n * n,
                    "api": ("Engine.write_positions/write_velocities + Engine.simulate per band"
                            if exchange == "p2p" else
                            "Engine.write_positions/write_velocities + per frame BandedEngine.step "
                            "(step + NCCL halo swap) + Engine.read_positions"),
                    "frames": k_e2e},
            "gpu_launches": args.steps * band.engine.kernels_per_frame * world,
            "finite": finite,
            "devices": torch.cuda.device_count(),
        }
        if clock_sampler:
            line["clocks"] = dict(clk.summary(), remeasured=attempt)
            line["attempts"] = attempts
        if torch.cuda.device_count() < world:
            line["note"] = (f"{world} ranks shared {torch.cuda.device_count()} GPU(s): a "
                            "functional run, not a scaling measurement")
        print(json.dumps(line))
    if exchange == "p2p":
        band.close()
    dist.destroy_process_group()
