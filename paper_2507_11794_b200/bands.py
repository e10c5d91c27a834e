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

Because each node's force sums the same springs in the same program order
whatever band it sits in, a banded run is bit-identical to the single-GPU
run (tests/test_bands_gloo.py checks the exchange on CPU; the GPU test steps
several bands in one process).  The obstacle (if any) would be replicated per
rank; collision across band seams is not implemented in this round.
"""

from __future__ import annotations

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
                 height=1.0, node_mass=0.05, pinned_rows="first"):
        from .engine import Engine
        from .mesh import grid_band

        self.plan = HaloPlan(ny, world, rank)
        self.nx, self.ny = nx, ny
        mesh = grid_band(nx, ny, self.plan.l0, self.plan.l1, width, height,
                         total_mass=node_mass * nx * ny, pinned_rows=pinned_rows)
        rot = np.zeros_like(mesh.positions)  # scenes._rotate_xz_to_xy
        rot[:, 0] = mesh.positions[:, 0]
        rot[:, 1] = -mesh.positions[:, 2]
        mesh.positions = rot
        self.mesh = mesh
        self.engine = Engine(mesh, params=params, stream=stream)
        self.group = group
        self.local_rows = self.plan.l1 - self.plan.l0

    def planes(self):
        import torch

        out = []
        for q in range(6):
            ptr, pitch = self.engine.state_plane(q)
            out.append(torch.as_tensor(_CudaPlane(ptr, self.local_rows, pitch), device="cuda"))
        return out

    def step(self):
        self.engine.step()
        exchange_halos(self.planes(), self.plan, self.group)

    def owned_positions(self):
        p = self.engine.read_positions()
        a = (self.plan.j0 - self.plan.l0) * self.nx
        b = (self.plan.j1 - self.plan.l0) * self.nx
        return p[a:b]


def run_banded_bench(args, metric):
    """bench.py for N > 1 (torchrun): config 5 split in row bands, one per GPU;
    value = whole-job steps/s, timed with CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from .scenes import CONTACT_DT, NODE_MASS, stable_coefficients
    from .mesh import SimParams

    n = 4096
    k, c = stable_coefficients(NODE_MASS, CONTACT_DT)
    params = SimParams(dt=CONTACT_DT, stiffness=k, damping=c)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    band = BandedEngine(n, n, params, rank, world, stream=stream.cuda_stream)
    for _ in range(args.warmup):
        band.step()
    torch.cuda.synchronize()
    dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.steps):
        band.step()
    b.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([a.elapsed_time(b) / args.steps], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    if rank == 0:
        line = {
            "metric": metric, "value": 1000.0 / ms, "unit": "steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (hanging 4096^2, dt 0.004)",
            "config": {"workload": "C5: 4096x4096 hanging cloth, row bands + 2-row NCCL halos",
                       "nodes": n * n, "parallelism": f"rowband{world}",
                       "l2": "inputs (16.8M nodes, 805 MB/step) larger than L2"},
            "node_updates_per_s": 1000.0 / ms * n * n,
            "gpu_launches": args.steps * band.engine.kernels_per_frame,
        }
        print(json.dumps(line))
    dist.destroy_process_group()
