"""Multi-rank row bands on CPU: world_size 2 (and 3) over gloo.

Each rank steps its band (owned rows + 2-row halos) with the float64 oracle
and swaps halos through paper_2507_11794_b200.bands.exchange_halos -- the
same function the GPU ranks call over NCCL.  The owned rows must equal the
single-process solve bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_11794_b200.bands import HaloPlan, band_rows, exchange_halos, local_rows
from paper_2507_11794_b200.mesh import SimParams, generate_cloth_grid, grid_band

NX, NY, STEPS = 9, 17, 6


def _params():
    return SimParams(dt=0.004, stiffness=(468.75, 300.0, 120.0), damping=0.97)


def _rotate(mesh):
    rot = np.zeros_like(mesh.positions)
    rot[:, 0] = mesh.positions[:, 0]
    rot[:, 1] = -mesh.positions[:, 2]
    mesh.positions = rot
    return mesh


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O

    plan = HaloPlan(NY, world, rank)
    mesh = _rotate(grid_band(NX, NY, plan.l0, plan.l1, total_mass=0.05 * NX * NY,
                             pinned_rows="first"))
    so = O.SolverOracle(mesh, _params())
    pos, vel = torch.from_numpy(so.pos), torch.from_numpy(so.vel)
    rows = plan.l1 - plan.l0
    planes = [pos[:, q].view(rows, NX) for q in range(3)] + [vel[:, q].view(rows, NX) for q in range(3)]
    for _ in range(STEPS):
        so.step(normals=False)
        exchange_halos(planes, plan)
    a, b = (plan.j0 - plan.l0) * NX, (plan.j1 - plan.l0) * NX
    out[rank] = (so.pos[a:b].copy(), so.vel[a:b].copy())
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_banded_solve_equals_single_process(world):
    from oracle import oracle as O

    full = _rotate(generate_cloth_grid(NX, NY, total_mass=0.05 * NX * NY, pinned_rows="first"))
    ref = O.SolverOracle(full, _params())
    for _ in range(STEPS):
        ref.step(normals=False)
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        got = dict(out)
    pos = np.concatenate([got[r][0] for r in range(world)])
    vel = np.concatenate([got[r][1] for r in range(world)])
    np.testing.assert_array_equal(pos, ref.pos)
    np.testing.assert_array_equal(vel, ref.vel)


def test_band_partition_covers_grid():
    for ny in (4, 17, 4096):
        for world in (1, 2, 3, 8):
            if ny < 2 * world:
                continue
            rows = [band_rows(ny, world, r) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == ny
            assert all(rows[r][1] == rows[r + 1][0] for r in range(world - 1))
            for r in range(world):
                l0, l1 = local_rows(ny, world, r)
                assert l0 == max(0, rows[r][0] - 2) and l1 == min(ny, rows[r][1] + 2)


def test_grid_band_matches_global_grid_rows():
    g = generate_cloth_grid(7, 11, 1.3, 0.9, total_mass=0.05 * 77, pinned_rows="first")
    b = grid_band(7, 11, 3, 9, 1.3, 0.9, total_mass=0.05 * 77, pinned_rows="first")
    np.testing.assert_array_equal(b.positions, g.positions[3 * 7:9 * 7])
    np.testing.assert_array_equal(b.masses, g.masses[3 * 7:9 * 7])
    assert set(np.unique(b.spring_rest_lengths.astype(np.float32))) <= \
        set(np.unique(g.spring_rest_lengths.astype(np.float32)))


@pytest.mark.parametrize("ny,world", [(64, 2), (97, 3), (4096, 8), (10, 4)])
def test_peer_rows_land_on_the_neighbours_halo(ny, world):
    """The p2p link (bands.peer_rows): the local rows a band stores into each
    neighbour are exactly the global rows that neighbour's halo holds."""
    from paper_2507_11794_b200.bands import peer_rows

    plans = [HaloPlan(ny, world, r) for r in range(world)]
    for r, me in enumerate(plans):
        for direction, q in (("up", r - 1), ("down", r + 1)):
            if not 0 <= q < world:
                continue
            nb = plans[q]
            src, dst, rows = peer_rows(me, nb, direction)
            assert rows == 2
            assert me.j0 <= me.l0 + src and me.l0 + src + rows <= me.j1  # owned rows
            assert me.l0 + src == nb.l0 + dst  # same global rows
            halo = nb.recv_down if direction == "up" else nb.recv_up
            assert (dst, dst + rows) == halo
