"""Multi-process row bands on ONE device through the CUDA IPC link.

Two processes (gloo for the handle swap), both on cuda:0, each owning one
band linked with BandedEngine.link_ipc(); after 30 frames rank 0 compares the
gathered owned rows with a single engine, bit for bit.  This exercises the
same IPC + peer-store + flag-handshake path bench.py --gpus N uses across
GPUs (streams wait on flag words; no kernel waits on another).

    timeout 300 python tools/ipc_bands_smoke.py [n] [world] [obstacle, e.g. icosphere:3 | stream]

Collision-free bands do the seam handshake inside the step kernel (seam
warps spin on the neighbour's flag words); "stream" keeps the stream-memop
handshake.
"""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, n, q, obstacle, seam="kernel"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2507_11794_b200 as P
    from paper_2507_11794_b200.bands import BandedEngine
    from paper_2507_11794_b200.scenes import CONTACT_DT, NODE_MASS, stable_coefficients

    k, c = stable_coefficients(NODE_MASS, CONTACT_DT)
    params = P.SimParams(dt=CONTACT_DT, stiffness=k, damping=c)
    sc = None
    if obstacle:
        sc = P.build_scene(P.ScenarioConfig("drop", (n, n), obstacle=obstacle))
        params = sc.params
        band = BandedEngine(n, n, params, rank, world, exchange="p2p", mesh=sc.mesh,
                            obstacle=sc.obstacle, pair_budget=10**13)
    else:
        band = BandedEngine(n, n, params, rank, world, exchange="p2p", seam=seam)
    band.link_ipc()
    frames = 120 if obstacle else 30
    band.step(frames)
    pos = band.owned_positions()
    vel = band.owned_velocities()
    hits = band.engine.stats()["hit_counter"] if obstacle else 0
    out = [None] * world
    dist.all_gather_object(out, (pos, vel, hits))
    dist.barrier()
    band.close()
    if rank == 0:
        if obstacle:
            whole = P.Engine(sc.mesh, sc.obstacle, params, pair_budget=10**13)
        else:
            whole = P.Engine(P.build_scene(P.ScenarioConfig("hanging", (n, n), dt=CONTACT_DT)).mesh,
                             params=params)
        whole.step_frames(frames)
        gp = np.concatenate([o[0] for o in out])
        gv = np.concatenate([o[1] for o in out])
        ok = (np.array_equal(gp, whole.read_positions()) and
              np.array_equal(gv, whole.read_velocities()))
        if obstacle:
            total = whole.stats()["hit_counter"]
            ok = ok and total > 0 and sum(o[2] for o in out) == total
        q.put(("ok" if ok else "MISMATCH", float(np.abs(gp - whole.read_positions()).max())))
    dist.destroy_process_group()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    obstacle = sys.argv[3] if len(sys.argv) > 3 else None
    seam = "kernel"
    if obstacle == "stream":  # collision-free bands on the stream-memop handshake
        obstacle, seam = None, "stream"
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q, obstacle, seam)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    res = q.get(timeout=5)
    print("ipc bands", n, world, res)
    sys.exit(0 if res[0] == "ok" and all(p.exitcode == 0 for p in procs) else 1)


if __name__ == "__main__":
    main()
