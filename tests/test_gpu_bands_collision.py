"""GPU: row bands (several bands on one GPU, halos swapped by the same row
plans the NCCL path uses) and the full-size collision scene."""

import numpy as np
import pytest

import paper_2507_11794_b200 as P
from paper_2507_11794_b200.bands import BandedEngine
from paper_2507_11794_b200.scenes import CONTACT_DT, NODE_MASS, stable_coefficients

pytestmark = pytest.mark.gpu


def _swap(bands):
    """In-process equivalent of exchange_halos for bands on one device."""
    planes = [b.planes() for b in bands]
    for r in range(len(bands) - 1):
        up, dn = bands[r].plan, bands[r + 1].plan
        for q in range(6):
            a, b = up.send_down, dn.recv_up
            planes[r + 1][q][b[0]:b[1]].copy_(planes[r][q][a[0]:a[1]])
            a, b = dn.send_up, up.recv_down
            planes[r][q][b[0]:b[1]].copy_(planes[r + 1][q][a[0]:a[1]])


@pytest.mark.parametrize("world,precision", [(2, "fast"), (3, "fast"), (4, "fixed")])
def test_banded_run_is_bit_identical_to_one_engine(world, precision):
    import torch

    n = 160
    k, c = stable_coefficients(NODE_MASS, CONTACT_DT)
    params = P.SimParams(dt=CONTACT_DT, stiffness=k, damping=c)
    whole = P.Engine(P.baseline_scene("C2").mesh if n == 800 else
                     P.build_scene(P.ScenarioConfig("hanging", (n, n), dt=CONTACT_DT)).mesh,
                     params=params, precision=precision)
    bands = [BandedEngine(n, n, params, r, world) for r in range(world)]
    for b in bands:
        b.engine.close()
        b.engine = P.Engine(b.mesh, params=params, precision=precision)
    for _ in range(25):
        whole.step()
        for b in bands:
            b.engine.step()
        torch.cuda.synchronize()
        _swap(bands)
        torch.cuda.synchronize()
    got = np.concatenate([b.owned_positions() for b in bands])
    np.testing.assert_array_equal(got, whole.read_positions())


def _assert_diff_on_boundary(diff, mesh, obstacle, pos, tol=1e-6):
    """Every (node, triangle) pair in `diff` has a segment-triangle test whose
    predicate quantities lie within `tol` of a decision boundary
    (oracle.boundary_distance, tests/oracles.py:81-116)."""
    from oracle import oracle as O

    tris = np.asarray(mesh.triangles)
    ov, ot = obstacle.vertices, obstacle.triangles
    p64 = pos.astype(np.float64)
    for node, t in diff:
        cand = []
        for c in np.nonzero((tris == node).any(axis=1))[0]:
            a, b, d = tris[c]
            for u, w in ((a, b), (b, d), (d, a)):  # cloth edges through the node
                if node in (u, w):
                    cand.append(O.boundary_distance(p64[u], p64[w], *ov[ot[t]]))
            for s in range(3):  # obstacle edges of t vs this cloth triangle
                cand.append(O.boundary_distance(ov[ot[t][s]], ov[ot[t][(s + 1) % 3]],
                                                p64[a], p64[b], p64[d]))
        assert min(cand) < tol, (node, t, min(cand))


@pytest.mark.parametrize("spec", [("icosphere:2", (24, 24), 120), ("uvsphere:40x40", (64, 64), 90)])
def test_contact_set_matches_f64_solver_except_boundary_pairs(spec):
    """North-star contact gate: the (node, triangle) contact set of a GPU
    detect pass equals the float64 reference solver's (detect_all,
    collision.py:243-315) at the same positions, except pairs whose
    predicate quantities lie within 1e-6 of a decision boundary (no count
    allowance)."""
    from collections import Counter

    from oracle import oracle as O
    from paper_2507_11794_b200 import _native as N

    obstacle, grid, frames = spec
    sc = P.build_scene(P.ScenarioConfig("drop", grid, obstacle=obstacle))
    eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13)
    eng.step_frames(frames)
    eng.enable_contact_log(1 << 20)
    N.check(eng._lib.cs_run_pass(eng._handle, N.PASS_FORCE_INTEGRATE))
    pos = eng.read_positions()
    N.check(eng._lib.cs_run_pass(eng._handle, N.PASS_DETECT))
    gpu = Counter(map(tuple, eng.read_contacts().tolist()))
    so = O.SolverOracle(sc.mesh, sc.params, sc.obstacle)
    so.pos[...] = pos.astype(np.float64)
    O.set_threads(O.max_threads())
    hits, ref_arr = so.detect_contacts()
    ref = Counter(map(tuple, ref_arr.tolist()))
    assert hits > 0 and sum(ref.values()) > 0
    diff = (gpu - ref) + (ref - gpu)
    _assert_diff_on_boundary(diff, sc.mesh, sc.obstacle, pos, tol=1e-6)


def test_contact_set_at_c3_scale_against_the_solver_exact_fp64_engine():
    """The contact gate at full C3 size (316^2 cloth draped on the 99,904-
    triangle sphere): the fast engine's contact set against the float64
    engine's, which is bit-identical to the reference solver (golden
    trajectories with obstacles), at the same positions."""
    from collections import Counter

    from paper_2507_11794_b200 import _native as N

    sc = P.baseline_scene("C3")
    fast = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13)
    fast.step_frames(300)
    fast.enable_contact_log(1 << 22)
    N.check(fast._lib.cs_run_pass(fast._handle, N.PASS_FORCE_INTEGRATE))
    pos = fast.read_positions()
    N.check(fast._lib.cs_run_pass(fast._handle, N.PASS_DETECT))
    got = Counter(map(tuple, fast.read_contacts().tolist()))
    ref = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, precision="fp64")
    ref.write_state64(pos=pos.astype(np.float64))
    ref.enable_contact_log(1 << 22)
    N.check(ref._lib.cs_run_pass(ref._handle, N.PASS_DETECT))
    want = Counter(map(tuple, ref.read_contacts().tolist()))
    assert sum(want.values()) > 10_000
    diff = (got - want) + (want - got)
    _assert_diff_on_boundary(diff, sc.mesh, sc.obstacle, pos, tol=1e-6)


def test_c3_drapes_finite_with_contacts_in_both_modes():
    sc = P.baseline_scene("C3")
    hits = {}
    for precision in ("fast", "fixed"):
        eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, precision=precision)
        eng.step_frames(400)
        pos = eng.read_positions()
        assert np.isfinite(pos).all()
        hits[precision] = eng.stats()["hit_counter"]
        assert hits[precision] > 100_000
        # nobody tunnels far into the sphere (radius 0.3, margin 1e-3)
        r = np.linalg.norm(pos.astype(np.float64), axis=1)
        assert (r > 0.27).mean() > 0.999
    assert abs(hits["fast"] - hits["fixed"]) / hits["fixed"] < 0.05


@pytest.mark.parametrize("world,precision,n,normals,seam", [
    (2, "fast", 160, "auto", "kernel"), (3, "fast", 161, "auto", "kernel"),
    (3, "fast", 130, "split", "kernel"), (4, "fixed", 96, "auto", "kernel"),
    (2, "fast", 64, "fused", "kernel"), (3, "fast", 161, "auto", "stream"),
    (4, "fast", 300, "auto", "kernel"), (8, "fast", 300, "auto", "kernel"),
    (8, "fast", 97, "auto", "kernel"), (8, "fixed", 140, "auto", "kernel"),
])
def test_p2p_bands_bit_identical_to_one_engine(world, precision, n, normals, seam):
    """Row bands linked by peer stores inside the step kernel (the NVLink
    path of bench.py --gpus N), several bands on one device, each on its own
    stream: owned rows equal the single-engine run bit for bit (positions,
    velocities, normals).  Within ONE CUDA context a stream waiting on a flag
    that another stream of the same context has yet to write can stall the
    context, so this single-process test enqueues one frame per band and
    synchronises before the next (every wait is then already satisfied); the
    cross-process tests below exercise the real blocking handshake.  Fast
    collision-free bands do the handshake inside the step kernel (seam
    warps wait, graph-replayed frames: seam="kernel"); seam="stream" keeps
    the stream-memop handshake."""
    from paper_2507_11794_b200.bands import link_local

    k, c = stable_coefficients(NODE_MASS, CONTACT_DT)
    params = P.SimParams(dt=CONTACT_DT, stiffness=k, damping=c)
    whole = P.Engine(P.build_scene(P.ScenarioConfig("hanging", (n, n), dt=CONTACT_DT)).mesh,
                     params=params, precision=precision, normals=normals)
    bands = [BandedEngine(n, n, params, r, world, exchange="p2p", precision=precision,
                          normals=normals, seam=seam) for r in range(world)]
    link_local(bands)
    whole.step_frames(30)
    for _ in range(30):
        for b in bands:
            b.step(1)
        for b in bands:
            b.engine.synchronize()
    for what in ("positions", "velocities", "normals"):
        got = np.concatenate([getattr(b, f"owned_{what}")() for b in bands])
        np.testing.assert_array_equal(got, getattr(whole, f"read_{what}")(), err_msg=what)
    for b in bands:
        b.close()


def test_p2p_link_validation():
    from paper_2507_11794_b200 import _native as N  # noqa: F401
    from paper_2507_11794_b200.bands import link_local

    k, c = stable_coefficients(NODE_MASS, CONTACT_DT)
    params = P.SimParams(dt=CONTACT_DT, stiffness=k, damping=c)
    bands = [BandedEngine(64, 64, params, r, 2, exchange="p2p") for r in range(2)]
    with pytest.raises(RuntimeError):
        bands[0].step()  # not linked
    bands[0].engine.step()  # a frame before linking breaks lockstep parity
    with pytest.raises(ValueError):
        link_local(bands)


@pytest.mark.parametrize("n,world,obstacle", [(192, 2, None), (192, 3, "stream"),
                                              (48, 2, "icosphere:3"), (60, 3, "uvsphere:40x40")])
def test_ipc_linked_bands_across_processes(n, world, obstacle):
    """The multi-process link (CUDA IPC handles swapped over torch.distributed,
    as bench.py --gpus N does across GPUs), one process per band on one
    device, blocking flag handshake included.  With a replicated obstacle
    (collision across band seams) the owned rows stay
    bit-identical to one engine through contact and the bands' hit counts
    sum to its count."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "tools/ipc_bands_smoke.py", str(n), str(world)]
    if obstacle:
        cmd.append(obstacle)
    res = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=280)
    assert res.returncode == 0 and "'ok'" in res.stdout, res.stdout + res.stderr[-2000:]


def test_bench_gpus_2_under_torchrun_prints_one_banded_line():
    """The driver's N > 1 launch of bench.py (torchrun, one process per
    band, p2p halo stores + flag handshake) on this box -- functional only
    (both ranks may share one GPU): rank 0 prints one JSON line for config
    5 with the whole-job fields, and the sheet stays finite."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
           "--steps", "5", "--warmup", "3"]
    res = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=280)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["nodes"] == 4096 * 4096 and d["finite"]
    assert {"roofline", "e2e", "gpu_launches", "clocks"} <= set(d)


@pytest.mark.parametrize("world", [2, 3])
def test_fixed_bands_guard_rerun_bit_identical(world):
    """Reference-exact row bands whose springs all leave the exact kernel's
    guard (k = 1e7: forces far above 2^22 / scale), so every chunk -- seam
    chunks included, with their peer stores -- is recomputed by the builtin
    re-run (spring1x_ref); the owned rows still equal one engine bit for
    bit."""
    from paper_2507_11794_b200.bands import link_local

    params = P.SimParams(dt=CONTACT_DT, stiffness=1e7, damping=0.5)
    n = 70
    whole = P.Engine(P.build_scene(P.ScenarioConfig("hanging", (n, n), dt=CONTACT_DT)).mesh,
                     params=params, precision="fixed")
    bands = [BandedEngine(n, n, params, r, world, exchange="p2p", precision="fixed")
             for r in range(world)]
    link_local(bands)
    whole.step_frames(6)
    for _ in range(6):
        for b in bands:
            b.step(1)
        for b in bands:
            b.engine.synchronize()
    for what in ("positions", "velocities", "normals"):
        got = np.concatenate([getattr(b, f"owned_{what}")() for b in bands])
        np.testing.assert_array_equal(got, getattr(whole, f"read_{what}")(), err_msg=what)
    assert np.abs(whole.read_forces_raw()).max() > (1 << 22)  # the guard really failed
    for b in bands:
        b.close()
