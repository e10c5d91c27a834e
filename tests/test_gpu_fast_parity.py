"""GPU: the default fast mode against the CPU oracle, clause by clause of the
north star (BASELINE.json):

* bit-exact grid-cell assignment -- the device-built broad phase equals the
  numpy float32 restatement (oracle.broadphase_grid) reference by reference;
* the fast kernel's OWN forces (k_pair3, not a reference-arithmetic
  recompute) against the f64 solver: from the velocity change of one step,
  and through read_forces_raw (k_pair3's read-only forces mode);
* springs shorter than 1e-12 apply no force (solver.py:111-113);
* the (node, triangle) contact set at C4 size equals the f64 solver's except
  pairs within 1e-6 of a predicate boundary, with no count allowance;
* a C3 frame's detect pass bit-identical to the CPU engine oracle;
* the C1 100-step drift bounded by the reference float32 engine's own drift
  (tests/golden/c1_drift.npz);
* the golden drop / pull / flags scenes (substeps, explicit Euler, raw
  response, ext accel) within tolerance of the f64 solver.
"""

from collections import Counter

import numpy as np
import pytest

from conftest import TRAJ, load_golden, mesh_from_golden, obstacle_from_golden, params_from_golden
from oracle import oracle as O

import paper_2507_11794_b200 as P
from paper_2507_11794_b200 import SimParams, generate_cloth_grid

pytestmark = pytest.mark.gpu
SCALE = 1 << 16


def _extent(mesh):
    p = np.asarray(mesh.positions)
    return float((p.max(axis=0) - p.min(axis=0)).max())


# ---- broad phase: bit-exact grid-cell assignment -------------------------------------

@pytest.mark.parametrize("scene,cell", [("C4", None), ("C4", 0.004), ("ico2", None),
                                        ("ico2", 0.02), ("ico2", 0.003)])
def test_broadphase_cell_assignment_is_bit_exact(scene, cell):
    """Grid geometry (origin, 1/cell, cell edge, dims), every sorted (cell key,
    triangle) reference and every cell's [begin, end) equal the restatement."""
    if scene == "C4":
        sc = P.baseline_scene("C4")
    else:
        sc = P.build_scene(P.ScenarioConfig("drop", (24, 24), obstacle="icosphere:2"))
    eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13, cell_size=cell)
    got = eng.broadphase_dump()
    corners = np.asarray(sc.obstacle.vertices)[np.asarray(sc.obstacle.triangles)]
    want = O.broadphase_grid(corners.astype(np.float32), cell_size=cell)
    np.testing.assert_array_equal(got["origin"], want["origin"])
    assert got["inv_cell"] == want["inv_cell"] and got["cell"] == want["cell"]
    assert got["dims"] == want["dims"]
    np.testing.assert_array_equal(got["ref_keys"], want["ref_keys"])
    np.testing.assert_array_equal(got["ref_tris"], want["ref_tris"])
    np.testing.assert_array_equal(got["cell_begin"], want["cell_begin"])
    np.testing.assert_array_equal(got["cell_end"], want["cell_end"])
    assert len(got["ref_keys"]) >= len(corners)


# ---- the fast kernel's own forces ----------------------------------------------------

def _perturbed_6x6(rng):
    mesh = generate_cloth_grid(6, 6)
    mesh.positions += rng.normal(scale=0.02, size=mesh.positions.shape)
    vel = rng.normal(scale=0.3, size=mesh.positions.shape).astype(np.float32)
    return mesh, vel


def _forces_from_velocity_step(mesh, vel, params):
    """One fast step with gravity off: F = (v1 - v0) * m / dt (semi-implicit
    Euler, kernels.py:113-133), i.e. the forces k_pair3 integrated."""
    eng = P.Engine(mesh, params=params)  # precision="fast", kernel="pair"
    assert eng.stencil
    eng.write_positions(np.asarray(mesh.positions, dtype=np.float32))
    eng.write_velocities(vel)
    eng.step()
    v1 = eng.read_velocities().astype(np.float64)
    m = np.asarray(mesh.masses, dtype=np.float64)[:, None]
    return (v1 - vel.astype(np.float64)) * m / params.dt, eng


def _solver_forces(mesh, vel, params):
    so = O.SolverOracle(mesh, params)
    so.pos[...] = np.asarray(mesh.positions, dtype=np.float32).astype(np.float64)
    so.vel[...] = vel.astype(np.float64)
    return so.forces_now().copy(), so


def test_fast_kernel_forces_from_the_velocity_change(rng):
    params = SimParams(dt=1.0, gravity=(0.0, 0.0, 0.0), stiffness=30.0, damping=0.4)
    mesh, vel = _perturbed_6x6(rng)
    got, _ = _forces_from_velocity_step(mesh, vel, params)
    want, _ = _solver_forces(mesh, vel, params)
    scale = np.abs(want).max()
    assert scale > 0.1
    np.testing.assert_allclose(got, want, rtol=0, atol=2e-6 * scale)


def test_fast_read_forces_raw_is_the_fast_kernels_own(rng):
    """read_forces_raw on a fast engine runs k_pair3 in its read-only forces
    mode on the pre-step state: i32 fixed point within half a quantum plus
    the kernel's float error of the f64 solver (test_gpu_engine.py:92-106
    asks for 5e-4)."""
    params = SimParams(gravity=(0.0, 0.0, 0.0), stiffness=30.0, damping=0.4)
    mesh, vel = _perturbed_6x6(rng)
    eng = P.Engine(mesh, params=params)
    eng.write_velocities(vel)
    raw0 = eng.read_forces_raw()
    assert raw0.dtype == np.int32 and not raw0.any()  # no spring pass yet
    eng.step()
    got = P.decode_values(eng.read_forces_raw(), SCALE, float32=False)
    want, _ = _solver_forces(mesh, vel, params)
    np.testing.assert_allclose(got, want, rtol=0, atol=0.5 / SCALE + 2e-6 * np.abs(want).max())


def test_springs_shorter_than_1e_12_apply_no_force(rng):
    """solver.py:111-113 skips a spring with length < 1e-12 (kernels.py:97:
    only length > 1e-12 contributes).  Node 1 sits 1e-13 from node 0 (its
    structural spring is skipped), node 6 sits 2e-12 from node 0 (its spring
    acts), node 14 coincides with node 15 (skipped)."""
    mesh, vel = _perturbed_6x6(rng)
    pos = np.asarray(mesh.positions, dtype=np.float32).copy()
    pos[0] = (0.0, 0.0, 0.0)
    pos[1] = (1e-13, 0.0, 0.0)
    pos[6] = (2e-12, 0.0, 0.0)
    pos[15] = pos[14]
    mesh.positions = pos.astype(np.float64)
    params = SimParams(dt=1.0, gravity=(0.0, 0.0, 0.0), stiffness=30.0, damping=0.4)
    got, eng = _forces_from_velocity_step(mesh, vel, params)
    want, so = _solver_forces(mesh, vel, params)
    assert so.degenerate_springs == 2
    scale = np.abs(want).max()
    np.testing.assert_allclose(got, want, rtol=0, atol=2e-6 * scale)
    # and through the forces-mode readback (pre-step state)
    raw = P.decode_values(eng.read_forces_raw(), SCALE, float32=False)
    np.testing.assert_allclose(raw, want, rtol=0, atol=0.5 / SCALE + 2e-6 * scale)


# ---- contacts ---------------------------------------------------------------------------

def _drape(sc, frames):
    eng = P.Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**13)
    eng.step_frames(frames)
    return eng


def _fast_detect_at_current_state(eng, capacity=1 << 22):
    """Force pass, then the detect pass alone with the contact log on:
    (positions the detect pass saw, contact multiset, acc, count)."""
    from paper_2507_11794_b200 import _native as N

    eng.enable_contact_log(capacity)
    N.check(eng._lib.cs_run_pass(eng._handle, N.PASS_FORCE_INTEGRATE))
    pos = eng.read_positions()
    N.check(eng._lib.cs_run_pass(eng._handle, N.PASS_DETECT))
    return pos, Counter(map(tuple, eng.read_contacts().tolist())), \
        eng.read_accumulator_raw(), eng.read_counts()


def test_c4_contact_set_equals_the_f64_solver_outside_the_1e6_band():
    """C4 (64^2 cloth on the 99,904-triangle sphere), fast mode, after 120
    frames of draping: the GPU contact multiset against detect_all
    (collision.py:243-315, brute force in float64) at the same positions.
    Every differing pair must lie within 1e-6 of a predicate boundary; no
    count allowance."""
    from test_gpu_bands_collision import _assert_diff_on_boundary

    sc = P.baseline_scene("C4")
    eng = _drape(sc, 120)
    pos, gpu, _, _ = _fast_detect_at_current_state(eng)
    so = O.SolverOracle(sc.mesh, sc.params, sc.obstacle)
    so.pos[...] = pos.astype(np.float64)
    O.set_threads(O.max_threads())
    hits, ref_arr = so.detect_contacts()
    ref = Counter(map(tuple, ref_arr.tolist()))
    assert hits > 0 and sum(ref.values()) > 100
    diff = (gpu - ref) + (ref - gpu)
    _assert_diff_on_boundary(diff, sc.mesh, sc.obstacle, pos, tol=1e-6)


def test_c3_detect_pass_is_bit_identical_to_the_cpu_engine_oracle():
    """C3 (316^2 cloth draped 300 frames on the 99,904-triangle sphere), fast
    mode: one detect pass at the engine's positions against the CPU engine
    oracle (kernels.py:186-290 with the reference's padded-box prefilter,
    every pair, all host cores) -- hits, accumulators and counts equal."""
    sc = P.baseline_scene("C3")
    eng = _drape(sc, 300)
    pos, gpu, acc, cnt = _fast_detect_at_current_state(eng)
    hits = eng.stats()["hits"]
    eo = O.EngineOracle(sc.mesh, sc.params, sc.obstacle, prefilter=True)
    eo.pos[...] = pos
    O.set_threads(O.max_threads())
    ha, hb = eo.detect()
    assert ha + hb > 1000 and hits == ha + hb
    np.testing.assert_array_equal(acc, eo.acc)
    np.testing.assert_array_equal(cnt, eo.count)
    assert sum(gpu.values()) == int(eo.count.sum())


# ---- trajectories ------------------------------------------------------------------------

def test_c1_fast_drift_is_bounded_by_the_reference_engines_own():
    """C1 (64^2, two pinned corners, dt 0.004): fast mode vs the f64 solver
    oracle at steps 1/10/50/100, against the reference float32 engine's drift
    from the same solver (tests/golden/c1_drift.npz, made by the unmodified
    reference): at most 2x that drift, and at least within the per-step
    1e-5-of-extent gate while the drift is still sub-1e-5."""
    g = load_golden("c1_drift.npz")
    sc = P.baseline_scene("C1")
    ext = _extent(sc.mesh)
    so = O.SolverOracle(sc.mesh, sc.params)
    O.set_threads(O.max_threads())
    eng = P.Engine(sc.mesh, params=sc.params)
    done = 0
    for cp, ref_gap in zip(g["checkpoints"].tolist(), g["eng_vs_sol_dx"].tolist()):
        for _ in range(cp - done):
            so.step(normals=False)
        eng.step_frames(cp - done)
        done = cp
        gap = np.abs(eng.read_positions().astype(np.float64) - so.pos).max()
        print(f"C1 step {cp}: fast {gap:.3e}, reference f32 engine {ref_gap:.3e}")
        assert gap <= max(2.0 * ref_gap, 1e-5 * ext), (cp, gap, ref_gap)


@pytest.mark.parametrize("name", TRAJ)
def test_fast_mode_golden_trajectories_within_tolerance(name):
    """Every golden scene (hanging, corner, drop, pull with ext accel, flags:
    substeps 2 + explicit Euler + raw response + margin 0.006) in the fast
    mode.  Over the whole run: within 1e-3 of extent of the f64 solver, or
    within 2x the reference f32 engine's own distance from it where the
    scene is chaotic (flags: the reference engine and solver end 3.6 apart
    at frame 50 -- contact flips under the raw response).  From each
    checkpoint's solver state (identical input): one fast frame within 1e-5
    of extent of one solver frame (the per-step gate)."""
    g = load_golden(name)
    mesh, params, obs = mesh_from_golden(g), params_from_golden(g), obstacle_from_golden(g)
    eng = P.Engine(mesh, obstacle=obs, params=params, pair_budget=10**13)
    if "ext" in g:
        eng.set_external_accel(g["ext"])
    ext = _extent(mesh)
    done = 0
    for cp in g["checkpoints"].tolist():
        eng.step_frames(cp - done)
        done = cp
        got = eng.read_positions().astype(np.float64)
        d_sol = np.abs(got - g[f"sol_pos_{cp}"]).max()
        d_ref = np.abs(g[f"eng_pos_{cp}"].astype(np.float64) - g[f"sol_pos_{cp}"]).max()
        print(f"{name} frame {cp}: fast vs solver {d_sol:.3e}, reference engine vs solver "
              f"{d_ref:.3e}")
        assert d_sol <= max(1e-3 * ext, 2.0 * d_ref), (cp, d_sol, d_ref)
    O.set_threads(O.max_threads())
    for cp in g["checkpoints"].tolist():
        pos = g[f"sol_pos_{cp}"].astype(np.float32)
        vel = g[f"sol_vel_{cp}"].astype(np.float32)
        one = P.Engine(mesh, obstacle=obs, params=params, pair_budget=10**13)
        if "ext" in g:
            one.set_external_accel(g["ext"])
        one.write_positions(pos)
        one.write_velocities(vel)
        one.step()
        so = O.SolverOracle(mesh, params, obs, external_accel=g.get("ext"))
        so.pos[...] = pos.astype(np.float64)
        so.vel[...] = vel.astype(np.float64)
        so.step(normals=False)
        dx = np.abs(one.read_positions().astype(np.float64) - so.pos).max()
        dv = np.abs(one.read_velocities().astype(np.float64) - so.vel).max()
        print(f"{name} one frame from frame {cp}: |dx| {dx:.3e}, |dv| {dv:.3e}")
        assert dx <= 1e-5 * ext and dv <= 1e-5 * ext, (cp, dx, dv)
