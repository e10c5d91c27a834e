"""Generate the golden fixtures under tests/golden/ from the REFERENCE package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Every array written here comes from the unmodified reference (`clothsim`,
arxiv 2507.11794, /root/reference/pkg/src) -- its solver, its numpy "GPU"
engine and its mesh/scene builders.  The fixtures pin the CPU oracle
(oracle/) and, through it, the CUDA path on the GPU box, where the reference
is absent.  Sizes are kept small so the whole set stays a few hundred KB.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from clothsim.collision import (  # noqa: E402
    ContactAccumulator,
    apply_collision_response,
    edge_triangle_intersect,
)
from clothsim.gpu.engine import Engine  # noqa: E402
from clothsim.gpu.fixedpoint import encode_values  # noqa: E402
from clothsim.gpu.kernels import _segment_triangle_f32  # noqa: E402
from clothsim.mesh import (  # noqa: E402
    SimParams,
    compute_vertex_normals,
    generate_cloth_grid,
    generate_icosphere,
    spring_count_formula,
    unique_edges,
)
from clothsim.scenes import ScenarioConfig, build_scene, stable_coefficients  # noqa: E402
from clothsim.solver import accumulate_forces, make_state, step  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def save(name, **arrays):
    path = os.path.join(OUT, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def topology():
    out = {}
    for nx, ny in ((2, 2), (3, 5), (7, 4), (16, 16), (13, 9)):
        m = generate_cloth_grid(nx, ny, width=1.3, height=0.7, total_mass=0.05 * nx * ny,
                                pinned_rows="first")
        key = f"{nx}x{ny}"
        out[f"{key}_positions"] = m.positions
        out[f"{key}_springs"] = m.spring_indices
        out[f"{key}_kinds"] = m.spring_kinds
        out[f"{key}_rest"] = m.spring_rest_lengths
        out[f"{key}_tris"] = m.triangles
        out[f"{key}_edges"] = unique_edges(m.triangles)
        out[f"{key}_census"] = np.array(spring_count_formula(nx, ny))
        out[f"{key}_pinned"] = m.pinned
        out[f"{key}_masses"] = m.masses
    save("topology.npz", **out)


def corner_pinned(n, dt):
    """BASELINE config 1: n x n, two top corners pinned."""
    m = generate_cloth_grid(n, n, 1.0, 1.0, total_mass=0.05 * n * n, pinned_rows=None)
    rot = np.zeros_like(m.positions)
    rot[:, 0] = m.positions[:, 0]
    rot[:, 1] = -m.positions[:, 2]
    m.positions = rot
    m.pinned[[0, n - 1]] = True
    k, c = stable_coefficients(0.05, dt)
    return m, SimParams(dt=dt, stiffness=k, damping=c)


def trajectories():
    # (label, mesh, params, obstacle, ext, frames, checkpoints)
    scenes = []
    sc = build_scene(ScenarioConfig("hanging", (8, 8)))
    scenes.append(("hang8", sc.mesh, sc.params, None, None, 20, (1, 20)))
    m, p = corner_pinned(16, 0.004)
    scenes.append(("corner16", m, p, None, None, 30, (1, 30)))
    sc = build_scene(ScenarioConfig("hanging", (12, 10), dt=0.004))
    scenes.append(("hang12x10", sc.mesh, sc.params, None, None, 25, (1, 25)))
    sc = build_scene(ScenarioConfig("drop", (10, 10), obstacle="icosphere:1"))
    scenes.append(("drop10", sc.mesh, sc.params, sc.obstacle, None, 60, (20, 40, 60)))
    sc = build_scene(ScenarioConfig("pull", (8, 8), obstacle="icosphere:1"))
    scenes.append(("pull8", sc.mesh, sc.params, sc.obstacle, sc.external_accel, 40, (40,)))
    p = SimParams(dt=0.004, stiffness=(300.0, 120.0, 40.0), damping=0.7, substeps=2,
                  explicit_euler=True, average_response=False,
                  response_margin=0.006)
    sc = build_scene(ScenarioConfig("drop", (9, 11), obstacle="icosphere:1"))
    scenes.append(("flags", sc.mesh, p, sc.obstacle, None, 50, (50,)))

    for label, mesh, params, obstacle, ext, frames, checkpoints in scenes:
        out = {
            "nx": mesh.nx, "ny": mesh.ny, "positions0": mesh.positions, "pinned": mesh.pinned,
            "masses": mesh.masses, "springs": mesh.spring_indices, "kinds": mesh.spring_kinds,
            "rest": mesh.spring_rest_lengths, "tris": mesh.triangles,
            "dt": params.dt, "gravity": np.array(params.gravity),
            "stiffness": np.array(params.stiffness), "damping": params.damping,
            "epsilon_mt": params.epsilon_mt, "response_margin": params.response_margin,
            "fixed_point_scale": params.fixed_point_scale, "substeps": params.substeps,
            "explicit_euler": params.explicit_euler,
            "average_response": params.average_response,
        }
        if obstacle is not None:
            out["obs_vertices"] = obstacle.vertices
            out["obs_triangles"] = obstacle.triangles
            out["obs_normals"] = obstacle.face_normals
        if ext is not None:
            out["ext"] = ext
        state = make_state(mesh)
        eng = Engine(mesh, obstacle=obstacle, params=params, pair_budget=10**12)
        if ext is not None:
            eng.set_external_accel(ext)
        sol_hits, eng_hits = [], []
        for f in range(1, frames + 1):
            sol_hits.append(step(state, mesh, params, obstacle=obstacle, external_accel=ext,
                                 pair_budget=10**12))
            r = eng.step()
            eng_hits.append(r.hits)
            if f in checkpoints:
                out[f"sol_pos_{f}"] = state.positions.copy()
                out[f"sol_vel_{f}"] = state.velocities.copy()
                out[f"sol_nrm_{f}"] = state.normals.copy()
                out[f"eng_pos_{f}"] = eng.read_positions()
                out[f"eng_vel_{f}"] = eng.read_velocities()
                out[f"eng_nrm_{f}"] = eng.read_normals()
                out[f"eng_frc_{f}"] = eng.read_forces_raw()
        out["checkpoints"] = np.array(checkpoints)
        out["sol_hits"] = np.array(sol_hits)
        out["eng_hits"] = np.array(eng_hits)
        save(f"traj_{label}.npz", **out)


def kats():
    rng = np.random.default_rng(20240817)
    out = {}
    vals = np.array([0.0, 0.1, -0.25, 1.0, -3.5, 100.125, 1e9, -1e9, 2.5e-5, -7.6e-6,
                     0.5 / 65536, -0.5 / 65536, 1.5 / 65536, 32767.99])
    vals = np.concatenate([vals, rng.normal(scale=3.0, size=200)])
    out["codec_values"] = vals
    out["codec_encoded"] = encode_values(vals, 1 << 16)
    # segment/triangle, f64 (collision.py) and f32 (kernels.py) on random pairs
    k = 4000
    seg = rng.uniform(-1.5, 1.5, size=(k, 2, 3))
    tri = rng.uniform(-1.0, 1.0, size=(k, 3, 3))
    # bias half the corpus toward hits: segments through the triangle centroid
    cen = tri.mean(axis=1)
    half = k // 2
    dirs = rng.normal(size=(half, 3))
    seg[:half, 0] = cen[:half] - 0.5 * dirs
    seg[:half, 1] = cen[:half] + 0.5 * dirs
    hit64 = np.zeros(k, dtype=bool)
    pt64 = np.zeros((k, 3))
    for i in range(k):
        h = edge_triangle_intersect(seg[i, 0], seg[i, 1], tri[i, 0], tri[i, 1], tri[i, 2], 1e-6)
        if h is not None:
            hit64[i] = True
            pt64[i] = h.point
    s32 = seg.astype(np.float32)
    t32 = tri.astype(np.float32)
    valid, t, pt = _segment_triangle_f32(s32[:, 0], s32[:, 1], t32[:, 0], t32[:, 1], t32[:, 2],
                                         np.float32(1e-6))
    out.update(mt_seg=seg, mt_tri=tri, mt_hit64=hit64, mt_point64=pt64,
               mt_hit32=valid, mt_point32=np.where(valid[:, None], pt, 0).astype(np.float32))
    # response trace (test_acceptance.py:175-196 / test_gpu_engine.py:198-242)
    positions = np.zeros((1, 3))
    velocities = np.array([[0.0, 0.0, 2.0]])
    acc = ContactAccumulator(1)
    acc.add(0, (0.0, 0.1, 0.0))
    apply_collision_response(positions, velocities, acc)
    out["resp_pos"] = positions
    out["resp_vel"] = velocities
    # perturbed 6x6 spring forces (test_gpu_engine.py:92-106)
    mesh = generate_cloth_grid(6, 6)
    mesh.positions += rng.normal(scale=0.02, size=mesh.positions.shape)
    vel = rng.normal(scale=0.3, size=mesh.positions.shape).astype(np.float32)
    params = SimParams(gravity=(0.0, 0.0, 0.0), stiffness=30.0, damping=0.4)
    eng = Engine(mesh, params=params)
    eng.buffers.vel[...] = vel
    eng.step()
    st = make_state(mesh)
    st.velocities[...] = vel.astype(np.float64)
    accumulate_forces(st, mesh, params)
    out.update(pert_positions=mesh.positions, pert_vel=vel, pert_eng_forces=eng.read_forces_raw(),
               pert_sol_forces=st.forces, pert_eng_pos1=eng.read_positions(),
               pert_eng_vel1=eng.read_velocities())
    # icosphere (mesh.py:350-387) for the obstacle builder
    ico = generate_icosphere(2, radius=0.3, center=(0.1, -0.2, 0.3))
    out.update(ico2_vertices=ico.vertices, ico2_triangles=ico.triangles,
               ico2_normals=ico.face_normals)
    # host vertex normals on a crumpled grid
    m = generate_cloth_grid(9, 7)
    crumple = m.positions + rng.normal(scale=0.05, size=m.positions.shape)
    out.update(vn_positions=crumple, vn_tris=m.triangles,
               vn_normals=compute_vertex_normals(m, positions=crumple))
    save("kats.npz", **out)


def drift():
    """BASELINE config 1 (64x64, two pinned corners, dt 0.004): the reference
    float32 engine against the reference float64 solver, stepped in lockstep
    from the same state -- max |dx| at steps 1/10/50/100.  This is the drift
    any float32 implementation shows on this (chaotic) scene; the fast mode's
    100-step gate is pinned to it instead of a hand-picked bound."""
    mesh, params = corner_pinned(64, 0.004)
    state = make_state(mesh)
    eng = Engine(mesh, params=params)
    checkpoints = (1, 10, 50, 100)
    gaps, vgaps = [], []
    out = {}
    for f in range(1, max(checkpoints) + 1):
        step(state, mesh, params)
        eng.step()
        if f in checkpoints:
            gaps.append(np.abs(eng.read_positions().astype(np.float64) - state.positions).max())
            vgaps.append(np.abs(eng.read_velocities().astype(np.float64) - state.velocities).max())
            out[f"eng_pos_{f}"] = eng.read_positions()
    ext = float((mesh.positions.max(axis=0) - mesh.positions.min(axis=0)).max())
    out.update(checkpoints=np.array(checkpoints), eng_vs_sol_dx=np.array(gaps),
               eng_vs_sol_dv=np.array(vgaps), extent=np.float64(ext))
    print("C1 reference f32 engine vs f64 solver, max|dx|:", dict(zip(checkpoints, gaps)))
    save("c1_drift.npz", **out)


if __name__ == "__main__":
    topology()
    trajectories()
    kats()
    drift()
