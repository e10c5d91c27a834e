"""Pin the CPU oracle (oracle/) to golden vectors produced by the reference.

The fixtures in tests/golden/ were generated from the unmodified reference
package by tests/golden/make_golden.py; these tests run without it.
"""

import numpy as np
import pytest

from conftest import TRAJ, load_golden, mesh_from_golden, obstacle_from_golden, params_from_golden
from oracle import oracle as O


@pytest.mark.parametrize("name", TRAJ)
def test_solver_oracle_matches_reference_solver_bit_for_bit(name):
    g = load_golden(name)
    mesh, params, obs = mesh_from_golden(g), params_from_golden(g), obstacle_from_golden(g)
    so = O.SolverOracle(mesh, params, obs, external_accel=g.get("ext"))
    cps = set(g["checkpoints"].tolist())
    hits = []
    for f in range(1, max(cps) + 1):
        hits.append(so.step())
        if f in cps:
            np.testing.assert_array_equal(so.pos, g[f"sol_pos_{f}"])
            np.testing.assert_array_equal(so.vel, g[f"sol_vel_{f}"])
            np.testing.assert_array_equal(so.normals, g[f"sol_nrm_{f}"])
    np.testing.assert_array_equal(hits, g["sol_hits"][: len(hits)])


@pytest.mark.parametrize("name", TRAJ)
def test_engine_oracle_matches_reference_engine_bit_for_bit(name):
    g = load_golden(name)
    mesh, params, obs = mesh_from_golden(g), params_from_golden(g), obstacle_from_golden(g)
    eo = O.EngineOracle(mesh, params, obs)
    if "ext" in g:
        eo.set_external_accel(g["ext"])
    cps = set(g["checkpoints"].tolist())
    hits = []
    for f in range(1, max(cps) + 1):
        hits.append(eo.step()[0])
        if f in cps:
            np.testing.assert_array_equal(eo.pos, g[f"eng_pos_{f}"])
            np.testing.assert_array_equal(eo.vel, g[f"eng_vel_{f}"])
            np.testing.assert_array_equal(eo.normals, g[f"eng_nrm_{f}"])
            np.testing.assert_array_equal(eo.forces, g[f"eng_frc_{f}"])
    np.testing.assert_array_equal(hits, g["eng_hits"][: len(hits)])


def test_engine_oracle_prefilter_is_brute_force():
    """kernels.py's padded-box prefilter never drops a hit (the reference's own
    claim, test_gpu_engine.py:267-307), restated on the oracle."""
    g = load_golden("traj_drop10.npz")
    mesh, params, obs = mesh_from_golden(g), params_from_golden(g), obstacle_from_golden(g)
    a = O.EngineOracle(mesh, params, obs, prefilter=True)
    b = O.EngineOracle(mesh, params, obs, prefilter=False)
    for _ in range(40):
        a.step()
        b.step()
    np.testing.assert_array_equal(a.pos, b.pos)
    assert a.hit_counter == b.hit_counter > 0


def test_codec_known_answers():
    k = load_golden("kats.npz")
    got = [O.encode(v) for v in k["codec_values"]]
    np.testing.assert_array_equal(got, k["codec_encoded"])
    assert O.encode(0.1) == 6554 and O.encode(-0.25) == -16384
    assert O.encode(1e9) == 2147483520 and O.encode(-1e9) == -2147483520


def test_segment_triangle_f32_known_answers():
    k = load_golden("kats.npz")
    seg, tri = k["mt_seg"], k["mt_tri"]
    for i in range(len(seg)):
        ok, pt = O.segment_triangle_f32(seg[i, 0], seg[i, 1], tri[i, 0], tri[i, 1], tri[i, 2])
        assert ok == bool(k["mt_hit32"][i]), i
        if ok:
            np.testing.assert_array_equal(pt, k["mt_point32"][i])
    assert k["mt_hit32"].sum() > 100


def test_topology_restatement_matches_reference():
    t = load_golden("topology.npz")
    for key in ("2x2", "3x5", "7x4", "16x16", "13x9"):
        nx, ny = map(int, key.split("x"))
        pos, springs, kinds, rest, tris = O.grid_topology(nx, ny, 1.3, 0.7)
        np.testing.assert_array_equal(pos, t[f"{key}_positions"])
        np.testing.assert_array_equal(springs, t[f"{key}_springs"])
        np.testing.assert_array_equal(kinds, t[f"{key}_kinds"])
        np.testing.assert_array_equal(rest, t[f"{key}_rest"])
        np.testing.assert_array_equal(tris, t[f"{key}_tris"])
        np.testing.assert_array_equal(O.unique_edges(tris), t[f"{key}_edges"])


def test_vertex_normals_known_answer():
    k = load_golden("kats.npz")
    got = O.vertex_normals(len(k["vn_positions"]), k["vn_tris"], k["vn_positions"])
    np.testing.assert_array_equal(got, k["vn_normals"])


def test_thread_count_does_not_change_bits():
    g = load_golden("traj_drop10.npz")
    mesh, params, obs = mesh_from_golden(g), params_from_golden(g), obstacle_from_golden(g)
    runs = []
    for threads in (1, 4):
        O.set_threads(threads)
        so = O.SolverOracle(mesh, params, obs)
        eo = O.EngineOracle(mesh, params, obs)
        for _ in range(30):
            so.step()
            eo.step()
        runs.append((so.pos.copy(), eo.pos.copy()))
    O.set_threads(1)
    np.testing.assert_array_equal(runs[0][1], runs[1][1])
    np.testing.assert_array_equal(runs[0][0], runs[1][0])


def test_c1_drift_golden_reproduced_by_the_engine_oracle():
    """tests/golden/c1_drift.npz holds the reference float32 engine's C1
    positions at steps 1/10/50/100; the engine oracle reproduces them bit for
    bit, and with the solver oracle the recorded drift."""
    from paper_2507_11794_b200.scenes import baseline_scene

    g = load_golden("c1_drift.npz")
    sc = baseline_scene("C1")
    eo = O.EngineOracle(sc.mesh, sc.params)
    so = O.SolverOracle(sc.mesh, sc.params)
    O.set_threads(O.max_threads())
    done = 0
    for cp, gap in zip(g["checkpoints"].tolist(), g["eng_vs_sol_dx"].tolist()):
        for _ in range(cp - done):
            eo.step()
            so.step(normals=False)
        done = cp
        np.testing.assert_array_equal(eo.pos, g[f"eng_pos_{cp}"])
        assert np.abs(eo.pos.astype(np.float64) - so.pos).max() == gap


def _grid_loops(corners, cell_size=None):
    """Plain-loop restatement of the cell assignment (small obstacles only)."""
    origin, inv, _, dims = O.grid_geometry(corners, cell_size)
    refs = []
    for t, c in enumerate(np.asarray(corners, np.float32).reshape(-1, 3, 3)):
        lo, hi = c.min(axis=0), c.max(axis=0)
        a = O.grid_cell_of(lo, origin, inv, dims)
        b = O.grid_cell_of(hi, origin, inv, dims)
        for z in range(a[2], b[2] + 1):
            for y in range(a[1], b[1] + 1):
                for x in range(a[0], b[0] + 1):
                    refs.append(((z * dims[1] + y) * dims[0] + x, t))
    refs.sort(key=lambda r: r[0])  # stable: triangle order within a cell
    return np.array(refs, dtype=np.int64).reshape(-1, 2)


@pytest.mark.parametrize("sub,cell", [(1, None), (2, None), (2, 0.05), (3, 0.011)])
def test_broadphase_restatement_is_a_conservative_prefilter(sub, cell):
    """The grid restatement (oracle.broadphase_grid, the checker of the
    device build) equals its plain-loop form, and as a prefilter it loses no
    pair the reference's brute force would box-test: for random query boxes,
    every triangle whose box overlaps the query is referenced by a cell of
    the query's cell range (the contract of test_gpu_engine.py:267-307,
    prefilter == brute force)."""
    from paper_2507_11794_b200.mesh import generate_icosphere

    ico = generate_icosphere(sub, radius=0.3, center=(0.1, -0.2, 0.3))
    corners = np.asarray(ico.vertices)[np.asarray(ico.triangles)].astype(np.float32)
    g = O.broadphase_grid(corners, cell)
    loops = _grid_loops(corners, cell)
    np.testing.assert_array_equal(g["ref_keys"], loops[:, 0])
    np.testing.assert_array_equal(g["ref_tris"], loops[:, 1])
    nz = g["cell_end"] > g["cell_begin"]
    assert (g["cell_end"][nz] - g["cell_begin"][nz]).sum() == len(g["ref_keys"])
    lo = corners.min(axis=1)
    hi = corners.max(axis=1)
    rng = np.random.default_rng(7)
    for _ in range(200):
        c = rng.uniform(-0.3, 0.5, size=3).astype(np.float32)
        w = rng.uniform(0.0, 0.08, size=3).astype(np.float32)
        ql, qh = c - w, c + w
        brute = set(np.flatnonzero((lo <= qh).all(axis=1) & (hi >= ql).all(axis=1)).tolist())
        a = O.grid_cell_of(ql, g["origin"], g["inv_cell"], g["dims"])
        b = O.grid_cell_of(qh, g["origin"], g["inv_cell"], g["dims"])
        dx, dy = g["dims"][0], g["dims"][1]
        found = set()
        for z in range(a[2], b[2] + 1):
            for y in range(a[1], b[1] + 1):
                for x in range(a[0], b[0] + 1):
                    k = (z * dy + y) * dx + x
                    found.update(g["ref_tris"][g["cell_begin"][k]:g["cell_end"][k]].tolist())
        assert brute <= found
