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
