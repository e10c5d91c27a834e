"""Bit-exact topology / geometry of the product's input builders vs the
reference (golden fixtures) and the oracle's loop restatement."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O
from paper_2507_11794_b200 import mesh as M
from paper_2507_11794_b200.engine import _grid_stencil_rest
from paper_2507_11794_b200.scenes import ScenarioConfig, baseline_scene, build_scene


@pytest.mark.parametrize("key", ["2x2", "3x5", "7x4", "16x16", "13x9"])
def test_generate_cloth_grid_bit_exact(key):
    t = load_golden("topology.npz")
    nx, ny = map(int, key.split("x"))
    m = M.generate_cloth_grid(nx, ny, 1.3, 0.7, total_mass=0.05 * nx * ny, pinned_rows="first")
    np.testing.assert_array_equal(m.positions, t[f"{key}_positions"])
    np.testing.assert_array_equal(m.spring_indices, t[f"{key}_springs"])
    np.testing.assert_array_equal(m.spring_kinds, t[f"{key}_kinds"])
    np.testing.assert_array_equal(m.spring_rest_lengths, t[f"{key}_rest"])
    np.testing.assert_array_equal(m.triangles, t[f"{key}_tris"])
    np.testing.assert_array_equal(m.pinned, t[f"{key}_pinned"])
    np.testing.assert_array_equal(m.masses, t[f"{key}_masses"])
    np.testing.assert_array_equal(M.unique_edges(m.triangles), t[f"{key}_edges"])
    np.testing.assert_array_equal(M.grid_unique_edges(nx, ny), t[f"{key}_edges"])
    assert M.spring_count_formula(nx, ny) == tuple(t[f"{key}_census"])


@pytest.mark.parametrize("nx,ny", [(2, 2), (2, 7), (7, 2), (3, 3), (31, 17), (64, 64)])
def test_grid_builders_match_loop_restatement(nx, ny):
    pos, springs, kinds, rest, tris = O.grid_topology(nx, ny)
    m = M.generate_cloth_grid(nx, ny)
    np.testing.assert_array_equal(m.spring_indices, springs)
    np.testing.assert_array_equal(m.spring_kinds, kinds)
    np.testing.assert_array_equal(m.spring_rest_lengths, rest)
    np.testing.assert_array_equal(m.triangles, tris)
    np.testing.assert_array_equal(M.grid_unique_edges(nx, ny), O.unique_edges(tris))


def test_census_formula_matches_enumeration():
    for nx in range(2, 13):
        for ny in range(2, 13):
            m = M.generate_cloth_grid(nx, ny)
            counts = tuple(int((m.spring_kinds == k).sum()) for k in range(3))
            assert counts == M.spring_count_formula(nx, ny)


def test_single_f32_rest_length_per_family_at_baseline_sizes():
    """SURVEY.md finding 4: the 12-spring stencil with 6 constant rest lengths
    is bit-identical to the per-spring f32 table (checked where it matters)."""
    for n in (64, 316, 800):
        sc = build_scene(ScenarioConfig("hanging", (n, n), dt=0.004))
        got = _grid_stencil_rest(sc.mesh)
        assert got is not None, n
        nx, ny, rest6 = got
        assert (nx, ny) == (n, n) and all(r > 0 for r in rest6)


def test_stencil_detection_rejects_modified_topology():
    m = M.generate_cloth_grid(8, 8)
    assert _grid_stencil_rest(m) is not None
    m.spring_rest_lengths = m.spring_rest_lengths.copy()
    m.spring_rest_lengths[5] *= 1.1
    assert _grid_stencil_rest(m) is None  # falls back to the CSR gather
    m2 = M.generate_cloth_grid(8, 8)
    m2.spring_indices = m2.spring_indices[::-1].copy()
    assert _grid_stencil_rest(m2) is None


def test_icosphere_matches_reference():
    k = load_golden("kats.npz")
    ico = M.generate_icosphere(2, radius=0.3, center=(0.1, -0.2, 0.3))
    np.testing.assert_array_equal(ico.triangles, k["ico2_triangles"])
    np.testing.assert_array_equal(ico.vertices, k["ico2_vertices"])
    np.testing.assert_array_equal(ico.face_normals, k["ico2_normals"])


def test_uv_sphere_is_the_100k_obstacle():
    s = M.generate_uv_sphere(224, 224, radius=0.3)
    assert (s.num_vertices, s.num_triangles) == (49954, 99904)
    centroids = s.vertices[s.triangles].mean(axis=1)
    assert (np.einsum("ij,ij->i", s.face_normals, centroids) > 0).all()  # outward
    e = M.unique_edges(s.triangles)
    assert len(e) * 2 == 3 * s.num_triangles  # watertight: every edge in 2 faces


def test_host_vertex_normals_match_reference():
    k = load_golden("kats.npz")
    from types import SimpleNamespace

    got = M.compute_vertex_normals(SimpleNamespace(triangles=k["vn_tris"]), k["vn_positions"])
    np.testing.assert_allclose(got, k["vn_normals"], atol=1e-15)


def test_baseline_scenes_shapes():
    c1 = baseline_scene("C1")
    assert c1.mesh.num_nodes == 4096 and c1.mesh.pinned.sum() == 2
    assert c1.mesh.pinned[0] and c1.mesh.pinned[63]
    c4 = baseline_scene("C4")
    assert c4.obstacle.num_triangles == 99904 and c4.params.dt == 0.004


@pytest.mark.parametrize("nx,ny", [(2, 2), (2, 7), (7, 2), (3, 3), (31, 17), (64, 64)])
def test_separable_rest_lengths_equal_per_spring_norm(nx, ny):
    """mesh._grid_rest (tables per column / row) == |p_b - p_a| per spring."""
    m = M.generate_cloth_grid(nx, ny, 1.3, 0.7)
    ref = np.linalg.norm(m.positions[m.spring_indices[:, 1]] - m.positions[m.spring_indices[:, 0]],
                         axis=1)
    np.testing.assert_array_equal(m.spring_rest_lengths, ref)
    np.testing.assert_array_equal(M._rest_lengths(m.positions, m.spring_indices), ref)
    b = M.grid_band(nx, ny, 0, ny, 1.3, 0.7)
    np.testing.assert_array_equal(b.spring_rest_lengths, ref)


@pytest.mark.parametrize("nx,ny", [(2, 2), (2, 7), (7, 2), (3, 3), (31, 17)])
def test_grid_families_partition_the_springs(nx, ny):
    """mesh.grid_families groups grid_springs exactly by (kind, index delta)."""
    springs, kinds = M.grid_springs(nx, ny)
    ids = np.arange(len(springs))
    seen = []
    for (kind, delta), views in zip(((0, 1), (0, nx), (1, nx + 1), (1, nx - 1), (2, 2),
                                     (2, 2 * nx)), M.grid_families(ids, nx, ny)):
        got = np.sort(np.concatenate([np.ravel(v) for v in views]))
        off = springs[:, 1] - springs[:, 0]
        want = np.nonzero((kinds == kind) & (off == delta))[0]
        if (kind, delta) == (1, nx - 1):  # shear (c+1 -> c+nx)
            want = np.nonzero((kinds == 1) & (off == nx - 1))[0]
        np.testing.assert_array_equal(got, want)
        seen.append(got)
    assert sum(len(x) for x in seen) == len(springs)


def test_frame_stats_csv_round_trip_and_reference_header(tmp_path):
    """frames.FrameStats CSV: the reference's eight columns first, in its
    order (clothsim/io.py STATS_FIELDS), extras after, round-trips."""
    import sys

    from paper_2507_11794_b200 import frames as F

    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        from clothsim.io import STATS_FIELDS as REF
    except Exception:  # the reference is only in the build container
        REF = F.STATS_FIELDS
    assert F.STATS_FIELDS == tuple(REF)
    rows = [F.FrameStats(frame=i, wall_ms=1.5 + i, fps=600.0, nodes=64, springs=306,
                         obstacle_triangles=80, collision_hits=i, backend="cuda", device_ms=0.02,
                         stencil_bytes=3840, achieved_gbs=192.0, hbm_frac=0.03) for i in range(3)]
    p = tmp_path / "f.csv"
    F.write_stats_csv(p, rows)
    back = F.parse_stats_csv(p)
    assert [r.collision_hits for r in back] == [0, 1, 2]
    assert back[1].stencil_bytes == 3840 and abs(back[2].wall_ms - 3.5) < 1e-9
