"""Device-rendered snapshot_png (io.py:225-287) vs the reference's pixels.

tests/golden/snapshots.npz holds the uint8 images the reference's own
snapshot_png wrote (tests/golden/make_snapshots.py); the CUDA rasteriser must
reproduce them bit for bit, from host arrays and from an Engine's device
state.
"""

import os

import numpy as np
import pytest

import paper_2507_11794_b200 as P
from paper_2507_11794_b200 import snapshot as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "snapshots.npz")
HOST_CASES = ["tints", "flat_y", "crumpled_x", "crumpled_y", "crumpled_z", "bounds_only"]


def _case(name):
    g = np.load(GOLDEN)
    d = {k.split("__", 1)[1]: g[k] for k in g.files if k.startswith(name + "__")}
    d["axis"] = str(d["axis"])
    return d


def test_golden_snapshots_are_present_and_lit():
    for name in HOST_CASES + ["engine_drop"]:
        d = _case(name)
        w, h = (int(x) for x in d["size"])
        assert d["pixels"].shape == (h, w, 3) and d["pixels"].dtype == np.uint8
        assert (d["pixels"].sum(axis=2) > 0).any()


def test_argument_errors_match_the_reference():
    with pytest.raises(ValueError, match="axis"):
        S.snapshot_png("x.png", np.zeros((3, 3)), np.zeros((1, 3), np.int32), axis="w")
    with pytest.raises(ValueError, match="too small"):
        S.snapshot_png("x.png", np.zeros((3, 3)), np.zeros((1, 3), np.int32), size=(4, 100))


def test_camera_matches_io_py_setup():
    lo, hi = np.array([0.0, -1.0, 0.25]), np.array([1.0, 0.5, 0.25])
    span = np.maximum(hi - lo, 1e-9)
    l2, h2 = lo - 0.05 * span, hi + 0.05 * span
    sp = h2 - l2
    scale = min(319 / sp[0], 239 / sp[2])
    assert S.camera(lo, hi, 320, 240, "y") == (l2[0], l2[2], scale)


@pytest.mark.gpu
@pytest.mark.parametrize("name", HOST_CASES)
def test_device_snapshot_is_bit_identical_to_reference(name):
    d = _case(name)
    px = P.render_snapshot(d["pos"], d["tris"], obstacle_vertices=d.get("ov"),
                           obstacle_triangles=d.get("ot"), size=tuple(int(x) for x in d["size"]),
                           axis=d["axis"])
    assert px.shape == d["pixels"].shape
    bad = np.argwhere((px != d["pixels"]).any(axis=2))
    assert len(bad) == 0, f"{len(bad)} pixels differ, first {bad[:5].tolist()}"


@pytest.mark.gpu
def test_snapshot_png_bytes_deterministic_and_decode_to_the_pixels(tmp_path):
    from PIL import Image

    d = _case("crumpled_y")
    a, b = tmp_path / "a.png", tmp_path / "b.png"
    for p in (a, b):
        P.snapshot_png(p, d["pos"], d["tris"], obstacle_vertices=d["ov"], obstacle_triangles=d["ot"])
    assert a.read_bytes() == b.read_bytes()
    assert np.array_equal(np.asarray(Image.open(a).convert("RGB")), d["pixels"])


@pytest.mark.gpu
def test_engine_snapshot_from_device_state_matches_reference():
    d = _case("engine_drop")
    sc = P.build_scene(P.ScenarioConfig("drop", (12, 12), obstacle="icosphere:2"))
    eng = P.Engine(sc.mesh, sc.obstacle, sc.params, precision="fixed", pair_budget=10**12)
    for _ in range(30):
        eng.step()
    assert np.array_equal(eng.read_positions().astype(np.float64), d["pos"])  # same state
    px = eng.render_snapshot(size=tuple(int(x) for x in d["size"]), axis=d["axis"])
    bad = np.argwhere((px != d["pixels"]).any(axis=2))
    assert len(bad) == 0, f"{len(bad)} pixels differ, first {bad[:5].tolist()}"
    # the cloth alone: obstacle pixels vanish, cloth ones keep their tint family
    cloth_only = eng.render_snapshot(size=tuple(int(x) for x in d["size"]), axis=d["axis"],
                                     obstacle=False)
    assert (cloth_only.sum(axis=2) > 0).sum() <= (px.sum(axis=2) > 0).sum()
