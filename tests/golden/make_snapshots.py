"""Golden snapshot pixels from the REFERENCE's clothsim.io.snapshot_png.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_snapshots.py

Writes tests/golden/snapshots.npz: for every case its inputs (float64
positions, triangles, optional obstacle) and the uint8 (H, W, 3) pixels the
reference wrote to PNG.  The "engine_drop" case renders the reference numpy
engine's positions after 30 frames of a drop scene; the GPU test replays it
with the bit-identical fixed-mode Engine and renders from device memory.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np
from PIL import Image

sys.path.insert(0, "/root/reference/pkg/src")

from clothsim.gpu.engine import Engine  # noqa: E402
from clothsim.io import snapshot_png  # noqa: E402
from clothsim.mesh import generate_cloth_grid, generate_icosphere  # noqa: E402
from clothsim.scenes import ScenarioConfig, build_scene  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "snapshots.npz")


def render(pos, tris, ov=None, ot=None, size=(320, 240), axis="y"):
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "s.png")
        snapshot_png(path, pos, tris, obstacle_vertices=ov, obstacle_triangles=ot, size=size,
                     axis=axis)
        return np.asarray(Image.open(path).convert("RGB"))


def main():
    cases = {}

    def add(name, pos, tris, ov=None, ot=None, size=(320, 240), axis="y"):
        px = render(pos, tris, ov, ot, size, axis)
        d = {"pos": np.asarray(pos, np.float64), "tris": np.asarray(tris, np.int32),
             "size": np.asarray(size, np.int32), "axis": np.asarray(axis), "pixels": px}
        if ov is not None:
            d["ov"] = np.asarray(ov, np.float64)
        if ot is not None:
            d["ot"] = np.asarray(ot, np.int32)
        for k, v in d.items():
            cases[f"{name}__{k}"] = v
        print(name, px.shape, int((px.sum(axis=2) > 0).sum()), "lit pixels")

    # the reference's own tint test scene (test_io.py:130-152)
    mesh = generate_cloth_grid(8, 8)
    ball = generate_icosphere(1, radius=0.25, center=(0.5, -0.5, 0.5))
    add("tints", mesh.positions, mesh.triangles, ball.vertices, ball.triangles, (200, 160), "z")
    # a flat sheet seen edge-on / face-on (constant depth: zspan clamps to 1e-12)
    flat = generate_cloth_grid(6, 6)
    add("flat_y", flat.positions, flat.triangles, size=(64, 48), axis="y")
    # crumpled sheet over a sphere, three axes
    rng = np.random.default_rng(7)
    sheet = generate_cloth_grid(24, 24)
    pos = sheet.positions + rng.normal(0.0, 0.03, sheet.positions.shape)
    ball2 = generate_icosphere(2, radius=0.3, center=(0.5, -0.2, 0.5))
    for ax in ("x", "y", "z"):
        add(f"crumpled_{ax}", pos, sheet.triangles, ball2.vertices, ball2.triangles, (320, 240), ax)
    # obstacle vertices in the bounds but no obstacle triangles
    add("bounds_only", pos, sheet.triangles, ball2.vertices, None, (96, 80), "y")
    # the reference numpy engine after 30 frames of a drop (f32 positions)
    sc = build_scene(ScenarioConfig("drop", (12, 12), obstacle="icosphere:2"))
    eng = Engine(sc.mesh, sc.obstacle, sc.params, pair_budget=10**12)
    for _ in range(30):
        eng.step()
    epos = eng.read_positions().astype(np.float64)
    add("engine_drop", epos, sc.mesh.triangles, sc.obstacle.vertices, sc.obstacle.triangles,
        (160, 120), sc.snapshot_axis)
    np.savez_compressed(OUT, **cases)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} B)")


if __name__ == "__main__":
    main()
