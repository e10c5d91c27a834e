"""Benchmark scenes (inputs of the hot path), mirroring clothsim/scenes.py.

``build_scene(ScenarioConfig(...))`` builds the reference's hanging / drop /
pull scenes with the same derived coefficients (``stable_coefficients``,
scenes.py:90-94) and placement (scenes.py:226-289).  ``baseline_scene(k)``
builds BASELINE.json's five configurations with the dt the survey fixes for
stable, well-conditioned parity gates (dt = 0.004; SURVEY.md section 0,
findings 1-2):

  C1  64x64, two pinned top corners, gravity, no collision
  C2  800x800 hanging, top row pinned, no collision (the headline workload)
  C3  316x316 dropped on a procedural 100K-triangle sphere
  C4  64x64 dropped on the same 100K-triangle sphere
  C5  4096x4096 hanging (row-band partitioned across GPUs)
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .mesh import (
    ClothMesh,
    SimParams,
    TriangleMesh,
    generate_cloth_grid,
    generate_icosphere,
    generate_uv_sphere,
)

__all__ = [
    "CLOTH_SIZE", "NODE_MASS", "SPHERE_RADIUS", "ScenarioConfig", "Scene",
    "stable_coefficients", "build_scene", "baseline_scene", "parse_obstacle_spec",
    "corner_pinned_cloth", "BASELINE_CONFIGS",
]

SCENE_NAMES = ("hanging", "drop", "pull")
CLOTH_SIZE = 1.0
NODE_MASS = 0.05
SPHERE_RADIUS = 0.3
CLEARANCE_FACTOR = 0.05
MARGIN_FACTOR = 0.02
MAX_ICOSPHERE_SUBDIV = 7
CONTACT_DT = 0.004
HANGING_DT = 0.016


def stable_coefficients(node_mass: float, dt: float) -> tuple:
    """k = 0.15 m / dt^2, c = 0.2 sqrt(k m) (scenes.py:90-94)."""
    stiffness = 0.15 * node_mass / (dt * dt)
    return stiffness, 0.2 * math.sqrt(stiffness * node_mass)


@dataclass
class ScenarioConfig:
    scene: str = "hanging"
    grid: tuple = (32, 32)
    obstacle: str | None = None
    frames: int = 120
    dt: float | None = None
    stiffness: float | None = None
    damping: float | None = None
    pull_accel: float = 4.0

    def __post_init__(self):
        if self.scene not in SCENE_NAMES:
            raise ValueError(f"scene must be one of {SCENE_NAMES}, got {self.scene!r}")
        nx, ny = self.grid
        if nx < 2 or ny < 2:
            raise ValueError(f"grid must be at least 2x2, got {nx}x{ny}")
        if self.scene == "hanging" and self.obstacle is not None:
            raise ValueError("the hanging scene excludes collision processing; drop --obstacle")
        if self.scene in ("drop", "pull") and self.obstacle is None:
            raise ValueError(f"the {self.scene} scene requires an obstacle")
        if self.dt is not None and not self.dt > 0:
            raise ValueError(f"dt must be positive, got {self.dt}")


@dataclass
class Scene:
    name: str
    mesh: ClothMesh
    params: SimParams
    obstacle: TriangleMesh | None = None
    external_accel: np.ndarray | None = None
    sphere_center: np.ndarray | None = None
    sphere_radius: float | None = None
    snapshot_axis: str = "y"  # scenes.py:157 (hanging "z", drop / pull "x")


def parse_obstacle_spec(spec: str):
    """'icosphere:K', 'uvsphere:SLICES[xSTACKS]' (procedural, this package) or
    an OBJ path (scenes.py:182-194)."""
    if spec.startswith("icosphere:"):
        k = int(spec.split(":", 1)[1])
        if not 0 <= k <= MAX_ICOSPHERE_SUBDIV:
            raise ValueError(f"icosphere subdivision must be in [0, {MAX_ICOSPHERE_SUBDIV}]")
        return ("icosphere", k)
    if spec.startswith("uvsphere:"):
        tail = spec.split(":", 1)[1].lower().split("x")
        slices = int(tail[0])
        stacks = int(tail[1]) if len(tail) > 1 else slices
        return ("uvsphere", (slices, stacks))
    return ("obj", spec)


def _params(config, response_margin=None, default_dt=HANGING_DT) -> SimParams:
    dt = config.dt if config.dt is not None else default_dt
    k, c = stable_coefficients(NODE_MASS, dt)
    kw = dict(dt=dt, stiffness=config.stiffness if config.stiffness is not None else k,
              damping=config.damping if config.damping is not None else c)
    if response_margin is not None:
        kw["response_margin"] = response_margin
    return SimParams(**kw)


def _rotate_xz_to_xy(p: np.ndarray) -> np.ndarray:
    """(x, 0, z) -> (x, -z, 0) (scenes.py:226-231)."""
    out = np.zeros_like(p)
    out[:, 0] = p[:, 0]
    out[:, 1] = -p[:, 2]
    return out


def _load_obstacle(spec: str):
    kind, value = parse_obstacle_spec(spec)
    radius = SPHERE_RADIUS * CLOTH_SIZE
    if kind == "icosphere":
        return generate_icosphere(value, radius=radius), np.zeros(3), radius, MARGIN_FACTOR * radius
    if kind == "uvsphere":
        # an analytic sphere, but placed like an OBJ obstacle (scenes.py:254-266)
        return generate_uv_sphere(value[0], value[1], radius=radius), None, None, None
    from .objio import load_obj

    v, t = load_obj(value)
    return TriangleMesh(vertices=v, triangles=t), None, None, None


def _cloth_over_obstacle(config):
    nx, ny = config.grid
    obstacle, center, radius, margin = _load_obstacle(config.obstacle)
    if radius is not None:
        size, top = CLOTH_SIZE, center[1] + radius
        clearance, cx, cz = CLEARANCE_FACTOR * radius, center[0], center[2]
    else:
        lo, hi = obstacle.vertices.min(axis=0), obstacle.vertices.max(axis=0)
        size = 1.25 * max(hi[0] - lo[0], hi[2] - lo[2])
        top = hi[1]
        clearance = 0.05 * max(hi[1] - lo[1], 1e-6)
        cx, cz = 0.5 * (lo[0] + hi[0]), 0.5 * (lo[2] + hi[2])
    mesh = generate_cloth_grid(nx, ny, width=size, height=size,
                               total_mass=NODE_MASS * nx * ny, pinned_rows=None)
    mesh.positions[:, 0] += cx - 0.5 * size
    mesh.positions[:, 2] += cz - 0.5 * size
    mesh.positions[:, 1] = top + clearance
    params = _params(config, response_margin=margin, default_dt=CONTACT_DT)
    return mesh, params, obstacle, center, radius


def build_scene(config: ScenarioConfig) -> Scene:
    """The reference scenes (scenes.py:234-298)."""
    if config.scene == "hanging":
        nx, ny = config.grid
        mesh = generate_cloth_grid(nx, ny, CLOTH_SIZE, CLOTH_SIZE,
                                   total_mass=NODE_MASS * nx * ny, pinned_rows="first")
        mesh.positions = _rotate_xz_to_xy(mesh.positions)
        return Scene("hanging", mesh, _params(config), snapshot_axis="z")
    mesh, params, obstacle, center, radius = _cloth_over_obstacle(config)
    if config.scene == "drop":
        return Scene("drop", mesh, params, obstacle, None, center, radius, snapshot_axis="x")
    nx, ny = config.grid
    accel = np.zeros((mesh.num_nodes, 3))
    accel[[mesh.node_index(nx - 1, j) for j in range(ny)], 0] = config.pull_accel
    return Scene("pull", mesh, params, obstacle, accel, center, radius, snapshot_axis="x")


def corner_pinned_cloth(n: int, dt: float = CONTACT_DT) -> Scene:
    """BASELINE config 1: n x n vertical cloth with its two top corners pinned
    (the reference has no corner preset: generate, rotate, pin [0, n-1];
    SURVEY.md 8(d))."""
    mesh = generate_cloth_grid(n, n, 1.0, 1.0, total_mass=NODE_MASS * n * n, pinned_rows=None)
    mesh.positions = _rotate_xz_to_xy(mesh.positions)
    mesh.pinned[[0, n - 1]] = True
    k, c = stable_coefficients(NODE_MASS, dt)
    return Scene("corners", mesh, SimParams(dt=dt, stiffness=k, damping=c))


BASELINE_CONFIGS = {
    "C1": "64x64 cloth, two pinned corners, gravity, dt 0.004, no collision",
    "C2": "800x800 (640K-node) hanging cloth, dt 0.004, no collision",
    "C3": "316x316 cloth dropped on a 99,904-triangle UV sphere, dt 0.002 (k 468.75, c 0.968)",
    "C4": "64x64 cloth dropped on a 99,904-triangle UV sphere, dt 0.004",
    "C5": "4096x4096 (16.8M-node) hanging cloth, dt 0.004",
}


def baseline_scene(name: str) -> Scene:
    name = name.upper()
    if name == "C1":
        return corner_pinned_cloth(64)
    if name == "C2":
        return build_scene(ScenarioConfig("hanging", (800, 800), dt=CONTACT_DT))
    if name == "C3":
        # The contact default (dt 0.004, k = 0.15 m/dt^2) diverges by frame
        # ~100 at 316^2 in the reference engine's own arithmetic, and so does
        # dt 0.002 with the coefficients re-derived for it (4x stiffer).  The
        # same material as C1/C2/C4 (k 468.75, c 0.968) at half the step drapes
        # stably ("scene parameters").
        k, c = stable_coefficients(NODE_MASS, CONTACT_DT)
        return build_scene(ScenarioConfig("drop", (316, 316), obstacle="uvsphere:224x224",
                                          dt=CONTACT_DT / 2, stiffness=k, damping=c))
    if name == "C4":
        return build_scene(ScenarioConfig("drop", (64, 64), obstacle="uvsphere:224x224"))
    if name == "C5":
        return build_scene(ScenarioConfig("hanging", (4096, 4096), dt=CONTACT_DT))
    raise ValueError(f"unknown baseline config {name!r}")
