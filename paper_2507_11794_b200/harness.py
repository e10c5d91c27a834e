"""The benchmark harness on the B200 backend.

Mirrors the reference harness (clothsim/bench.py): timed scenario runs
(``run_backend`` bench.py:128-210, ``run_scenario`` :213-253), the resolution
sweep (``run_resolution_sweep`` :324-378, SweepRow / SWEEP_FIELDS :256-321)
and the device probe (``probe_limits`` :390-415) -- with the "gpu" backend
being this package's Engine on a B200 ("cuda").  The per-frame rows are the
reference's FrameStats (io.py:29-74) plus device-time and roofline columns
(frames.py); the sweep CSV has the reference's header so its tools read it.

The reference's CPU solver is not part of this package (it is the
reference's own code path); a sweep here fills the gpu columns and leaves
the cpu ones empty, exactly as the reference does for ``--backend gpu``.
"""

from __future__ import annotations

import csv
import dataclasses
import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .engine import DEFAULT_PAIR_BUDGET, Engine, get_adapter
from .errors import CapacityError, CollisionBudgetError
from .frames import run_frames, write_stats_csv
from .mesh import spring_count_formula
from .scenes import ScenarioConfig, build_scene

__all__ = [
    "STEADY_STATE_SKIP", "REALTIME_FPS", "BackendRun", "ScenarioResult", "SweepRow",
    "SWEEP_FIELDS", "ProbeReport", "grid_for_nodes", "run_backend", "run_scenario",
    "run_resolution_sweep", "write_sweep_csv", "first_below_realtime", "probe_limits",
    "steady_state_mean",
]

STEADY_STATE_SKIP = 10  # bench.py:94-99
REALTIME_FPS = 30.0


def grid_for_nodes(nodes: int) -> tuple:
    """Square grid whose node count is closest to the request (scenes.py:174-179)."""
    if nodes < 4:
        raise ValueError(f"need at least 4 nodes for a 2x2 grid, got {nodes}")
    side = max(2, round(math.sqrt(nodes)))
    return side, side


def steady_state_mean(stats) -> tuple:
    """Mean (wall_ms, fps) over the frames after the first 10 (bench.py:94-99)."""
    window = stats[STEADY_STATE_SKIP:] if len(stats) > STEADY_STATE_SKIP else stats
    return float(np.mean([r.wall_ms for r in window])), float(np.mean([r.fps for r in window]))


@dataclass
class BackendRun:
    backend: str
    stats: list
    final_positions: np.ndarray
    mean_wall_ms: float
    mean_fps: float
    mean_device_ms: float
    total_hits: int
    snapshot_paths: list


@dataclass
class ScenarioResult:
    config: ScenarioConfig
    scene: object
    runs: dict
    csv_path: Path | None


def run_backend(scene, config: ScenarioConfig, *, precision: str = "fast",
                pair_budget: int = DEFAULT_PAIR_BUDGET, snapshot_every: int | None = None,
                output: Path | None = None, device=None) -> BackendRun:
    """config.frames frames of the B200 engine, each timed (wall clock around
    the step, as bench.py:157-168, plus CUDA events on the engine's stream)."""
    eng = Engine(scene.mesh, scene.obstacle, scene.params, device or get_adapter(), pair_budget,
                 precision=precision)
    if scene.external_accel is not None:
        eng.set_external_accel(scene.external_accel)
    rows, snaps = [], []
    done = 0
    every = snapshot_every or config.frames
    while done < config.frames:
        chunk = min(every - done % every, config.frames - done)
        part = run_frames(eng, chunk)
        rows += [dataclasses.replace(r, frame=r.frame + done) for r in part]
        done += chunk
        if snapshot_every and done % snapshot_every == 0:
            stem = Path(output).with_suffix("")
            path = Path(f"{stem}_cuda_{done - 1:04d}.png")
            eng.snapshot_png(path, axis=getattr(scene, "snapshot_axis", "y"))
            snaps.append(path)
    final = eng.read_positions().astype(np.float64)
    wall, fps = steady_state_mean(rows)
    window = rows[STEADY_STATE_SKIP:] if len(rows) > STEADY_STATE_SKIP else rows
    eng.close()
    return BackendRun("cuda", rows, final, wall, fps, float(np.mean([r.device_ms for r in window])),
                      sum(r.collision_hits for r in rows), snaps)


def run_scenario(config: ScenarioConfig, *, precision: str = "fast",
                 pair_budget: int = DEFAULT_PAIR_BUDGET, output=None,
                 snapshot_every: int | None = None) -> ScenarioResult:
    """Build the scene and run it on the B200 backend (bench.py:213-253);
    the stats CSV goes to `output` when given."""
    if snapshot_every is not None and output is None:
        raise ValueError("snapshots need an output path; pass --out")
    scene = build_scene(config)
    run = run_backend(scene, config, precision=precision, pair_budget=pair_budget,
                      snapshot_every=snapshot_every, output=output)
    csv_path = None
    if output is not None:
        csv_path = Path(output)
        write_stats_csv(csv_path, run.stats)
    return ScenarioResult(config, scene, {"cuda": run}, csv_path)


SWEEP_FIELDS = ("nodes_requested", "nx", "ny", "nodes", "springs", "cpu_mean_wall_ms",
                "cpu_mean_fps", "cpu_below_30fps", "gpu_mean_wall_ms", "gpu_mean_fps",
                "gpu_below_30fps", "cpu_over_gpu_ratio", "status", "reason")


@dataclass
class SweepRow:
    """bench.py:276-321, the gpu columns filled from the B200 backend; plus
    the device time per frame (not a CSV column: the reference's header)."""

    nodes_requested: int
    nx: int
    ny: int
    nodes: int
    springs: int
    cpu_mean_wall_ms: float | None = None
    cpu_mean_fps: float | None = None
    cpu_below_30fps: bool | None = None
    gpu_mean_wall_ms: float | None = None
    gpu_mean_fps: float | None = None
    gpu_below_30fps: bool | None = None
    cpu_over_gpu_ratio: float | None = None
    status: str = "ok"
    reason: str = ""
    gpu_mean_device_ms: float | None = None

    def as_row(self) -> list:
        def num(x, places):
            return "" if x is None else f"{x:.{places}f}"

        def flag(x):
            return "" if x is None else ("yes" if x else "no")

        return [str(self.nodes_requested), str(self.nx), str(self.ny), str(self.nodes),
                str(self.springs), num(self.cpu_mean_wall_ms, 3), num(self.cpu_mean_fps, 2),
                flag(self.cpu_below_30fps), num(self.gpu_mean_wall_ms, 3),
                num(self.gpu_mean_fps, 2), flag(self.gpu_below_30fps),
                num(self.cpu_over_gpu_ratio, 3), self.status, self.reason]


def write_sweep_csv(path, rows) -> None:
    with Path(path).open("w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(SWEEP_FIELDS)
        for r in rows:
            w.writerow(r.as_row())


def run_resolution_sweep(base_config: ScenarioConfig, resolutions, *, precision: str = "fast",
                         pair_budget: int = DEFAULT_PAIR_BUDGET) -> list:
    """One summary row per requested node count, ascending (bench.py:324-378);
    a resolution that fails (capacity, collision budget, runtime) records its
    status and reason and the sweep moves on."""
    resolutions = list(resolutions)
    if not resolutions:
        raise ValueError("sweep needs at least one resolution")
    if any(b <= a for a, b in zip(resolutions, resolutions[1:])):
        raise ValueError(f"sweep resolutions must be strictly ascending, got {resolutions}")
    rows = []
    for requested in resolutions:
        nx, ny = grid_for_nodes(requested)
        row = SweepRow(requested, nx, ny, nx * ny, sum(spring_count_formula(nx, ny)))
        config = dataclasses.replace(base_config, grid=(nx, ny))
        try:
            res = run_scenario(config, precision=precision, pair_budget=pair_budget)
        except (CapacityError, CollisionBudgetError, RuntimeError) as exc:
            row.status = type(exc).__name__
            row.reason = str(exc).splitlines()[0]
            rows.append(row)
            continue
        run = res.runs["cuda"]
        row.gpu_mean_wall_ms = run.mean_wall_ms
        row.gpu_mean_fps = run.mean_fps
        row.gpu_below_30fps = run.mean_fps < REALTIME_FPS
        row.gpu_mean_device_ms = run.mean_device_ms
        rows.append(row)
    return rows


def first_below_realtime(rows, backend: str = "gpu"):
    key = f"{backend}_below_30fps"
    for r in rows:
        if getattr(r, key):
            return r.nodes
    return None


@dataclass
class ProbeReport:
    device_name: str
    total_bytes: int
    free_bytes: int
    bytes_per_node: float
    max_side: int
    max_nodes: int
    limit: str


def _grid_engine_bytes(side: int, precision: str = "fast") -> int:
    """Device bytes of a collision-free side x side grid engine, by the same
    census Engine.layout checks against free memory (engine.py Layout)."""
    esz = 8 if precision == "fp64" else 4
    pitch_nodes = ((side + 31) // 32 * 32) * side
    tris = 2 * (side - 1) ** 2
    return 2 * 6 * pitch_nodes * esz + 3 * pitch_nodes * esz + 24 * pitch_nodes + 12 * tris


def probe_limits(device=None, precision: str = "fast") -> tuple:
    """The real device's capacity for square cloth grids (bench.py:390-415
    probes the WebGPU binding limits; here the limit is device memory and
    the 2^31 - 1 node index space of cs_create).  Returns (ProbeReport, text)."""
    dev = device if device is not None else get_adapter()
    free, total = dev.mem_info()
    name = "cuda"
    try:
        import torch

        name = torch.cuda.get_device_name(0)
    except Exception:
        pass
    lo, hi = 2, 2
    while _grid_engine_bytes(hi * 2, precision) <= free and (hi * 2) ** 2 <= (1 << 31) - 1:
        hi *= 2
    hi *= 2
    while hi - lo > 1:  # largest side whose engine fits
        mid = (lo + hi) // 2
        fits = _grid_engine_bytes(mid, precision) <= free and mid * mid <= (1 << 31) - 1
        lo, hi = (mid, hi) if fits else (lo, mid)
    side = lo
    limit = "device memory" if (side + 1) ** 2 <= (1 << 31) - 1 else "2^31-1 node indices"
    rep = ProbeReport(name, total, free, _grid_engine_bytes(side, precision) / (side * side), side,
                      side * side, limit)
    lines = [
        "device limits:",
        f"  device:                   {name}",
        f"  total memory:             {total} bytes",
        f"  free memory:              {free} bytes",
        f"largest square cloth that fits: {side} x {side} ({side * side} nodes)",
        f"limiting resource: {limit}; {rep.bytes_per_node:.1f} bytes per node ({precision}: "
        "two ping-pong SoA state buffers, normals, pins, collision accumulators, triangles)",
        "layout arithmetic: nodes = side^2; pitch = round_up(side, 32); "
        "bytes = 12*esz*pitch*side + 3*esz*pitch*side + 24*pitch*side + 24*(side-1)^2",
    ]
    return rep, "\n".join(lines)
