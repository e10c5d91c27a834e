"""Per-frame statistics of a run: the reference harness's FrameStats CSV
(clothsim/io.py:29-74, filled by bench.run_backend, bench.py:148-200)
extended with device time and roofline columns.

    rows = run_frames(engine, frames=100)
    write_stats_csv("frames.csv", rows)

The first eight columns are the reference's, in its order and format, so
its `parse_stats_csv` reads the file; the extra columns follow them.
"""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass
from pathlib import Path

STATS_FIELDS = ("frame", "wall_ms", "fps", "nodes", "springs", "obstacle_triangles",
                "collision_hits", "backend")
EXTRA_FIELDS = ("device_ms", "stencil_bytes", "achieved_gbs", "hbm_frac")


@dataclass(frozen=True)
class FrameStats:
    frame: int
    wall_ms: float
    fps: float
    nodes: int
    springs: int
    obstacle_triangles: int
    collision_hits: int
    backend: str
    device_ms: float = float("nan")
    stencil_bytes: int = 0
    achieved_gbs: float = float("nan")
    hbm_frac: float = float("nan")

    def as_row(self) -> list:
        return [str(self.frame), f"{self.wall_ms:.3f}", f"{self.fps:.2f}", str(self.nodes),
                str(self.springs), str(self.obstacle_triangles), str(self.collision_hits),
                self.backend, f"{self.device_ms:.4f}", str(self.stencil_bytes),
                f"{self.achieved_gbs:.1f}", f"{self.hbm_frac:.4f}"]


def write_stats_csv(path, rows) -> None:
    with Path(path).open("w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(STATS_FIELDS + EXTRA_FIELDS)
        for r in rows:
            w.writerow(r.as_row())


def parse_stats_csv(path) -> list:
    with Path(path).open("r", newline="") as fh:
        rd = csv.reader(fh)
        header = tuple(next(rd))
        if header[:len(STATS_FIELDS)] != STATS_FIELDS:
            raise ValueError(f"unexpected stats header {header}")
        out = []
        for row in rd:
            extra = row[len(STATS_FIELDS):] + [""] * (len(EXTRA_FIELDS) - len(row) + len(STATS_FIELDS))
            out.append(FrameStats(
                frame=int(row[0]), wall_ms=float(row[1]), fps=float(row[2]), nodes=int(row[3]),
                springs=int(row[4]), obstacle_triangles=int(row[5]), collision_hits=int(row[6]),
                backend=row[7],
                device_ms=float(extra[0]) if extra[0] else float("nan"),
                stencil_bytes=int(extra[1]) if extra[1] else 0,
                achieved_gbs=float(extra[2]) if extra[2] else float("nan"),
                hbm_frac=float(extra[3]) if extra[3] else float("nan")))
        return out


def run_frames(engine, frames: int, peak_gbs: float = 6558.1, backend: str = "cuda") -> list:
    """Step `engine` frame by frame like bench.run_backend: wall time around
    each step (host, synchronised), device time from CUDA events on the
    engine's stream, and the stencil pass's achieved HBM bandwidth."""
    import torch

    stream = torch.cuda.ExternalStream(engine.stream_handle)
    mesh = engine.mesh
    springs = len(mesh.spring_indices)
    n_obs = len(engine.obstacle.triangles) if engine.obstacle is not None else 0
    nbytes = engine.stencil_bytes_per_frame
    rows = []
    for f in range(frames):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(stream)
        res = engine.step()
        b.record(stream)
        b.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        dev = a.elapsed_time(b)
        gbs = nbytes / (dev * 1e-3) / 1e9 if dev > 0 else float("nan")
        rows.append(FrameStats(frame=f, wall_ms=wall, fps=1e3 / max(wall, 1e-9),
                               nodes=engine.num_nodes, springs=springs, obstacle_triangles=n_obs,
                               collision_hits=int(res.hits), backend=backend, device_ms=dev,
                               stencil_bytes=nbytes, achieved_gbs=gbs,
                               hbm_frac=gbs / peak_gbs if peak_gbs else float("nan")))
    return rows
