"""The drop-in boundary: a B200 ``Engine`` with the reference's API.

Mirrors clothsim/gpu/engine.py:108-394 -- constructor signature
``Engine(mesh, obstacle=None, params=None, device=None, pair_budget=...)``,
``step(readback=False, debug=False) -> StepResult``, ``run_respond_pass``,
``inject_response``, ``set_external_accel``, the ``read_*`` readbacks, the
writable ``buffers.pos`` / ``buffers.vel`` views, ``build_pipeline`` and
``step_gpu`` -- plus ``get_adapter`` with the ``CLOTHSIM_ADAPTER`` switch
(gpu/device.py:156-172).  Every frame runs as hand-written sm_100a kernels
behind the C ABI of include/clothsim_b200.h; this module only marshals
arguments.  There is no CPU path: without the CUDA library or a device the
constructor raises ``AdapterUnavailable``.

Arithmetic modes (keyword-only ``precision=``):

* ``"fast"`` (default) -- fp32 warp-strip stencil (six forward springs per
  node, exact reaction exchange, paired FFMA2 math); parity with the
  reference CPU solver within the north star's tolerances, collision in the
  reference engine's exact f32 arithmetic.
* ``"fixed"`` -- the reference engine's arithmetic (per-spring f32 force,
  i32 fixed point at ``fixed_point_scale``): bit-identical to the reference's
  ``gpu.engine.Engine`` in every buffer, hit count and contact.
* ``"fp64"`` -- float64 gather and collision in the reference solver's
  operation order: bit-identical to ``solver.step``, obstacles included.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import AdapterUnavailable, CapacityError, CollisionBudgetError
from .fixedpoint import encode_values
from .mesh import (SimParams, grid_families, grid_springs, grid_triangles, grid_unique_edges,
                   unique_edges)

__all__ = [
    "ADAPTER_ENV", "CudaDevice", "get_adapter", "Engine", "StepResult", "Layout",
    "build_pipeline", "step_gpu", "DEFAULT_PAIR_BUDGET", "PRECISIONS",
]

ADAPTER_ENV = "CLOTHSIM_ADAPTER"
DEFAULT_PAIR_BUDGET = 20_000_000  # collision.py:40
PRECISIONS = ("fast", "fixed", "fp64")
_F32 = np.float32


class CudaDevice:
    """The compute adapter (gpu/device.py SoftwareDevice's counterpart)."""

    name = "cuda"

    def __init__(self):
        lib = N.load()
        count = lib.cs_device_count()
        if count < 1:
            raise AdapterUnavailable("no CUDA device is visible to the cloth engine")
        self.device_count = count

    def mem_info(self):
        free, total = ctypes.c_int64(), ctypes.c_int64()
        N.check(N.load().cs_mem_info(ctypes.byref(free), ctypes.byref(total)))
        return free.value, total.value


def get_adapter() -> CudaDevice:
    """Adapter selection honouring CLOTHSIM_ADAPTER (device.py:156-172):
    "none" simulates a host without an adapter; "cuda" (default), "b200" and
    the reference's "software" all select the B200 engine."""
    choice = os.environ.get(ADAPTER_ENV, "cuda").strip().lower()
    if choice == "none":
        raise AdapterUnavailable(f"{ADAPTER_ENV}=none: no compute adapter requested")
    if choice not in ("", "cuda", "b200", "gpu", "software"):
        raise AdapterUnavailable(f"unknown {ADAPTER_ENV} value {choice!r}")
    return CudaDevice()


@dataclass
class Layout:
    """Buffer census (gpu/layout.py GpuBufferLayout's counts) plus the device
    bytes this engine allocates."""

    num_nodes: int
    num_springs: int
    num_cloth_tris: int
    num_cloth_edges: int
    num_obstacle_tris: int
    state_bytes: int = 0
    total_bytes: int = 0

    def validate(self, free_bytes: int) -> None:
        if self.total_bytes > free_bytes:
            raise CapacityError(
                f"engine needs {self.total_bytes} B of device memory, {free_bytes} B free")


class StepResult:
    """Per-frame result (engine.py:100-105).  ``hits`` and ``responded`` are
    read from a device-side ring on first access, so ``step()`` never blocks."""

    __slots__ = ("_engine", "_frame", "_hits", "_responded", "positions", "debug")

    def __init__(self, engine=None, frame=-1, positions=None, debug=None, hits=None,
                 responded=None):
        self._engine, self._frame = engine, frame
        self._hits, self._responded = hits, responded
        self.positions = positions
        self.debug = {} if debug is None else debug

    def _resolve(self):
        if self._hits is None:
            if self._engine is None or not self._engine.has_obstacle:
                self._hits, self._responded = 0, 0
            else:
                self._hits, self._responded = self._engine._frame_hits(self._frame)

    @property
    def hits(self) -> int:
        self._resolve()
        return self._hits

    @property
    def responded(self) -> int:
        self._resolve()
        return self._responded

    def __repr__(self):
        return f"StepResult(frame={self._frame}, hits={self.hits}, responded={self.responded})"


class _StateView:
    """numpy-like read/write view of one (N,3) device buffer, so reference
    code such as ``eng.buffers.vel[0] = (0, 0, 2)`` keeps working."""

    # a float64 engine's state goes through its f64 buffers, so writing one
    # node leaves every other node's f64 value untouched (a round trip
    # through the f32 buffers would round them all)
    _F64 = {N.BUF_POSITIONS: N.BUF_POSITIONS64, N.BUF_VELOCITIES: N.BUF_VELOCITIES64}

    def __init__(self, engine, read_id, write_id):
        self._e, self._r, self._w = engine, read_id, write_id

    def _wide(self, buf):
        return self._e.precision == "fp64" and buf in self._F64

    def _get(self):
        if self._wide(self._r):
            return self._e._read(self._F64[self._r], np.float64, 3)
        return self._e._read(self._r, np.float32, 3)

    def __array__(self, dtype=None, copy=None):
        a = self._get()
        return a if dtype is None else a.astype(dtype)

    def __getitem__(self, idx):
        return self._get()[idx]

    def __setitem__(self, idx, value):
        if self._w is None:
            raise TypeError("this buffer is read-only")
        a = self._get()
        a[idx] = value
        if self._wide(self._w):
            self._e._write(self._F64[self._w], a)
        else:
            self._e._write(self._w, a.astype(np.float32))

    @property
    def shape(self):
        return (self._e.num_nodes, 3)

    @property
    def dtype(self):
        return np.dtype(np.float64 if self._wide(self._r) else np.float32)

    def copy(self):
        return self._get()

    def __len__(self):
        return self._e.num_nodes


class PipelineBuffers:
    def __init__(self, engine):
        self.pos = _StateView(engine, N.BUF_POSITIONS, N.BUF_POSITIONS)
        self.vel = _StateView(engine, N.BUF_VELOCITIES, N.BUF_VELOCITIES)
        self.prev = _StateView(engine, N.BUF_PREV_POSITIONS, None)
        self.normals = _StateView(engine, N.BUF_NORMALS, None)


def _grid_stencil_rest(mesh):
    """(nx, ny, rest6) when `mesh` holds generate_cloth_grid's exact topology
    and every spring family/direction has a single f32 rest length (SURVEY.md
    finding 4); None otherwise (generic CSR path)."""
    nx, ny = getattr(mesh, "nx", None), getattr(mesh, "ny", None)
    if nx is None or ny is None or nx < 2 or ny < 2:
        return None
    springs = np.asarray(mesh.spring_indices)
    kinds = np.asarray(mesh.spring_kinds)
    if len(springs) == 0 or len(np.asarray(mesh.positions)) != nx * ny:
        return None
    ref_springs, ref_kinds = grid_springs(nx, ny)
    if springs.shape != ref_springs.shape or not np.array_equal(springs, ref_springs) \
            or not np.array_equal(kinds, ref_kinds):
        return None
    if not np.array_equal(np.asarray(mesh.triangles), grid_triangles(nx, ny)):
        return None
    rest32 = np.asarray(mesh.spring_rest_lengths).astype(_F32)
    rest6 = []
    for views in grid_families(rest32, nx, ny):  # +i, +j, shear +nx+1, +nx-1, bend +2, +2nx
        vals = [v for v in views if v.size]
        if not vals:
            rest6.append(0.0)
            continue
        lo, hi = min(float(v.min()) for v in vals), max(float(v.max()) for v in vals)
        if lo != hi:  # one f32 rest length per family, else no stencil
            return None
        rest6.append(lo)
    return nx, ny, rest6


def _p(a):
    return None if a is None else a.ctypes.data


def _is_cuda_tensor(x) -> bool:
    """A torch CUDA tensor (duck-typed: torch is imported only by callers)."""
    return getattr(x, "is_cuda", False) is True and hasattr(x, "data_ptr")


_TORCH_DTYPE_NAMES = {np.dtype(np.float32): "torch.float32", np.dtype(np.float64): "torch.float64",
                      np.dtype(np.int32): "torch.int32"}


def pinned_empty(shape, dtype=np.float32) -> np.ndarray:
    """Page-locked host array (through torch's pinned allocator when torch is
    importable, else an ordinary numpy array)."""
    try:
        import torch

        tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
               np.dtype(np.int32): torch.int32}[np.dtype(dtype)]
        return torch.empty(tuple(shape), dtype=tdt, pin_memory=True).numpy()
    except Exception:
        return np.empty(shape, dtype=dtype)


def _engine_flags(p, precision, graph, force_csr, kernel, normals, narrow, seam) -> int:
    """cs_desc.flags of an Engine's keyword options."""
    flags = 0
    if p.explicit_euler:
        flags |= N.FLAG_EXPLICIT_EULER
    if p.average_response:
        flags |= N.FLAG_AVERAGE_RESPONSE
    if precision == "fixed":
        flags |= N.FLAG_FIXED_POINT
    if precision == "fp64":
        flags |= N.FLAG_FP64
    if not graph:
        flags |= N.FLAG_NO_GRAPH
    if force_csr:
        flags |= N.FLAG_FORCE_CSR
    if kernel not in ("strip", "pair", "tile"):
        raise ValueError("kernel must be 'pair' (paired-column f32x2 warp strips, default), "
                         "'strip' (scalar warp strips) or 'tile' (shared-memory tiles)")
    if kernel == "tile":
        flags |= N.FLAG_TILE_KERNEL
    if normals not in ("auto", "fused", "split"):
        raise ValueError("normals must be 'auto', 'fused' (inside the next frame's step "
                         "kernel) or 'split' (stand-alone kernel after each step)")
    flags |= {"auto": 0, "split": N.FLAG_SPLIT_NORMALS, "fused": N.FLAG_FUSE_NORMALS}[normals]
    if narrow not in ("tri", "batch", "warp", "thread"):
        raise ValueError("narrow must be 'tri' (one fused candidate enumeration per cloth "
                         "triangle for both passes, default), 'batch' (batched queries per "
                         "pass), 'warp' (warp per query) or 'thread' (thread per query)")
    if narrow == "thread":
        flags |= N.FLAG_THREAD_NARROW
    elif narrow == "warp":
        flags |= N.FLAG_WARP_NARROW
    elif narrow == "batch":
        flags |= N.FLAG_SPLIT_NARROW
    if kernel == "pair":
        flags |= N.FLAG_PAIRED
    if seam not in ("kernel", "stream"):
        raise ValueError("seam must be 'kernel' (row-band handshake inside the step kernel, "
                         "graph-replayed frames) or 'stream' (stream waits on flag words)")
    if seam == "stream":
        flags |= N.FLAG_MEMOP_SEAM
    return flags


def _stream_handle(stream) -> int:
    handle = int(getattr(stream, "cuda_stream", stream))
    if handle == 0:
        raise ValueError("pass a non-default CUDA stream (the legacy default stream "
                         "handle 0 means 'let the engine create its own')")
    return handle


class Engine:
    """A built B200 pipeline bound to one cloth/obstacle/params configuration."""

    def __init__(self, mesh, obstacle=None, params=None, device=None,
                 pair_budget: int = DEFAULT_PAIR_BUDGET, *, precision: str = "fast",
                 graph: bool = True, stream=None, cell_size: float | None = None,
                 force_csr: bool = False, kernel: str = "pair", narrow: str = "tri",
                 normals: str = "auto", seam: str = "kernel"):
        if precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {PRECISIONS}")
        self.mesh = mesh
        self.obstacle = obstacle
        self.params = params if params is not None else SimParams()
        self.device = device if device is not None else get_adapter()
        self.pair_budget = pair_budget
        self.precision = precision
        self._lib = N.load()
        self._handle = None
        p = self.params

        n = int(len(np.asarray(mesh.positions)))
        tris = np.ascontiguousarray(mesh.triangles, dtype=np.int32)
        stencil = _grid_stencil_rest(mesh)
        has_obs = obstacle is not None and len(obstacle.triangles) > 0
        n_obs = len(obstacle.triangles) if obstacle is not None else 0
        # the unique cloth edges feed only the collision passes
        if stencil is not None:
            gx, gy = stencil[0], stencil[1]
            n_edges = (gx - 1) * gy + gx * (gy - 1) + (gx - 1) * (gy - 1)
            edges = grid_unique_edges(gx, gy) if has_obs else np.zeros((0, 2), np.int32)
        else:
            edges = unique_edges(tris) if len(tris) else np.zeros((0, 2), np.int32)
            n_edges = len(edges)
            if not has_obs:
                edges = np.zeros((0, 2), np.int32)
        springs = np.ascontiguousarray(mesh.spring_indices, dtype=np.int32).reshape(-1, 2)
        esz = 8 if precision == "fp64" else 4
        pitch_nodes = ((stencil[0] + 31) // 32 * 32) * stencil[1] if stencil else n
        state_bytes = 2 * 6 * pitch_nodes * esz
        total = state_bytes + 3 * pitch_nodes * esz + 24 * pitch_nodes + 12 * len(tris) \
            + 8 * len(edges) + 48 * n_obs
        if stencil is None:
            total += 16 * len(springs) * 2 + 8 * n + 12 * len(tris) + 12 * len(tris) * esz
        self.layout = Layout(n, len(springs), len(tris), n_edges, n_obs, state_bytes, total)
        free, _ = self.device.mem_info()
        self.layout.validate(free)

        # collision.py:258-266 / engine.py:137-142: same census, same refusal
        self.pairs_per_frame = n_edges * n_obs + 3 * n_obs * len(tris)
        if self.pairs_per_frame > pair_budget:
            raise CollisionBudgetError(
                f"frame needs {self.pairs_per_frame} edge-triangle tests, "
                f"budget is {pair_budget}; raise the budget or reduce resolution")

        masses = np.asarray(mesh.masses, dtype=np.float64)
        pinned = np.asarray(mesh.pinned, dtype=bool)
        inv = np.ascontiguousarray(np.where(pinned, 0.0, 1.0 / masses).astype(_F32))
        pos32 = np.ascontiguousarray(np.asarray(mesh.positions).astype(_F32))
        keep = dict(tris=tris, edges=np.ascontiguousarray(edges, dtype=np.int32), inv=inv,
                    pos32=pos32, springs=springs,
                    kinds=np.ascontiguousarray(mesh.spring_kinds, dtype=np.int32),
                    rest32=np.ascontiguousarray(np.asarray(mesh.spring_rest_lengths).astype(_F32)))
        d = N.CsDesc()
        d.abi_version = N.ABI_VERSION
        flags = _engine_flags(p, precision, graph, force_csr, kernel, normals, narrow, seam)
        if precision == "fp64":
            keep["pos64"] = np.ascontiguousarray(mesh.positions, dtype=np.float64)
            keep["mass64"] = np.ascontiguousarray(masses)
            keep["pin8"] = np.ascontiguousarray(pinned.astype(np.uint8))
            keep["rest64"] = np.ascontiguousarray(mesh.spring_rest_lengths, dtype=np.float64)
            d.positions64 = _p(keep["pos64"])
            d.masses64 = _p(keep["mass64"])
            d.pinned = _p(keep["pin8"])
            d.spring_rest64 = _p(keep["rest64"])
        d.flags = flags
        if stencil is not None:
            d.nx, d.ny = stencil[0], stencil[1]
            for q in range(6):
                d.grid_rest[q] = stencil[2][q]
        d.num_nodes = n
        d.num_springs = len(springs)
        d.springs = _p(keep["springs"])
        d.spring_kinds = _p(keep["kinds"])
        d.spring_rest = _p(keep["rest32"])
        d.num_tris = len(tris)
        d.tris = _p(tris)
        d.num_edges = len(edges)
        d.edges = _p(keep["edges"])
        d.positions = _p(pos32)
        d.inv_mass = _p(inv)
        if has_obs:
            corners = np.asarray(obstacle.vertices)[np.asarray(obstacle.triangles)]
            keep["corners"] = np.ascontiguousarray(corners.astype(_F32))
            keep["onorm"] = np.ascontiguousarray(np.asarray(obstacle.face_normals).astype(_F32))
            d.num_obstacle_tris = n_obs
            d.obstacle_corners = _p(keep["corners"])
            d.obstacle_normals = _p(keep["onorm"])
            if precision == "fp64":  # solver-exact float64 collision
                keep["corners64"] = np.ascontiguousarray(corners, dtype=np.float64)
                keep["onorm64"] = np.ascontiguousarray(obstacle.face_normals, dtype=np.float64)
                d.obstacle_corners64 = _p(keep["corners64"])
                d.obstacle_normals64 = _p(keep["onorm64"])
        d.dt = p.dt / p.substeps
        for q in range(3):
            d.gravity[q] = float(p.gravity[q])
            d.stiffness[q] = float(p.stiffness[q])
        d.damping = float(p.damping)
        d.epsilon_mt = float(p.epsilon_mt)
        d.response_margin = float(p.response_margin)
        d.epsilon_mt64 = float(p.epsilon_mt)
        d.response_margin64 = float(p.response_margin)
        d.fixed_point_scale = int(p.fixed_point_scale)
        d.substeps = int(p.substeps)
        d.cell_size = float(cell_size) if cell_size else 0.0
        if stream is not None:
            d.stream = _stream_handle(stream)
        h = ctypes.c_void_p()
        N.check(self._lib.cs_create(ctypes.byref(d), ctypes.byref(h)))
        self._handle = h
        self.kparams = d  # the baked parameter block (engine.py:274-285 KernelParams)
        self.stencil = stencil is not None and not force_csr and precision != "fp64"
        self._fused_normals = self.stencil and kernel != "tile" and normals != "split"
        self.frame_count = 0
        self.buffers = PipelineBuffers(self)
        self._has_obstacle = has_obs

    @classmethod
    def from_grid(cls, nx: int, ny: int, params=None, *, width: float = 1.0,
                  height: float = 1.0, total_mass: float | None = None, pinned_rows="first",
                  orientation: str = "hanging", row_lo: int = 0, row_hi: int | None = None,
                  device=None, precision: str = "fast", graph: bool = True, stream=None,
                  kernel: str = "pair", normals: str = "auto", seam: str = "kernel"):
        """An engine for generate_cloth_grid(nx, ny, width, height, total_mass,
        pinned_rows) (mesh.py:223-317) -- rows [row_lo, row_hi) of it for a
        row band -- generated on the device (cs_create_grid): no per-node or
        per-spring array is built on the host.  orientation "hanging" applies
        the hanging scene's rotation (scenes.py _rotate_xz_to_xy), "xz" keeps
        the generation plane.  Fast or fixed arithmetic (the float64 mode
        needs the mesh's arrays: Engine(mesh, ...))."""
        if precision not in ("fast", "fixed"):
            raise ValueError("Engine.from_grid builds fast or fixed engines")
        if orientation not in ("hanging", "xz"):
            raise ValueError("orientation must be 'hanging' or 'xz'")
        from .mesh import GridCloth

        row_hi = ny if row_hi is None else row_hi
        cloth = GridCloth(nx, ny, width, height, total_mass, pinned_rows, row_lo, row_hi,
                          orientation)
        self = cls.__new__(cls)
        self.mesh, self.obstacle = cloth, None
        self.params = params if params is not None else SimParams()
        self.device = device if device is not None else get_adapter()
        self.pair_budget = DEFAULT_PAIR_BUDGET
        self.precision = precision
        self._lib = N.load()
        self._handle = None
        p = self.params
        n = cloth.num_nodes
        pitch_nodes = ((nx + 31) // 32 * 32) * (row_hi - row_lo)
        state_bytes = 2 * 6 * pitch_nodes * 4
        self.layout = Layout(n, cloth.num_springs, cloth.num_triangles,
                             cloth.num_unique_edges, 0, state_bytes,
                             state_bytes + 3 * pitch_nodes * 4 + 24 * pitch_nodes)
        free, _ = self.device.mem_info()
        self.layout.validate(free)
        self.pairs_per_frame = 0
        g = N.CsGridDesc()
        g.abi_version = N.ABI_VERSION
        g.flags = _engine_flags(p, precision, graph, False, kernel, normals, "tri", seam)
        g.nx, g.ny, g.row_lo, g.row_hi = nx, ny, row_lo, row_hi
        g.width, g.height, g.total_mass = width, height, cloth.total_mass
        g.orientation = 1 if orientation == "hanging" else 0
        rows = np.ascontiguousarray(cloth.pinned_row_list, dtype=np.int32)
        g.num_pinned_rows = len(rows)
        g.pinned_rows = rows.ctypes.data if len(rows) else None
        g.dt = p.dt / p.substeps
        for q in range(3):
            g.gravity[q] = float(p.gravity[q])
            g.stiffness[q] = float(p.stiffness[q])
        g.damping = float(p.damping)
        g.epsilon_mt = float(p.epsilon_mt)
        g.response_margin = float(p.response_margin)
        g.fixed_point_scale = int(p.fixed_point_scale)
        g.substeps = int(p.substeps)
        if stream is not None:
            g.stream = _stream_handle(stream)
        h = ctypes.c_void_p()
        N.check(self._lib.cs_create_grid(ctypes.byref(g), ctypes.byref(h)))
        self._handle = h
        self.kparams = g
        self.stencil = True
        self._fused_normals = kernel != "tile" and normals != "split" and precision == "fast"
        self.frame_count = 0
        self.buffers = PipelineBuffers(self)
        self._has_obstacle = False
        return self

    # -- lifetime -----------------------------------------------------------------
    def close(self):
        if self._handle is not None and self._handle.value:
            self._lib.cs_destroy(self._handle)
        self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- properties ---------------------------------------------------------------
    @property
    def num_nodes(self) -> int:
        return self.layout.num_nodes

    @property
    def has_obstacle(self) -> bool:
        return self._has_obstacle

    @property
    def kernels_per_frame(self) -> int:
        c = ctypes.c_int32()
        N.check(self._lib.cs_kernels_per_frame(self._handle, ctypes.byref(c)))
        return c.value

    def broadphase_stats(self) -> dict:
        a = (ctypes.c_int64 * 4)()
        N.check(self._lib.cs_broadphase_stats(self._handle, a))
        return {"cells": a[0], "refs": a[1], "dims_x": a[2], "dims_yz": a[3]}

    def broadphase_dump(self) -> dict:
        """The device-built broad-phase grid (cs_broadphase_dump): origin,
        1/cell, cell edge (f32), dims, the sorted (cell key, triangle)
        references and each cell's [begin, end) into them."""
        st = self.broadphase_stats()
        geo = (ctypes.c_float * 8)()
        dims = (ctypes.c_int32 * 3)()
        keys = np.empty(st["refs"], dtype=np.uint32)
        tris = np.empty(st["refs"], dtype=np.uint32)
        beg = np.empty(st["cells"], dtype=np.uint32)
        end = np.empty(st["cells"], dtype=np.uint32)
        N.check(self._lib.cs_broadphase_dump(self._handle, geo, dims, keys.ctypes.data,
                                             tris.ctypes.data, beg.ctypes.data, end.ctypes.data))
        return {"origin": np.array(geo[0:3], dtype=np.float32), "inv_cell": np.float32(geo[3]),
                "cell": np.float32(geo[4]), "dims": tuple(dims), "ref_keys": keys,
                "ref_tris": tris, "cell_begin": beg, "cell_end": end}

    # -- runtime ------------------------------------------------------------------
    def set_external_accel(self, accel=None) -> None:
        """Constant per-node acceleration (N, 3), or None to clear (engine.py:297-302)."""
        if accel is None:
            N.check(self._lib.cs_write(self._handle, N.BUF_EXT_ACCEL, None))
            return
        if _is_cuda_tensor(accel):
            self._write(N.BUF_EXT_ACCEL, accel)
            return
        a = np.ascontiguousarray(np.broadcast_to(np.asarray(accel, dtype=_F32),
                                                 (self.num_nodes, 3)))
        N.check(self._lib.cs_write(self._handle, N.BUF_EXT_ACCEL, a.ctypes.data))

    def step(self, readback: bool = False, debug: bool = False) -> StepResult:
        """Advance one frame (engine.py:304-344)."""
        frame = self.frame_count
        snaps = {}
        if debug:
            L, h = self._lib, self._handle
            # the gather keeps no force accumulator: "zeroed" forces are the
            # registers each node starts its sum from
            snaps["forces_after_zero"] = np.zeros((self.num_nodes, 3), dtype=np.int32)
            N.check(L.cs_run_pass(h, N.PASS_FORCE_INTEGRATE))
            if self.has_obstacle:
                N.check(L.cs_run_pass(h, N.PASS_DETECT))
                snaps["accumulator_before_respond"] = self.read_accumulator_raw()
                snaps["counts_before_respond"] = self.read_counts()
                N.check(L.cs_run_pass(h, N.PASS_RESPOND))
                snaps["accumulator_after_respond"] = self.read_accumulator_raw()
                snaps["counts_after_respond"] = self.read_counts()
            N.check(L.cs_run_pass(h, N.PASS_NORMALS))
        else:
            N.check(self._lib.cs_step(self._handle, 1))
        self.frame_count += 1
        res = StepResult(self, frame, debug=snaps)
        if readback:
            res.positions = self.read_positions()
        return res

    def step_frames(self, frames: int) -> None:
        """Advance `frames` frames with one call (graph replays, no sync)."""
        N.check(self._lib.cs_step(self._handle, int(frames)))
        self.frame_count += int(frames)

    def simulate(self, frames: int, out=None) -> np.ndarray:
        """Advance `frames` frames and return every frame's positions as a
        (frames, N, 3) float32 array -- `step(readback=True)` for a whole run
        (engine.py:341-343), with frame f's device->host copy overlapping the
        computation of frame f+1.  `out` should be page-locked
        (`pinned_empty`); a pageable array works but copies synchronously."""
        frames = int(frames)
        if out is None:
            out = pinned_empty((frames, self.num_nodes, 3))
        if out.shape != (frames, self.num_nodes, 3) or out.dtype != np.float32 \
                or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous float32 array of shape (frames, N, 3)")
        N.check(self._lib.cs_record(self._handle, frames, out.ctypes.data))
        self.frame_count += frames
        return out

    def enable_contact_log(self, capacity: int = 1 << 22) -> None:
        """Record every (cloth node, obstacle triangle) contact of later
        frames (parity checks); capacity 0 switches it off."""
        N.check(self._lib.cs_contact_log(self._handle, int(capacity)))
        self._clog_cap = int(capacity)

    def read_contacts(self) -> np.ndarray:
        """The last frame's contacts as an (n, 2) int32 array of (node,
        triangle), one row per pushed node per hit (duplicates kept)."""
        cap = getattr(self, "_clog_cap", 0)
        out = np.empty((max(cap, 1), 2), dtype=np.int32)
        n = ctypes.c_int64()
        N.check(self._lib.cs_read_contacts(self._handle, out.ctypes.data, cap, ctypes.byref(n)))
        if n.value > cap:
            raise RuntimeError(f"contact log truncated: {n.value} contacts, capacity {cap}")
        return out[: n.value].copy()

    def run_respond_pass(self) -> int:
        """Respond kernel alone (engine.py:346-352); returns nodes moved."""
        r = ctypes.c_int64()
        N.check(self._lib.cs_respond(self._handle, ctypes.byref(r)))
        return int(r.value)

    def inject_response(self, node: int, offset, count: int = 1) -> None:
        """Write one node's accumulator cells (engine.py:354-358)."""
        enc = encode_values(np.asarray(offset, dtype=_F32), self.params.fixed_point_scale)
        raw = (ctypes.c_int32 * 3)(*[int(x) for x in enc])
        N.check(self._lib.cs_inject_response(self._handle, int(node), raw, int(count)))

    def synchronize(self) -> None:
        N.check(self._lib.cs_synchronize(self._handle))

    @property
    def stream_handle(self) -> int:
        """The engine's cudaStream_t (for events / torch.cuda.ExternalStream)."""
        s = ctypes.c_void_p()
        N.check(self._lib.cs_stream(self._handle, ctypes.byref(s)))
        return s.value or 0

    @property
    def stencil_bytes_per_frame(self) -> int:
        """Algorithmic HBM bytes of one frame's spring/integrate/normals pass:
        24 B read + 24 B written (pos, vel) + 12 B normals per node, fused
        (SURVEY.md 8(d)); 72 B when the normals run as a separate pass."""
        return (60 if self._fused_normals else 72) * self.num_nodes

    def _frame_hits(self, frame):
        hits, resp = ctypes.c_int64(), ctypes.c_int64()
        N.check(self._lib.cs_frame_hits(self._handle, int(frame), ctypes.byref(hits),
                                        ctypes.byref(resp)))
        return int(hits.value), int(resp.value)

    def stats(self) -> dict:
        s = N.CsStats()
        N.check(self._lib.cs_frame_stats(self._handle, ctypes.byref(s)))
        return {"hits": s.hits, "responded": s.responded, "frames": s.frames,
                "hit_counter": s.hit_counter}

    # -- transfers ------------------------------------------------------------------
    # Every read_* / write_* accepts either host arrays (the reference's numpy
    # readbacks, engine.py:362-378) or torch CUDA tensors: those move device
    # to device (cs_read_device / cs_write_device), enqueued on the tensor's
    # device's current torch stream and event-ordered against the engine's
    # own stream -- no host copy, no synchronisation.
    @property
    def cuda_device(self) -> int:
        d = ctypes.c_int32()
        N.check(self._lib.cs_device(self._handle, ctypes.byref(d)))
        return d.value

    def _check_tensor(self, t, dtype, shape):
        if str(t.dtype) != _TORCH_DTYPE_NAMES[np.dtype(dtype)] or tuple(t.shape) != shape \
                or not t.is_contiguous():
            raise ValueError(f"tensor must be a contiguous {_TORCH_DTYPE_NAMES[np.dtype(dtype)]} "
                             f"CUDA tensor of shape {shape}")
        if t.device.index != self.cuda_device:
            raise ValueError(f"tensor is on cuda:{t.device.index}, the engine on "
                             f"cuda:{self.cuda_device}")

    @staticmethod
    def _torch_stream(t) -> int:
        """The tensor's device's current torch stream as a cudaStream_t; torch's
        default stream is the legacy default stream, handle 0, which the C ABI
        reads as "the engine's stream" -- pass cudaStreamLegacy (1) instead."""
        import torch

        return torch.cuda.current_stream(t.device).cuda_stream or 1

    def _read(self, buf, dtype, comps, out=None):
        shape = (self.num_nodes, comps) if comps > 1 else (self.num_nodes,)
        if out is not None and _is_cuda_tensor(out):
            self._check_tensor(out, dtype, shape)
            N.check(self._lib.cs_read_device(self._handle, buf, out.data_ptr(),
                                             self._torch_stream(out)))
            return out
        if out is None:
            out = np.empty(shape, dtype=dtype)
        N.check(self._lib.cs_read(self._handle, buf, out.ctypes.data))
        return out

    def _write(self, buf, arr, dtype=np.float32):
        if _is_cuda_tensor(arr):
            self._check_tensor(arr, dtype, (self.num_nodes, 3))
            N.check(self._lib.cs_write_device(self._handle, buf, arr.data_ptr(),
                                              self._torch_stream(arr)))
            return
        N.check(self._lib.cs_write(self._handle, buf, np.ascontiguousarray(arr).ctypes.data))

    def set_stream(self, stream) -> None:
        """Launch every later frame / transfer on `stream` (a torch.cuda.Stream
        or a cudaStream_t handle); work already enqueued stays ordered first."""
        handle = int(getattr(stream, "cuda_stream", stream))
        N.check(self._lib.cs_set_stream(self._handle, handle))

    def read_positions(self, out=None) -> np.ndarray:
        return self._read(N.BUF_POSITIONS, _F32, 3, out)

    def read_velocities(self, out=None) -> np.ndarray:
        return self._read(N.BUF_VELOCITIES, _F32, 3, out)

    def read_normals(self, out=None) -> np.ndarray:
        return self._read(N.BUF_NORMALS, _F32, 3, out)

    def read_normals_lagged(self, out=None) -> np.ndarray:
        """The normals the last fused step kernel produced: those of the
        previous frame's final state (a one-frame lag), read without the
        stand-alone recompute read_normals() does for the current state."""
        return self._read(N.BUF_NORMALS_LAGGED, _F32, 3, out)

    def read_previous_positions(self, out=None) -> np.ndarray:
        return self._read(N.BUF_PREV_POSITIONS, _F32, 3, out)

    def read_forces_raw(self) -> np.ndarray:
        """Spring-only i32 fixed-point forces of the last spring pass
        (engine.py:368-369), recomputed from the pre-step state with the
        reference engine's exact arithmetic."""
        return self._read(N.BUF_FORCES_RAW, np.int32, 3)

    def read_accumulator_raw(self, out=None) -> np.ndarray:
        return self._read(N.BUF_ACCUMULATOR, np.int32, 3, out)

    def read_counts(self, out=None) -> np.ndarray:
        return self._read(N.BUF_COUNTS, np.int32, 1, out)

    def read_positions64(self, out=None) -> np.ndarray:
        return self._read(N.BUF_POSITIONS64, np.float64, 3, out)

    def read_velocities64(self, out=None) -> np.ndarray:
        return self._read(N.BUF_VELOCITIES64, np.float64, 3, out)

    def write_positions(self, arr) -> None:
        self._write(N.BUF_POSITIONS, arr if _is_cuda_tensor(arr) else np.asarray(arr, dtype=_F32))

    def write_velocities(self, arr) -> None:
        self._write(N.BUF_VELOCITIES, arr if _is_cuda_tensor(arr) else np.asarray(arr, dtype=_F32))

    def write_state64(self, pos=None, vel=None) -> None:
        for buf, a in ((N.BUF_POSITIONS64, pos), (N.BUF_VELOCITIES64, vel)):
            if a is not None:
                self._write(buf, a if _is_cuda_tensor(a) else np.asarray(a, dtype=np.float64),
                            dtype=np.float64)

    def render_snapshot(self, size=(320, 240), axis: str = "y", obstacle: bool = True) -> np.ndarray:
        """uint8 (H, W, 3) pixels of the current frame's snapshot (io.py:225-287),
        rendered from device memory: only the image crosses PCIe."""
        from .snapshot import engine_snapshot

        return engine_snapshot(self, size=size, axis=axis, obstacle=obstacle)

    def snapshot_png(self, path, size=(320, 240), axis: str = "y", obstacle: bool = True) -> None:
        """PNG of the current frame: the pixels of the reference's
        snapshot_png(path, read_positions().astype(float64), mesh.triangles,
        obstacle...) (bench.py:186-198), without the positions readback."""
        from .snapshot import _save_png

        _save_png(path, self.render_snapshot(size=size, axis=axis, obstacle=obstacle))

    def state_plane(self, which: int):
        """(device pointer, pitch) of plane `which` (x y z vx vy vz) of the
        current state -- zero-copy access for the row-band halo exchange."""
        ptr, pitch = ctypes.c_void_p(), ctypes.c_int64()
        N.check(self._lib.cs_state_plane(self._handle, int(which), ctypes.byref(ptr),
                                         ctypes.byref(pitch)))
        return ptr.value, pitch.value


def build_pipeline(mesh, obstacle=None, params=None, device=None,
                   pair_budget: int = DEFAULT_PAIR_BUDGET, **kw) -> Engine:
    """Validate and build a ready Engine (engine.py:381-389)."""
    return Engine(mesh, obstacle, params, device, pair_budget, **kw)


def step_gpu(engine: Engine, readback: bool = False, debug: bool = False) -> StepResult:
    """Function-style alias of Engine.step (engine.py:392-394)."""
    return engine.step(readback=readback, debug=debug)
