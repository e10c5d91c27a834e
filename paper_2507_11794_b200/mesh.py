"""Cloth and obstacle geometry for the B200 engine (inputs of the hot path).

Mirrors the reference data model (clothsim/mesh.py) so reference callers can
switch packages: ``ClothMesh``, ``TriangleMesh``, ``SimParams``,
``generate_cloth_grid``, ``generate_icosphere``, ``compute_face_normals``,
``compute_vertex_normals``, ``unique_edges``, ``spring_count_formula``.

The grid builder is vectorised (the reference loops in Python, ~100 s at
4096^2) but reproduces the reference topology bit for bit: node (i, j) at
(i*w/(nx-1), 0, j*h/(ny-1)), flat index j*nx+i; springs ordered structural
(+i, +j per node), shear (two per cell), bend (+2i, +2j per node); triangles
(v00, v01, v10), (v10, v01, v11) per cell (mesh.py:223-317).  The Engine also
accepts the reference's own ClothMesh objects (duck typing).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

__all__ = [
    "SpringKind",
    "ClothMesh",
    "TriangleMesh",
    "SimParams",
    "generate_cloth_grid",
    "generate_icosphere",
    "generate_uv_sphere",
    "compute_face_normals",
    "compute_vertex_normals",
    "spring_count_formula",
    "unique_edges",
    "grid_unique_edges",
    "grid_springs",
    "grid_triangles",
]


class SpringKind(IntEnum):
    STRUCTURAL = 0
    SHEAR = 1
    BEND = 2


@dataclass
class ClothMesh:
    """Regular nx x ny cloth: SoA node arrays, spring table, triangulation
    (field meaning as mesh.py:75-124)."""

    nx: int
    ny: int
    positions: np.ndarray            # (N, 3) float64 construction pose
    masses: np.ndarray               # (N,) float64
    pinned: np.ndarray               # (N,) bool
    spring_indices: np.ndarray       # (S, 2) int32
    spring_rest_lengths: np.ndarray  # (S,) float64
    spring_kinds: np.ndarray         # (S,) int32
    triangles: np.ndarray            # (C, 3) int32

    @property
    def num_nodes(self) -> int:
        return self.nx * self.ny

    @property
    def num_springs(self) -> int:
        return len(self.spring_indices)

    def node_index(self, i: int, j: int) -> int:
        if not (0 <= i < self.nx and 0 <= j < self.ny):
            raise IndexError(f"grid coordinate ({i}, {j}) outside {self.nx}x{self.ny}")
        return j * self.nx + i


@dataclass
class TriangleMesh:
    """Static obstacle: vertices, triangles, unit face normals (mesh.py:127-149)."""

    vertices: np.ndarray
    triangles: np.ndarray
    face_normals: np.ndarray = field(default=None)

    def __post_init__(self) -> None:
        self.vertices = np.asarray(self.vertices, dtype=np.float64)
        self.triangles = np.asarray(self.triangles, dtype=np.int32)
        if self.triangles.size and self.triangles.max() >= len(self.vertices):
            raise ValueError("triangle references a vertex that does not exist")
        if self.face_normals is None:
            self.face_normals = compute_face_normals(self.vertices, self.triangles)

    @property
    def num_vertices(self) -> int:
        return len(self.vertices)

    @property
    def num_triangles(self) -> int:
        return len(self.triangles)


@dataclass
class SimParams:
    """Simulation coefficients (mesh.py:152-204); same defaults and checks."""

    dt: float = 0.016
    gravity: tuple = (0.0, -9.8, 0.0)
    stiffness: object = 50.0
    damping: float = 0.5
    epsilon_mt: float = 1e-6
    response_margin: float = 1e-3
    fixed_point_scale: int = 1 << 16
    workgroup_size: int = 256
    substeps: int = 1
    explicit_euler: bool = False
    average_response: bool = True

    def __post_init__(self) -> None:
        if not self.dt > 0.0:
            raise ValueError("dt must be positive")
        if np.shape(self.gravity) != (3,):
            raise ValueError("gravity must be a 3-vector")
        self.gravity = tuple(float(g) for g in self.gravity)
        if np.isscalar(self.stiffness):
            self.stiffness = (float(self.stiffness),) * 3
        else:
            self.stiffness = tuple(float(s) for s in self.stiffness)
        if len(self.stiffness) != 3:
            raise ValueError("stiffness needs one value or (structural, shear, bend)")
        if any(s < 0.0 for s in self.stiffness):
            raise ValueError("stiffness must be non-negative")
        if self.damping < 0.0:
            raise ValueError("damping must be non-negative")
        if self.epsilon_mt <= 0.0:
            raise ValueError("epsilon_mt must be positive")
        if self.response_margin < 0.0:
            raise ValueError("response_margin must be non-negative")
        if int(self.fixed_point_scale) < 1:
            raise ValueError("fixed_point_scale must be >= 1")
        self.fixed_point_scale = int(self.fixed_point_scale)
        if int(self.workgroup_size) < 1:
            raise ValueError("workgroup_size must be >= 1")
        self.workgroup_size = int(self.workgroup_size)
        if int(self.substeps) < 1:
            raise ValueError("substeps must be >= 1")
        self.substeps = int(self.substeps)

    def stiffness_for(self, kind: int) -> float:
        return self.stiffness[int(kind)]


def spring_count_formula(nx: int, ny: int) -> tuple:
    """(structural, shear, bend) spring counts of an nx x ny grid (mesh.py:207-220)."""
    if nx < 2 or ny < 2:
        raise ValueError("grid needs at least 2 nodes per side")
    return (nx * (ny - 1) + ny * (nx - 1), 2 * (nx - 1) * (ny - 1),
            nx * max(ny - 2, 0) + ny * max(nx - 2, 0))


def _interleave(cands):
    """Flatten per-item candidate columns [(a, b, valid), ...] in item-major,
    column-minor order, keeping valid entries only."""
    a = np.stack([c[0] for c in cands], axis=1).ravel()
    b = np.stack([c[1] for c in cands], axis=1).ravel()
    ok = np.stack([c[2] for c in cands], axis=1).ravel()
    return a[ok], b[ok]


def grid_springs(nx: int, ny: int):
    """(S,2) int32 endpoints and (S,) int32 kinds in the reference order
    (mesh.py:274-289): per node (row-major) structural +i then +j; per cell
    the two shears; per node bend +2i then +2j -- built row block by row
    block straight into int32 (no per-spring Python, no int64 temporaries)."""
    i32 = np.int32
    cols = np.arange(nx, dtype=i32)
    base = (np.arange(ny, dtype=i32) * i32(nx))[:, None]
    # structural: rows j < ny-1 hold 2(nx-1)+1 springs, the last row nx-1
    st = np.empty((ny - 1, 2 * nx - 1, 2), i32)
    st[:, 0:2 * nx - 2:2, 0] = base[:-1] + cols[:-1]
    st[:, 0:2 * nx - 2:2, 1] = base[:-1] + cols[:-1] + 1
    st[:, 1:2 * nx - 2:2, 0] = base[:-1] + cols[:-1]
    st[:, 1:2 * nx - 2:2, 1] = base[:-1] + cols[:-1] + nx
    st[:, 2 * nx - 2, 0] = base[:-1, 0] + nx - 1
    st[:, 2 * nx - 2, 1] = base[:-1, 0] + 2 * nx - 1
    last = np.stack([base[-1, 0] + cols[:-1], base[-1, 0] + cols[:-1] + 1], axis=1)
    # shear: per cell (c, c+nx+1), (c+1, c+nx)
    c = base[:-1] + cols[:-1]
    sh = np.empty((ny - 1, nx - 1, 2, 2), i32)
    sh[:, :, 0, 0] = c
    sh[:, :, 0, 1] = c + nx + 1
    sh[:, :, 1, 0] = c + 1
    sh[:, :, 1, 1] = c + nx
    # bend: rows j < ny-2 hold 2(nx-2)+2 springs, the last two rows nx-2 each
    m = max(nx - 2, 0)
    bd = np.empty((max(ny - 2, 0), 2 * m + min(nx, 2), 2), i32)
    if ny > 2:
        b0 = base[:-2]
        bd[:, 0:2 * m:2, 0] = b0 + cols[:m]
        bd[:, 0:2 * m:2, 1] = b0 + cols[:m] + 2
        bd[:, 1:2 * m:2, 0] = b0 + cols[:m]
        bd[:, 1:2 * m:2, 1] = b0 + cols[:m] + 2 * nx
        tail = cols[m:]
        bd[:, 2 * m:, 0] = b0 + tail
        bd[:, 2 * m:, 1] = b0 + tail + 2 * nx
    tail_rows = base[max(ny - 2, 0):]
    bl = np.stack([(tail_rows + cols[:m]).ravel(), (tail_rows + cols[:m] + 2).ravel()], axis=1)
    pairs = np.concatenate([st.reshape(-1, 2), last, sh.reshape(-1, 2), bd.reshape(-1, 2),
                            bl.astype(i32)])
    n_st = st.shape[0] * st.shape[1] + len(last)
    n_sh = sh.shape[0] * sh.shape[1] * 2
    kinds = np.empty(len(pairs), i32)
    kinds[:n_st] = 0
    kinds[n_st:n_st + n_sh] = 1
    kinds[n_st + n_sh:] = 2
    return pairs, kinds


def grid_families(per_spring, nx: int, ny: int):
    """Views of a per-spring array laid out in grid_springs order, grouped by
    stencil family: [+i], [+j], [shear +nx+1], [shear +nx-1], [bend +2],
    [bend +2nx] -- each a list of strided views (no masks, no copies)."""
    m = max(nx - 2, 0)
    n_st = (ny - 1) * (2 * nx - 1)
    st = per_spring[:n_st].reshape(ny - 1, 2 * nx - 1)
    o = n_st
    last = per_spring[o:o + nx - 1]
    o += nx - 1
    n_sh = (ny - 1) * (nx - 1) * 2
    sh = per_spring[o:o + n_sh].reshape(ny - 1, nx - 1, 2)
    o += n_sh
    w = 2 * m + min(nx, 2)
    n_bd = max(ny - 2, 0) * w
    bd = per_spring[o:o + n_bd].reshape(max(ny - 2, 0), w)
    o += n_bd
    bl = per_spring[o:]
    return ([st[:, 0:2 * nx - 2:2], last], [st[:, 1:2 * nx - 2:2], st[:, 2 * nx - 2]],
            [sh[:, :, 0]], [sh[:, :, 1]], [bd[:, 0:2 * m:2], bl], [bd[:, 1:2 * m:2], bd[:, 2 * m:]])


def grid_triangles(nx: int, ny: int) -> np.ndarray:
    """(C,3) int32: per cell (v00, v01, v10), (v10, v01, v11) (mesh.py:296-305)."""
    i32 = np.int32
    v00 = (np.arange(ny - 1, dtype=i32) * i32(nx))[:, None] + np.arange(nx - 1, dtype=i32)
    t = np.empty((ny - 1, nx - 1, 2, 3), i32)
    t[..., 0, 0] = v00
    t[..., 0, 1] = v00 + nx
    t[..., 0, 2] = v00 + 1
    t[..., 1, 0] = v00 + 1
    t[..., 1, 1] = v00 + nx
    t[..., 1, 2] = v00 + nx + 1
    return t.reshape(-1, 3)


def grid_unique_edges(nx: int, ny: int) -> np.ndarray:
    """unique_edges(grid_triangles(nx, ny)) in closed form: node a's edges to
    larger indices are a+1 (if i < nx-1), a+nx-1 (the cell diagonal v10-v01,
    if i > 0 and j < ny-1) and a+nx (if j < ny-1), already in sorted order."""
    i32 = np.int32
    cols = np.arange(nx, dtype=i32)
    base = (np.arange(ny, dtype=i32) * i32(nx))[:, None]
    # rows j < ny-1: node 0 has (+1, +nx); nodes 1..nx-2 (+1, +nx-1, +nx);
    # node nx-1 (+nx-1, +nx) -> 3nx-2 edges per row; the last row nx-1
    e = np.empty((ny - 1, 3 * nx - 2, 2), i32)
    b0 = base[:-1, 0][:, None]
    e[:, 0, 0] = b0[:, 0]
    e[:, 0, 1] = b0[:, 0] + 1
    e[:, 1, 0] = b0[:, 0]
    e[:, 1, 1] = b0[:, 0] + nx
    mid = cols[1:nx - 1]
    if len(mid):
        e[:, 2:3 * nx - 4:3, 0] = b0 + mid
        e[:, 2:3 * nx - 4:3, 1] = b0 + mid + 1
        e[:, 3:3 * nx - 4:3, 0] = b0 + mid
        e[:, 3:3 * nx - 4:3, 1] = b0 + mid + nx - 1
        e[:, 4:3 * nx - 4:3, 0] = b0 + mid
        e[:, 4:3 * nx - 4:3, 1] = b0 + mid + nx
    e[:, 3 * nx - 4, 0] = b0[:, 0] + nx - 1
    e[:, 3 * nx - 4, 1] = b0[:, 0] + 2 * nx - 2
    e[:, 3 * nx - 3, 0] = b0[:, 0] + nx - 1
    e[:, 3 * nx - 3, 1] = b0[:, 0] + 2 * nx - 1
    last = np.stack([base[-1, 0] + cols[:-1], base[-1, 0] + cols[:-1] + 1], axis=1)
    return np.concatenate([e.reshape(-1, 2), last.astype(i32)])


def _grid_rest(xs, zs):
    """Rest lengths of grid_springs(len(xs), len(zs)) for the separable grid
    positions (xs[i], 0, zs[j]) of generate_cloth_grid, in the same block
    order and with the same float64 arithmetic as |p_b - p_a| =
    sqrt((dx^2 + dy^2) + dz^2) (mesh.py:293-294), dy = 0 -- from per-column
    and per-row tables instead of 100M-entry gathers."""
    nx, ny = len(xs), len(zs)
    z0 = np.zeros(1)

    def norm(dx, dz):
        return np.sqrt((dx * dx + z0 * z0) + dz * dz)

    ri = norm(xs[1:] - xs[:-1], z0)                    # struct +i, by i
    rj = norm(z0, zs[1:] - zs[:-1])                    # struct +j, by j
    rs = norm((xs[1:] - xs[:-1])[None, :], (zs[1:] - zs[:-1])[:, None])  # shears, by (j, i)
    m = max(nx - 2, 0)
    rbi = norm(xs[2:] - xs[:-2], z0) if m else np.zeros(0)   # bend +2i, by i
    rbj = norm(z0, zs[2:] - zs[:-2]) if ny > 2 else np.zeros(0)  # bend +2j, by j
    st = np.empty((ny - 1, 2 * nx - 1))
    st[:, 0:2 * nx - 2:2] = ri[None, :]
    st[:, 1:2 * nx - 2:2] = rj[:, None]
    st[:, 2 * nx - 2] = rj
    sh = np.empty((ny - 1, nx - 1, 2))
    sh[:, :, 0] = rs
    sh[:, :, 1] = rs  # (c+1 -> c+nx): dx = -(xs[i+1]-xs[i]), same square
    bd = np.empty((max(ny - 2, 0), 2 * m + min(nx, 2)))
    if ny > 2:
        bd[:, 0:2 * m:2] = rbi[None, :]
        bd[:, 1:2 * m:2] = rbj[:, None]
        bd[:, 2 * m:] = rbj[:, None]
    bl = np.tile(rbi, min(ny, 2))
    return np.concatenate([st.ravel(), ri, sh.ravel(), bd.ravel(), bl])


def _rest_lengths(positions, springs):
    """|p_b - p_a| in float64 with numpy's norm arithmetic ((dx^2+dy^2)+dz^2,
    no contraction) -- column by column instead of an (S,3) temporary."""
    a, b = springs[:, 0], springs[:, 1]
    acc = None
    for q in range(3):
        col = positions[:, q]
        d = col[b] - col[a]
        d *= d
        acc = d if acc is None else np.add(acc, d, out=acc)
    return np.sqrt(acc, out=acc)


def generate_cloth_grid(nx: int, ny: int, width: float = 1.0, height: float = 1.0,
                        total_mass: float = None, pinned_rows=None) -> ClothMesh:
    """Regular cloth grid in the xz-plane at y=0 (mesh.py:223-317)."""
    if nx < 2 or ny < 2:
        raise ValueError("grid needs at least 2 nodes per side")
    if width <= 0.0 or height <= 0.0:
        raise ValueError("cloth dimensions must be positive")
    n = nx * ny
    if total_mass is None:
        total_mass = 0.05 * n
    if total_mass <= 0.0:
        raise ValueError("total_mass must be positive")
    positions = np.zeros((n, 3), dtype=np.float64)
    positions[:, 0] = np.tile(np.linspace(0.0, width, nx), ny)
    positions[:, 2] = np.repeat(np.linspace(0.0, height, ny), nx)
    masses = np.full(n, total_mass / n, dtype=np.float64)
    pinned = np.zeros(n, dtype=bool)
    for j in _resolve_pinned_rows(pinned_rows, ny):
        pinned[j * nx:(j + 1) * nx] = True
    springs, kinds = grid_springs(nx, ny)
    rest = _grid_rest(np.linspace(0.0, width, nx), np.linspace(0.0, height, ny))
    return ClothMesh(nx=nx, ny=ny, positions=positions, masses=masses, pinned=pinned,
                     spring_indices=springs, spring_rest_lengths=rest, spring_kinds=kinds,
                     triangles=grid_triangles(nx, ny))


def grid_band(nx: int, ny: int, j0: int, j1: int, width: float = 1.0, height: float = 1.0,
              total_mass: float = None, pinned_rows=None) -> ClothMesh:
    """Rows [j0, j1) of generate_cloth_grid(nx, ny, ...) as a stand-alone
    ClothMesh: same node coordinates, masses and pins as the global grid, the
    grid topology of an nx x (j1-j0) sheet, and rest lengths computed from
    the same global coordinates -- so a row band steps exactly like the
    corresponding rows of the whole cloth (multi-GPU row bands, bands.py)."""
    if not (0 <= j0 < j1 <= ny) or j1 - j0 < 2:
        raise ValueError(f"band [{j0}, {j1}) outside a grid of {ny} rows")
    n = nx * ny
    if total_mass is None:
        total_mass = 0.05 * n
    lny = j1 - j0
    positions = np.zeros((nx * lny, 3), dtype=np.float64)
    positions[:, 0] = np.tile(np.linspace(0.0, width, nx), lny)
    positions[:, 2] = np.repeat(np.linspace(0.0, height, ny)[j0:j1], nx)
    masses = np.full(nx * lny, total_mass / n, dtype=np.float64)
    pinned = np.zeros(nx * lny, dtype=bool)
    for j in _resolve_pinned_rows(pinned_rows, ny):
        if j0 <= j < j1:
            pinned[(j - j0) * nx:(j - j0 + 1) * nx] = True
    springs, kinds = grid_springs(nx, lny)
    rest = _grid_rest(np.linspace(0.0, width, nx), np.linspace(0.0, height, ny)[j0:j1])
    return ClothMesh(nx=nx, ny=lny, positions=positions, masses=masses, pinned=pinned,
                     spring_indices=springs, spring_rest_lengths=rest, spring_kinds=kinds,
                     triangles=grid_triangles(nx, lny))


class GridCloth:
    """generate_cloth_grid's parameters without its arrays: what
    Engine.from_grid builds on the device (cs_create_grid).  Rows
    [row_lo, row_hi) of the nx x ny grid form the local sheet; the
    ClothMesh arrays (positions in the chosen orientation, masses, pins,
    springs, rest lengths, triangles) are built on the host only if
    something asks for them."""

    def __init__(self, nx, ny, width=1.0, height=1.0, total_mass=None, pinned_rows="first",
                 row_lo=0, row_hi=None, orientation="hanging"):
        if nx < 2 or ny < 2:
            raise ValueError("grid needs at least 2 nodes per side")
        self.full_nx, self.full_ny = nx, ny
        self.row_lo, self.row_hi = row_lo, (ny if row_hi is None else row_hi)
        if not (0 <= self.row_lo < self.row_hi <= ny) or self.row_hi - self.row_lo < 2:
            raise ValueError(f"local rows [{row_lo}, {row_hi}) outside a grid of {ny} rows")
        self.width, self.height = float(width), float(height)
        self.total_mass = float(total_mass) if total_mass is not None else 0.05 * nx * ny
        self.pinned_rows = pinned_rows
        self.pinned_row_list = _resolve_pinned_rows(pinned_rows, ny)
        self.orientation = orientation
        self.nx, self.ny = nx, self.row_hi - self.row_lo
        self._mesh = None

    @property
    def num_nodes(self) -> int:
        return self.nx * self.ny

    @property
    def num_springs(self) -> int:
        return sum(spring_count_formula(self.nx, self.ny))

    @property
    def num_triangles(self) -> int:
        return 2 * (self.nx - 1) * (self.ny - 1)

    @property
    def num_unique_edges(self) -> int:
        return (self.nx - 1) * self.ny + self.nx * (self.ny - 1) + (self.nx - 1) * (self.ny - 1)

    def materialize(self) -> ClothMesh:
        """The local sheet as a ClothMesh (host arrays, vectorised builders)."""
        if self._mesh is None:
            m = grid_band(self.full_nx, self.full_ny, self.row_lo, self.row_hi, self.width,
                          self.height, total_mass=self.total_mass, pinned_rows=self.pinned_rows)
            if self.orientation == "hanging":  # scenes._rotate_xz_to_xy
                rot = np.zeros_like(m.positions)
                rot[:, 0] = m.positions[:, 0]
                rot[:, 1] = -m.positions[:, 2]
                m.positions = rot
            self._mesh = m
        return self._mesh

    def __getattr__(self, name):
        if name in ("positions", "masses", "pinned", "spring_indices", "spring_rest_lengths",
                    "spring_kinds", "triangles"):
            return getattr(self.materialize(), name)
        raise AttributeError(name)


def band_of_mesh(mesh, nx: int, ny: int, rest6, j0: int, j1: int) -> ClothMesh:
    """Rows [j0, j1) of an nx x ny grid ClothMesh as a stand-alone sheet for
    a row band: the global node data of those rows, the grid topology of an
    nx x (j1-j0) sheet, and each spring family's rest length `rest6` (the
    global mesh's, engine._grid_stencil_rest) -- so the band's stencil
    coefficients are the global ones bit for bit, whatever pose the scene
    moved the cloth into after generate_cloth_grid."""
    if not (0 <= j0 < j1 <= ny) or j1 - j0 < 2:
        raise ValueError(f"band [{j0}, {j1}) outside a grid of {ny} rows")
    lny = j1 - j0
    sl = slice(j0 * nx, j1 * nx)
    springs, kinds = grid_springs(nx, lny)
    rest = np.empty(len(springs))
    for value, views in zip(rest6, grid_families(rest, nx, lny)):
        for v in views:
            v[...] = value
    return ClothMesh(nx=nx, ny=lny, positions=np.array(mesh.positions[sl], dtype=np.float64),
                     masses=np.array(mesh.masses[sl], dtype=np.float64),
                     pinned=np.array(mesh.pinned[sl], dtype=bool), spring_indices=springs,
                     spring_rest_lengths=rest, spring_kinds=kinds,
                     triangles=grid_triangles(nx, lny))


def _resolve_pinned_rows(pinned_rows, ny: int):
    if pinned_rows is None or (isinstance(pinned_rows, str) and pinned_rows == "none"):
        return []
    if isinstance(pinned_rows, str):
        if pinned_rows == "first":
            return [0]
        if pinned_rows == "last":
            return [ny - 1]
        raise ValueError(f"unknown pinned_rows {pinned_rows!r}")
    rows = [int(j) for j in pinned_rows]
    for j in rows:
        if not 0 <= j < ny:
            raise ValueError(f"pinned row {j} outside grid with ny={ny}")
    return rows


# --------------------------------------------------------------------------------
# obstacles
# --------------------------------------------------------------------------------
_PHI = (1.0 + math.sqrt(5.0)) / 2.0
# 12 icosahedron vertices (three golden rectangles) and its 20 outward faces,
# in the reference's order (mesh.py:334-347)
_ICO_V = np.array([
    (-1, _PHI, 0), (1, _PHI, 0), (-1, -_PHI, 0), (1, -_PHI, 0),
    (0, -1, _PHI), (0, 1, _PHI), (0, -1, -_PHI), (0, 1, -_PHI),
    (_PHI, 0, -1), (_PHI, 0, 1), (-_PHI, 0, -1), (-_PHI, 0, 1)], dtype=np.float64)
_ICO_F = np.array([
    (0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
    (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
    (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
    (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)], dtype=np.int64)


def generate_icosphere(subdivisions: int, radius: float = 1.0, center=(0.0, 0.0, 0.0)) -> TriangleMesh:
    """Subdivided icosahedron on a sphere (mesh.py:350-387): 20*4^k faces.

    Each level splits a face (a, b, c) into (a, ab, ca), (b, bc, ab),
    (c, ca, bc), (ab, bc, ca); an edge's midpoint vertex is created the first
    time a face (in face order) visits the edge, checked in the order ab, bc,
    ca -- the same numbering the reference produces.
    """
    if subdivisions < 0:
        raise ValueError("subdivisions must be >= 0")
    if radius <= 0.0:
        raise ValueError("radius must be positive")
    verts = [v / np.linalg.norm(v) for v in _ICO_V]
    faces = _ICO_F.copy()
    for _ in range(subdivisions):
        mid = {}
        out = np.empty((4 * len(faces), 3), dtype=np.int64)
        for f, (a, b, c) in enumerate(faces.tolist()):
            ids = []
            for u, v in ((a, b), (b, c), (c, a)):
                key = (u, v) if u < v else (v, u)
                k = mid.get(key)
                if k is None:
                    m = verts[u] + verts[v]
                    m /= np.linalg.norm(m)
                    verts.append(m)
                    k = mid[key] = len(verts) - 1
                ids.append(k)
            ab, bc, ca = ids
            out[4 * f:4 * f + 4] = ((a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca))
        faces = out
    vertices = np.array(verts) * radius + np.asarray(center, dtype=np.float64)
    return TriangleMesh(vertices=vertices, triangles=faces.astype(np.int32))


def generate_uv_sphere(slices: int = 224, stacks: int = 224, radius: float = 0.3,
                       center=(0.0, 0.0, 0.0)) -> TriangleMesh:
    """Procedural latitude/longitude sphere, outward (CCW from outside) faces.

    slices x stacks = 224 x 224 gives 49,954 vertices and 99,904 triangles: the
    paper's Dragon class (50K vertices / 100K triangles), used by
    BASELINE configs 3 and 4.
    """
    if slices < 3 or stacks < 2:
        raise ValueError("need slices >= 3 and stacks >= 2")
    theta = np.pi * np.arange(1, stacks) / stacks            # polar angle of the rings
    phi = 2.0 * np.pi * np.arange(slices) / slices
    st, ct = np.sin(theta)[:, None], np.cos(theta)[:, None]
    ring = np.stack([st * np.cos(phi)[None, :], np.broadcast_to(ct, (stacks - 1, slices)),
                     st * np.sin(phi)[None, :]], axis=-1).reshape(-1, 3)
    verts = np.concatenate([[[0.0, 1.0, 0.0]], ring, [[0.0, -1.0, 0.0]]]) * radius
    verts = verts + np.asarray(center, dtype=np.float64)
    top, bot = 0, 1 + (stacks - 1) * slices
    s = np.arange(slices)
    s1 = (s + 1) % slices
    tris = [np.stack([np.full(slices, top), 1 + s1, 1 + s], 1)]
    for r in range(stacks - 2):
        a = 1 + r * slices + s
        b = 1 + r * slices + s1
        c = 1 + (r + 1) * slices + s
        d = 1 + (r + 1) * slices + s1
        tris.append(np.stack([np.stack([a, b, c], 1), np.stack([b, d, c], 1)], 1).reshape(-1, 3))
    last = 1 + (stacks - 2) * slices
    tris.append(np.stack([last + s, last + s1, np.full(slices, bot)], 1))
    return TriangleMesh(vertices=verts, triangles=np.concatenate(tris).astype(np.int32))


def compute_face_normals(vertices: np.ndarray, triangles: np.ndarray) -> np.ndarray:
    """Unit float64 face normals; zero-area faces get +y (mesh.py:390-401)."""
    v = np.asarray(vertices, dtype=np.float64)
    t = np.asarray(triangles)
    n = np.cross(v[t[:, 1]] - v[t[:, 0]], v[t[:, 2]] - v[t[:, 0]])
    length = np.linalg.norm(n, axis=1)
    ok = length > 1e-30
    out = np.tile(np.array([0.0, 1.0, 0.0]), (len(t), 1))
    out[ok] = n[ok] / length[ok, None]
    return out


def compute_vertex_normals(mesh, positions: np.ndarray = None) -> np.ndarray:
    """Host float64 vertex normals (mesh.py:404-434), for inspection only --
    the engine computes normals on the device every frame."""
    if positions is None:
        positions = getattr(mesh, "positions", None)
        if positions is None:
            positions = mesh.vertices
    p = np.asarray(positions, dtype=np.float64)
    t = np.asarray(mesh.triangles)
    n = np.cross(p[t[:, 1]] - p[t[:, 0]], p[t[:, 2]] - p[t[:, 0]])
    length = np.linalg.norm(n, axis=1)
    ok = length > 1e-30
    face = np.zeros_like(n)
    face[ok] = n[ok] / length[ok, None]
    acc = np.zeros_like(p)
    for corner in range(3):
        np.add.at(acc, t[:, corner], face)
    ln = np.linalg.norm(acc, axis=1)
    good = ln > 1e-30
    out = np.tile(np.array([0.0, 1.0, 0.0]), (len(p), 1))
    out[good] = acc[good] / ln[good, None]
    return out


def unique_edges(triangles: np.ndarray) -> np.ndarray:
    """Sorted undirected edge set of a triangulation (mesh.py:437-442)."""
    t = np.asarray(triangles)
    e = np.sort(np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]]), axis=1)
    return np.unique(e, axis=0).astype(np.int32)
