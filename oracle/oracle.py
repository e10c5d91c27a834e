"""CPU oracle for the cloth step -- TEST INFRASTRUCTURE ONLY.

Restates the reference package `clothsim` (arxiv 2507.11794) on the CPU so the
B200 path can be checked on the GPU box, where /root/reference does not exist.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module.  The product package
``paper_2507_11794_b200`` never imports it.

Arithmetic lives in ``clothsim_oracle.c`` (built to ``liboracle.so`` by the
Makefile next to it); this file holds the step orchestration and a plain-loop
restatement of the grid topology.  Parity of the oracle itself is pinned by
``tests/golden/*.npz``, generated from the reference by
``tests/golden/make_golden.py``.

* ``SolverOracle``  -- solver.step (solver.py:185-216), float64, bit-exact.
* ``EngineOracle``  -- gpu.engine.Engine.step (engine.py:304-344), float32 with
  i32 fixed-point accumulation, bit-exact vs the numpy kernels.
* ``grid_topology`` -- mesh.generate_cloth_grid (mesh.py:223-317).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

BOX_PAD = np.float32(1e-5)  # kernels.py:48


def build() -> str:
    """Compile liboracle.so with the Makefile beside this file."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "clothsim_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        D = ctypes.c_double
        F = ctypes.c_float
        C = ctypes.c_int
        sig = {
            "or_set_threads": (None, [C]),
            "or_max_threads": (C, []),
            "or_sol_forces": (I, [I, I, P, P, P, P, D, P, P, P, P, P, P, P]),
            "or_sol_integrate": (I, [I, P, P, P, P, P, P, D, C]),
            "or_sol_detect": (I, [I, P, I, P, I, P, I, P, P, P, D, D, P, P]),
            "or_sol_respond": (I, [I, P, P, P, P, P, C]),
            "or_sol_contact_log": (None, [P, I]),
            "or_sol_contact_count": (I, []),
            "or_sol_face_normals": (None, [I, P, P, P]),
            "or_sol_vertex_normals": (None, [I, I, P, P, P]),
            "or_encode": (ctypes.c_int32, [F, F]),
            "or_decode": (F, [ctypes.c_int32, D]),
            "or_eng_spring_force": (None, [I, I, P, P, P, P, P, P, F, P]),
            "or_eng_integrate": (None, [I, P, P, P, P, P, P, P, F, D, C]),
            "or_eng_segment_triangle": (C, [P, P, P, P, P, F, P]),
            "or_eng_detect_cloth_edges": (I, [I, P, P, I, P, P, F, F, F, F, C, P, P]),
            "or_eng_detect_obstacle_edges": (I, [I, P, P, I, P, P, F, F, F, F, C, P, P]),
            "or_eng_respond": (I, [I, P, P, P, P, P, D, C]),
            "or_eng_normals": (None, [I, I, P, P, P, P, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    lib().or_set_threads(int(n))


def max_threads() -> int:
    """Host cores available to this process (not OMP_NUM_THREADS, which
    torchrun pins to 1): the reference arm uses every core it may."""
    try:
        cores = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        cores = os.cpu_count() or 1
    return max(cores, int(lib().or_max_threads()))


def _p(a):
    return None if a is None else a.ctypes.data


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------
# Topology: mesh.generate_cloth_grid (mesh.py:223-317), plain loops.
# ---------------------------------------------------------------------------

def grid_topology(nx, ny, width=1.0, height=1.0):
    """(positions f64 (N,3), springs i32 (S,2), kinds i32 (S,), rest f64 (S,),
    triangles i32 (C,3)) exactly as generate_cloth_grid builds them."""
    xs = np.linspace(0.0, width, nx)
    zs = np.linspace(0.0, height, ny)
    pos = np.zeros((nx * ny, 3))
    for j in range(ny):
        for i in range(nx):
            pos[j * nx + i, 0] = xs[i]
            pos[j * nx + i, 2] = zs[j]
    pairs, kinds = [], []
    for j in range(ny):                       # structural (mesh.py:274-279)
        for i in range(nx):
            if i + 1 < nx:
                pairs.append((j * nx + i, j * nx + i + 1)); kinds.append(0)
            if j + 1 < ny:
                pairs.append((j * nx + i, (j + 1) * nx + i)); kinds.append(0)
    for j in range(ny - 1):                   # shear (mesh.py:280-283)
        for i in range(nx - 1):
            pairs.append((j * nx + i, (j + 1) * nx + i + 1)); kinds.append(1)
            pairs.append((j * nx + i + 1, (j + 1) * nx + i)); kinds.append(1)
    for j in range(ny):                       # bend (mesh.py:284-289)
        for i in range(nx):
            if i + 2 < nx:
                pairs.append((j * nx + i, j * nx + i + 2)); kinds.append(2)
            if j + 2 < ny:
                pairs.append((j * nx + i, (j + 2) * nx + i)); kinds.append(2)
    springs = np.array(pairs, dtype=np.int32)
    kinds = np.array(kinds, dtype=np.int32)
    d = pos[springs[:, 1]] - pos[springs[:, 0]]
    rest = np.linalg.norm(d, axis=1)          # mesh.py:293-294
    tris = []
    for j in range(ny - 1):                   # mesh.py:296-305
        for i in range(nx - 1):
            v00, v10 = j * nx + i, j * nx + i + 1
            v01, v11 = (j + 1) * nx + i, (j + 1) * nx + i + 1
            tris.append((v00, v01, v10))
            tris.append((v10, v01, v11))
    return pos, springs, kinds, rest, np.array(tris, dtype=np.int32)


def unique_edges(triangles):
    """mesh.unique_edges (mesh.py:437-442): sorted undirected edge set."""
    s = set()
    for a, b, c in np.asarray(triangles).tolist():
        for u, v in ((a, b), (b, c), (c, a)):
            s.add((min(u, v), max(u, v)))
    return np.array(sorted(s), dtype=np.int32).reshape(-1, 2)


def incidence_csr(n, triangles):
    """engine.py:232-242: per node, incident triangles in ascending order."""
    lists = [[] for _ in range(n)]
    for t, tri in enumerate(np.asarray(triangles).tolist()):
        for v in tri:
            lists[v].append(t)
    off = np.zeros(n + 1, dtype=np.int64)
    for i in range(n):
        off[i + 1] = off[i] + len(lists[i])
    flat = np.array([t for l in lists for t in sorted(l)], dtype=np.int64)
    return off, flat


def face_normals(vertices, triangles):
    """mesh.compute_face_normals (mesh.py:390-401)."""
    v = _c(vertices, np.float64)
    t = _c(triangles, np.int32)
    out = np.empty((len(t), 3))
    lib().or_sol_face_normals(len(t), _p(v), _p(t), _p(out))
    return out


def vertex_normals(n, triangles, positions):
    """mesh.compute_vertex_normals (mesh.py:404-434)."""
    t = _c(triangles, np.int32)
    pos = _c(positions, np.float64)
    out = np.empty((n, 3))
    lib().or_sol_vertex_normals(n, len(t), _p(t), _p(pos), _p(out))
    return out


class OracleDivergence(RuntimeError):
    pass


# ---------------------------------------------------------------------------
# float64 solver: solver.step (solver.py:185-216)
# ---------------------------------------------------------------------------

class SolverOracle:
    """State + step of the reference CPU solver.  `mesh` is any object with
    the ClothMesh fields (num_nodes, positions, masses, pinned,
    spring_indices, spring_rest_lengths, spring_kinds, triangles)."""

    def __init__(self, mesh, params, obstacle=None, external_accel=None):
        self.n = int(mesh.num_nodes) if hasattr(mesh, "num_nodes") else len(mesh.positions)
        self.params = params
        self.springs = _c(mesh.spring_indices, np.int32)
        self.rest = _c(mesh.spring_rest_lengths, np.float64)
        self.kinds = _c(mesh.spring_kinds, np.int32)
        self.mass = _c(mesh.masses, np.float64)
        self.pinned = _c(mesh.pinned, np.uint8)
        self.tris = _c(mesh.triangles, np.int32)
        self.pos = _c(mesh.positions, np.float64).copy()
        self.prev = self.pos.copy()
        self.vel = np.zeros_like(self.pos)
        self.forces = np.zeros_like(self.pos)
        self.normals = vertex_normals(self.n, self.tris, self.pos)
        self.k3 = _c(params.stiffness, np.float64)
        self.g = _c(params.gravity, np.float64)
        self.ext = None if external_accel is None else _c(external_accel, np.float64)
        self.obstacle = obstacle
        if obstacle is not None:
            self.edges = unique_edges(self.tris)
            self.overt = _c(obstacle.vertices, np.float64)
            self.otris = _c(obstacle.triangles, np.int32)
            self.onorm = _c(obstacle.face_normals, np.float64)
        self.step_count = 0
        self.degenerate_springs = 0

    def forces_now(self):
        L = lib()
        self.degenerate_springs += L.or_sol_forces(
            self.n, len(self.springs), _p(self.springs), _p(self.rest), _p(self.kinds),
            _p(self.k3), float(self.params.damping), _p(self.pos), _p(self.vel),
            _p(self.mass), _p(self.pinned), _p(self.g), _p(self.ext), _p(self.forces))
        return self.forces

    def detect(self):
        acc = np.zeros((self.n, 3))
        cnt = np.zeros(self.n, dtype=np.int64)
        hits = lib().or_sol_detect(
            self.n, _p(self.pos), len(self.edges), _p(self.edges), len(self.tris),
            _p(self.tris), len(self.otris), _p(self.overt), _p(self.otris), _p(self.onorm),
            float(self.params.epsilon_mt), float(self.params.response_margin), _p(acc), _p(cnt))
        return acc, cnt, int(hits)

    def detect_contacts(self, capacity=1 << 22):
        """detect_all at the current positions, returning (hits, contacts):
        contacts is an (n, 2) int32 array of (cloth node, obstacle triangle)
        in the solver's order (collision.py:243-315, Contact.nodes)."""
        buf = np.zeros((capacity, 2), dtype=np.int32)
        L = lib()
        L.or_sol_contact_log(_p(buf), capacity)
        try:
            _, _, hits = self.detect()
            n = int(L.or_sol_contact_count())
        finally:
            L.or_sol_contact_log(None, 0)
        if n > capacity:
            raise RuntimeError("contact log truncated")
        return hits, buf[:n].copy()

    def step(self, normals=True) -> int:
        L = lib()
        p = self.params
        sub = int(p.substeps)
        dt = p.dt / sub
        for _ in range(sub):
            self.forces_now()
            self.step_count += 1
            bad = L.or_sol_integrate(self.n, _p(self.pos), _p(self.prev), _p(self.vel),
                                     _p(self.forces), _p(self.mass), _p(self.pinned),
                                     float(dt), int(bool(p.explicit_euler)))
            if bad >= 0:
                raise OracleDivergence(f"node {bad} became non-finite at step {self.step_count}")
        hits = 0
        if self.obstacle is not None:
            acc, cnt, hits = self.detect()
            L.or_sol_respond(self.n, _p(self.pos), _p(self.vel), _p(acc), _p(cnt),
                             _p(self.pinned), int(bool(p.average_response)))
        if normals:
            self.normals = vertex_normals(self.n, self.tris, self.pos)
        return hits


# ---------------------------------------------------------------------------
# float32 engine: gpu/engine.py Engine.step with gpu/kernels.py semantics
# ---------------------------------------------------------------------------

class EngineOracle:
    """Float32 / fixed-point restatement of the reference's Engine."""

    def __init__(self, mesh, params, obstacle=None, prefilter=True):
        f32 = np.float32
        self.n = n = int(mesh.num_nodes) if hasattr(mesh, "num_nodes") else len(mesh.positions)
        self.params = params
        self.scale = int(params.fixed_point_scale)
        self.scale_f = float(np.float32(self.scale))
        self.springs = _c(mesh.spring_indices, np.int32)
        self.rest = _c(np.asarray(mesh.spring_rest_lengths).astype(f32), f32)
        k = np.asarray(params.stiffness, dtype=np.float64)[np.asarray(mesh.spring_kinds)]
        self.stiff = _c(k.astype(f32), f32)
        self.damp = np.full(len(self.springs), params.damping, dtype=f32)
        self.pos = _c(np.asarray(mesh.positions).astype(f32), f32)
        self.prev = self.pos.copy()
        self.vel = np.zeros_like(self.pos)
        self.forces = np.zeros((n, 3), dtype=np.int32)
        inv = np.where(np.asarray(mesh.pinned), 0.0, 1.0 / np.asarray(mesh.masses))
        self.inv_mass = _c(inv.astype(f32), f32)
        self.ext = np.zeros((n, 3), dtype=f32)
        self.g = _c(np.asarray(params.gravity, dtype=f32), f32)
        self.dt = float(np.float32(params.dt / params.substeps))
        self.tris = _c(mesh.triangles, np.int32)
        self.inc_off, self.inc_tri = incidence_csr(n, self.tris)
        self.normals = np.zeros((n, 3), dtype=f32)
        self.acc = np.zeros((n, 3), dtype=np.int32)
        self.count = np.zeros(n, dtype=np.int32)
        self.prefilter = int(bool(prefilter))
        self.has_obstacle = obstacle is not None and len(obstacle.triangles) > 0
        if self.has_obstacle:
            self.edges = unique_edges(self.tris)
            corners = np.asarray(obstacle.vertices)[np.asarray(obstacle.triangles)]
            self.corners = _c(corners.astype(f32), f32)
            self.onorm = _c(np.asarray(obstacle.face_normals).astype(f32), f32)
        self.frame_count = 0
        self.hit_counter = 0

    def set_external_accel(self, accel):
        self.ext[...] = 0.0 if accel is None else np.asarray(accel, dtype=np.float32)

    def spring_forces(self):
        lib().or_eng_spring_force(self.n, len(self.springs), _p(self.springs), _p(self.rest),
                                  _p(self.stiff), _p(self.damp), _p(self.pos), _p(self.vel),
                                  self.scale_f, _p(self.forces))
        return self.forces

    def integrate(self):
        lib().or_eng_integrate(self.n, _p(self.pos), _p(self.prev), _p(self.vel),
                               _p(self.forces), _p(self.inv_mass), _p(self.ext), _p(self.g),
                               self.dt, float(self.scale), int(bool(self.params.explicit_euler)))

    def detect(self):
        L = lib()
        eps = float(np.float32(self.params.epsilon_mt))
        margin = float(np.float32(self.params.response_margin))
        ha = L.or_eng_detect_cloth_edges(len(self.edges), _p(self.edges), _p(self.pos),
                                         len(self.corners), _p(self.corners), _p(self.onorm),
                                         eps, margin, self.scale_f, float(BOX_PAD),
                                         self.prefilter, _p(self.acc), _p(self.count))
        hb = L.or_eng_detect_obstacle_edges(len(self.corners), _p(self.corners), _p(self.onorm),
                                            len(self.tris), _p(self.tris), _p(self.pos), eps,
                                            margin, self.scale_f, float(BOX_PAD), self.prefilter,
                                            _p(self.acc), _p(self.count))
        self.hit_counter += int(ha + hb)
        return int(ha), int(hb)

    def respond(self):
        return int(lib().or_eng_respond(self.n, _p(self.pos), _p(self.vel), _p(self.acc),
                                        _p(self.count), _p(self.inv_mass), float(self.scale),
                                        int(bool(self.params.average_response))))

    def update_normals(self):
        lib().or_eng_normals(self.n, len(self.tris), _p(self.tris), _p(self.pos),
                             _p(self.inc_off), _p(self.inc_tri), _p(self.normals))

    def step(self):
        """Returns (hits, responded)."""
        for _ in range(int(self.params.substeps)):
            self.spring_forces()
            self.integrate()
        hits = responded = 0
        if self.has_obstacle:
            ha, hb = self.detect()
            hits = ha + hb
            responded = self.respond()
        self.update_normals()
        self.frame_count += 1
        return hits, responded


def boundary_distance(start, end, v0, v1, v2, eps=1e-6):
    """Distance of the segment-triangle decision quantities to the nearest
    predicate boundary, in float64 -- used to classify contacts on which a
    float32 and a float64 evaluation may legitimately disagree.  Restates
    the reference test oracle's classifier (pkg/tests/oracles.py:81-116):
    |a| vs eps, u vs 0/1, v vs 0, u+v vs 1, t vs eps and |d|."""
    s, e = np.asarray(start, np.float64), np.asarray(end, np.float64)
    v0, v1, v2 = (np.asarray(x, np.float64) for x in (v0, v1, v2))
    d = e - s
    dl = float(np.linalg.norm(d))
    if dl == 0.0:
        return 0.0
    r = d / dl
    e1, e2 = v1 - v0, v2 - v0
    h = np.cross(r, e2)
    a = float(e1 @ h)
    m = [abs(abs(a) - eps)]
    if abs(a) >= eps:
        f = 1.0 / a
        q = np.cross(s - v0, e1)
        u = f * float((s - v0) @ h)
        v = f * float(r @ q)
        t = f * float(e2 @ q)
        m += [abs(u), abs(1.0 - u), abs(v), abs(u + v - 1.0), abs(t - eps), abs(dl - t)]
    return min(m)


# ---------------------------------------------------------------------------
# Broad-phase grid (no reference counterpart: the reference brute-forces every
# pair, collision.py:243-315 / kernels.py:186-290, and its own test pins a
# prefilter to brute force, test_gpu_engine.py:267-307).  A numpy float32
# restatement of the device build in csrc/cs_collide.cu build_broadphase, so
# the north star's "bit-exact grid-cell assignment" has a checker.
# ---------------------------------------------------------------------------

def grid_geometry(corners, cell_size=None):
    """(origin f32[3], inv_cell f32, cell f32, dims int[3]) of the uniform grid
    over the obstacle's triangle boxes: origin = min corner of the union box;
    cell edge = f32(mean over triangles of the largest box extent), summed in
    float64 in triangle order (or `cell_size`); dims[d] = ceil((hi-lo)/cell)+1,
    the edge grown x1.25 (f32) until the grid has at most 2^24 cells."""
    c = np.asarray(corners, dtype=np.float32).reshape(-1, 3, 3)
    lo = np.minimum(np.minimum(c[:, 0], c[:, 1]), c[:, 2])
    hi = np.maximum(np.maximum(c[:, 0], c[:, 1]), c[:, 2])
    glo, ghi = lo.min(axis=0), hi.max(axis=0)
    ext = (hi - lo).max(axis=1).astype(np.float64)
    mean = float(np.add.accumulate(ext)[-1]) / max(len(c), 1)  # sequential f64 sum
    cell = np.float32(cell_size) if cell_size else np.float32(mean)
    if not cell > 0:
        cell = np.float32(1.0)
    while True:
        dims = [max(1, int(math.ceil(float(ghi[d] - glo[d]) / float(cell))) + 1) for d in range(3)]
        if dims[0] * dims[1] * dims[2] <= (1 << 24):
            break
        cell = np.float32(cell * np.float32(1.25))
    return glo, np.float32(np.float32(1.0) / cell), cell, dims


def grid_cell_of(x, origin, inv_cell, dims):
    """cell_of per axis: floor(f32(f32(x - origin) * inv_cell)), clamped to
    [0, dims-1] (NaN -> 0); x is (..., 3) float32."""
    f = np.floor((np.asarray(x, np.float32) - origin) * inv_cell)
    out = np.zeros(f.shape, dtype=np.int64)
    for d in range(3):
        fd = f[..., d]
        v = np.where(fd >= 0, fd, 0.0)
        v = np.where(v >= dims[d] - 1, dims[d] - 1, v)
        out[..., d] = v.astype(np.int64)
    return out


def broadphase_grid(corners, cell_size=None):
    """The grid-cell assignment: every triangle is referenced by each cell its
    (unpadded) box covers, cells enumerated z-major then y then x, and the
    (cell key, triangle) references sorted stably by key (key = (z*dy + y)*dx
    + x).  Returns dict(origin, inv_cell, cell, dims, ref_keys, ref_tris,
    cell_begin, cell_end) -- empty cells have begin = end = 0."""
    c = np.asarray(corners, dtype=np.float32).reshape(-1, 3, 3)
    origin, inv_cell, cell, dims = grid_geometry(c, cell_size)
    lo = np.minimum(np.minimum(c[:, 0], c[:, 1]), c[:, 2])
    hi = np.maximum(np.maximum(c[:, 0], c[:, 1]), c[:, 2])
    a = grid_cell_of(lo, origin, inv_cell, dims)
    b = grid_cell_of(hi, origin, inv_cell, dims)
    w = b - a + 1
    counts = w[:, 0] * w[:, 1] * w[:, 2]
    tri = np.repeat(np.arange(len(c), dtype=np.int64), counts)
    start = np.concatenate([[0], np.cumsum(counts)[:-1]])
    q = np.arange(int(counts.sum()), dtype=np.int64) - np.repeat(start, counts)
    wx, wy = w[tri, 0], w[tri, 1]
    x = a[tri, 0] + q % wx
    y = a[tri, 1] + (q // wx) % wy
    z = a[tri, 2] + q // (wx * wy)
    keys = (z * dims[1] + y) * dims[0] + x
    order = np.argsort(keys, kind="stable")
    keys, tris = keys[order].astype(np.uint32), tri[order].astype(np.uint32)
    ncell = dims[0] * dims[1] * dims[2]
    beg = np.zeros(ncell, dtype=np.uint32)
    end = np.zeros(ncell, dtype=np.uint32)
    if len(keys):
        first = np.flatnonzero(np.r_[True, keys[1:] != keys[:-1]])
        last = np.r_[first[1:], len(keys)]
        beg[keys[first]] = first
        end[keys[first]] = last
    return {"origin": origin, "inv_cell": inv_cell, "cell": cell, "dims": tuple(dims),
            "ref_keys": keys, "ref_tris": tris, "cell_begin": beg, "cell_end": end}


def encode(x, scale=1 << 16):
    return int(lib().or_encode(float(np.float32(x)), float(np.float32(scale))))


def segment_triangle_f32(start, end, v0, v1, v2, eps=1e-6):
    pt = np.zeros(3, dtype=np.float32)
    args = [_c(a, np.float32) for a in (start, end, v0, v1, v2)]
    ok = lib().or_eng_segment_triangle(*[_p(a) for a in args], float(np.float32(eps)), _p(pt))
    return bool(ok), pt
