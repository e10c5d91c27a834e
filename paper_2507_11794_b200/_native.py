"""ctypes binding of the C ABI in include/clothsim_b200.h.

The shared library is built in-tree (``python -m paper_2507_11794_b200.build``
or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing or no CUDA device is visible, ``load()`` raises AdapterUnavailable.
"""

from __future__ import annotations

import ctypes
import os

from .errors import AdapterUnavailable, CapacityError, CollisionBudgetError

HERE = os.path.dirname(os.path.abspath(__file__))
# CLOTHSIM_LIB selects an alternative in-tree build (kernel A/B experiments)
LIB_PATH = os.environ.get("CLOTHSIM_LIB") or os.path.join(HERE, "_lib", "libclothsim_b200.so")

ABI_VERSION = 1
CS_OK, CS_E_INVALID, CS_E_CAPACITY, CS_E_BUDGET, CS_E_NODEVICE, CS_E_CUDA = 0, -1, -2, -3, -4, -5

FLAG_EXPLICIT_EULER = 1
FLAG_AVERAGE_RESPONSE = 2
FLAG_FIXED_POINT = 4
FLAG_FP64 = 8
FLAG_NO_GRAPH = 16
FLAG_FORCE_CSR = 32
FLAG_TILE_KERNEL = 64
FLAG_PAIRED = 128
FLAG_THREAD_NARROW = 256
FLAG_SPLIT_NORMALS = 512
FLAG_FUSE_NORMALS = 1024
FLAG_WARP_NARROW = 2048
FLAG_MEMOP_SEAM = 4096
FLAG_SPLIT_NARROW = 8192

BUF_POSITIONS, BUF_VELOCITIES, BUF_NORMALS, BUF_PREV_POSITIONS = 0, 1, 2, 3
BUF_FORCES_RAW, BUF_ACCUMULATOR, BUF_COUNTS, BUF_EXT_ACCEL = 4, 5, 6, 7
BUF_POSITIONS64, BUF_VELOCITIES64 = 8, 9
BUF_NORMALS_LAGGED = 10

PASS_FORCE_INTEGRATE, PASS_DETECT, PASS_RESPOND, PASS_NORMALS = 0, 1, 2, 3

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32


class CsDesc(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("nx", ctypes.c_int32),
        ("ny", ctypes.c_int32),
        ("grid_rest", ctypes.c_float * 6),
        ("num_nodes", _I64),
        ("num_springs", _I64),
        ("springs", _P),
        ("spring_kinds", _P),
        ("spring_rest", _P),
        ("num_tris", _I64),
        ("tris", _P),
        ("num_edges", _I64),
        ("edges", _P),
        ("positions", _P),
        ("positions64", _P),
        ("inv_mass", _P),
        ("masses64", _P),
        ("pinned", _P),
        ("spring_rest64", _P),
        ("num_obstacle_tris", _I64),
        ("obstacle_corners", _P),
        ("obstacle_normals", _P),
        ("dt", ctypes.c_double),
        ("gravity", ctypes.c_double * 3),
        ("stiffness", ctypes.c_double * 3),
        ("damping", ctypes.c_double),
        ("epsilon_mt", ctypes.c_float),
        ("response_margin", ctypes.c_float),
        ("fixed_point_scale", ctypes.c_int32),
        ("substeps", ctypes.c_int32),
        ("cell_size", ctypes.c_float),
        ("stream", _P),
        ("obstacle_corners64", _P),
        ("obstacle_normals64", _P),
        ("epsilon_mt64", ctypes.c_double),
        ("response_margin64", ctypes.c_double),
    ]


class CsGridDesc(ctypes.Structure):
    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("nx", ctypes.c_int32),
        ("ny", ctypes.c_int32),
        ("row_lo", ctypes.c_int32),
        ("row_hi", ctypes.c_int32),
        ("width", ctypes.c_double),
        ("height", ctypes.c_double),
        ("total_mass", ctypes.c_double),
        ("orientation", ctypes.c_int32),
        ("num_pinned_rows", ctypes.c_int32),
        ("pinned_rows", _P),
        ("dt", ctypes.c_double),
        ("gravity", ctypes.c_double * 3),
        ("stiffness", ctypes.c_double * 3),
        ("damping", ctypes.c_double),
        ("epsilon_mt", ctypes.c_float),
        ("response_margin", ctypes.c_float),
        ("fixed_point_scale", ctypes.c_int32),
        ("substeps", ctypes.c_int32),
        ("stream", _P),
    ]


class CsStats(ctypes.Structure):
    _fields_ = [("hits", _I64), ("responded", _I64), ("frames", _I64), ("hit_counter", _I64)]


class CsHaloPeer(ctypes.Structure):
    _fields_ = [
        ("state", _P * 2),
        ("plane", _I64),
        ("src_row0", _I64),
        ("dst_row0", _I64),
        ("rows", _I64),
        ("remote_flag", _P),
    ]


# every symbol include/clothsim_b200.h declares, with its signature
SIGNATURES = {
    "cs_create": (_I32, [ctypes.POINTER(CsDesc), ctypes.POINTER(_P)]),
    "cs_create_grid": (_I32, [ctypes.POINTER(CsGridDesc), ctypes.POINTER(_P)]),
    "cs_grid_topology": (_I32, [_I32, _I32, _I32, _I32, ctypes.c_double, ctypes.c_double, _P, _P,
                                _P, _P, _P, _P]),
    "cs_destroy": (_I32, [_P]),
    "cs_step": (_I32, [_P, _I32]),
    "cs_run_pass": (_I32, [_P, _I32]),
    "cs_record": (_I32, [_P, _I32, _P]),
    "cs_contact_log": (_I32, [_P, _I64]),
    "cs_read_contacts": (_I32, [_P, _P, _I64, ctypes.POINTER(_I64)]),
    "cs_respond": (_I32, [_P, ctypes.POINTER(_I64)]),
    "cs_frame_stats": (_I32, [_P, ctypes.POINTER(CsStats)]),
    "cs_frame_hits": (_I32, [_P, _I64, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "cs_read": (_I32, [_P, _I32, _P]),
    "cs_write": (_I32, [_P, _I32, _P]),
    "cs_inject_response": (_I32, [_P, _I64, ctypes.POINTER(_I32), _I32]),
    "cs_synchronize": (_I32, [_P]),
    "cs_stream": (_I32, [_P, ctypes.POINTER(_P)]),
    "cs_state_plane": (_I32, [_P, _I32, ctypes.POINTER(_P), ctypes.POINTER(_I64)]),
    "cs_state_buffers": (_I32, [_P, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_P),
                                ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "cs_set_halo_peers": (_I32, [_P, _I64, _I64, ctypes.POINTER(CsHaloPeer),
                                 ctypes.POINTER(CsHaloPeer)]),
    "cs_ipc_export": (_I32, [_P, ctypes.c_char_p]),
    "cs_ipc_open": (_I32, [ctypes.c_char_p, ctypes.POINTER(_P)]),
    "cs_ipc_close": (_I32, [_P]),
    "cs_kernels_per_frame": (_I32, [_P, ctypes.POINTER(_I32)]),
    "cs_broadphase_stats": (_I32, [_P, ctypes.POINTER(_I64)]),
    "cs_broadphase_dump": (_I32, [_P, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(_I32), _P,
                                  _P, _P, _P]),
    "cs_positions_device": (_I32, [_P, _P]),
    "cs_read_device": (_I32, [_P, _I32, _P, _P]),
    "cs_write_device": (_I32, [_P, _I32, _P, _P]),
    "cs_set_stream": (_I32, [_P, _P]),
    "cs_device": (_I32, [_P, ctypes.POINTER(_I32)]),
    "cs_snapshot_bounds": (_I32, [_P, _I64, ctypes.POINTER(ctypes.c_double), _P]),
    "cs_snapshot_render": (_I32, [_P, _P, _I64, _I64, ctypes.POINTER(ctypes.c_double),
                                  ctypes.POINTER(_I32), _I32, _I32, _P, _P, _P]),
    "cs_last_error": (ctypes.c_char_p, []),
    "cs_abi_version": (_I32, []),
    "cs_device_count": (_I32, []),
    "cs_mem_info": (_I32, [ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
}

_lib = None


def load(build_if_missing: bool = True):
    """Load the in-tree CUDA library (building it first if allowed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) and build_if_missing:
        from .build import build

        build()
    if not os.path.exists(LIB_PATH):
        raise AdapterUnavailable(f"CUDA extension not built: {LIB_PATH} is missing")
    try:
        lib = ctypes.CDLL(LIB_PATH)
    except OSError as exc:  # e.g. no libcudart / driver on this host
        raise AdapterUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.cs_abi_version() != ABI_VERSION:
        raise AdapterUnavailable("libclothsim_b200.so ABI version mismatch; rebuild it")
    _lib = lib
    return lib


def check(code: int) -> None:
    if code == CS_OK:
        return
    msg = (_lib.cs_last_error() or b"").decode(errors="replace")
    if code == CS_E_CAPACITY:
        raise CapacityError(msg)
    if code == CS_E_BUDGET:
        raise CollisionBudgetError(msg)
    if code == CS_E_NODEVICE:
        raise AdapterUnavailable(msg)
    if code == CS_E_INVALID:
        raise ValueError(msg)
    raise RuntimeError(f"CUDA error: {msg}")
