import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def mesh_from_golden(g):
    """ClothMesh-like object from a traj_*.npz fixture."""
    nx, ny = int(g["nx"]), int(g["ny"])
    return SimpleNamespace(
        nx=nx, ny=ny, num_nodes=nx * ny, positions=g["positions0"].copy(),
        masses=g["masses"], pinned=g["pinned"], spring_indices=g["springs"],
        spring_rest_lengths=g["rest"], spring_kinds=g["kinds"], triangles=g["tris"],
        num_springs=len(g["springs"]))


def params_from_golden(g):
    from paper_2507_11794_b200.mesh import SimParams

    return SimParams(dt=float(g["dt"]), gravity=tuple(g["gravity"]),
                     stiffness=tuple(g["stiffness"]), damping=float(g["damping"]),
                     epsilon_mt=float(g["epsilon_mt"]), response_margin=float(g["response_margin"]),
                     fixed_point_scale=int(g["fixed_point_scale"]), substeps=int(g["substeps"]),
                     explicit_euler=bool(g["explicit_euler"]),
                     average_response=bool(g["average_response"]))


def obstacle_from_golden(g):
    if "obs_vertices" not in g:
        return None
    from paper_2507_11794_b200.mesh import TriangleMesh

    return TriangleMesh(vertices=g["obs_vertices"], triangles=g["obs_triangles"],
                        face_normals=g["obs_normals"])


TRAJ = ["traj_hang8.npz", "traj_corner16.npz", "traj_hang12x10.npz", "traj_drop10.npz",
        "traj_pull8.npz", "traj_flags.npz"]


@pytest.fixture
def rng():
    return np.random.default_rng(20240817)


def cuda_available():
    try:
        from paper_2507_11794_b200 import _native

        return _native.load(build_if_missing=False).cs_device_count() > 0
    except Exception:
        return False
