"""B200-native cloth step (arxiv 2507.11794), behind the reference's Engine API.

Hot path: mass-spring forces + integration (fused node-gather stencil),
cloth vs static triangle mesh collision (uniform-grid broad phase + exact
Moller-Trumbore narrow phase + fixed-point response) and vertex normals --
all hand-written sm_100a CUDA in ``csrc/``, reached through the C ABI of
``include/clothsim_b200.h``.
"""

from .engine import (
    ADAPTER_ENV,
    DEFAULT_PAIR_BUDGET,
    PRECISIONS,
    CudaDevice,
    Engine,
    Layout,
    StepResult,
    build_pipeline,
    get_adapter,
    step_gpu,
)
from .errors import AdapterUnavailable, CapacityError, CollisionBudgetError, DivergenceError
from .fixedpoint import FIXED_SATURATION, decode_values, encode_values
from .mesh import (
    ClothMesh,
    SimParams,
    SpringKind,
    TriangleMesh,
    compute_face_normals,
    compute_vertex_normals,
    generate_cloth_grid,
    generate_icosphere,
    generate_uv_sphere,
    spring_count_formula,
    unique_edges,
)
from .scenes import ScenarioConfig, Scene, baseline_scene, build_scene, stable_coefficients
from .snapshot import render_snapshot, snapshot_png

__version__ = "0.1.0"

__all__ = [
    "ADAPTER_ENV", "DEFAULT_PAIR_BUDGET", "PRECISIONS", "CudaDevice", "Engine", "Layout",
    "StepResult", "build_pipeline", "get_adapter", "step_gpu", "AdapterUnavailable",
    "CapacityError", "CollisionBudgetError", "DivergenceError", "FIXED_SATURATION",
    "decode_values", "encode_values", "ClothMesh", "SimParams", "SpringKind", "TriangleMesh",
    "compute_face_normals", "compute_vertex_normals", "generate_cloth_grid",
    "generate_icosphere", "generate_uv_sphere", "spring_count_formula", "unique_edges",
    "ScenarioConfig", "Scene", "baseline_scene", "build_scene", "stable_coefficients",
    "render_snapshot", "snapshot_png",
]
