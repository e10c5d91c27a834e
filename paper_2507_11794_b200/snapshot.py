"""PNG snapshots of a frame, rendered on the device.

Drop-in for the reference's ``clothsim.io.snapshot_png`` (io.py:225-287;
called by bench.run_backend, bench.py:186-198): same signature, same
orthographic camera, z-buffer rule and shading, and bit-identical pixels --
but the rasterisation runs in ``cs_snapshot.cu`` (one thread per triangle, a
two-pass u64 z-buffer that keeps the reference's earlier-triangle tie rule),
so a large cloth is pictured without its positions crossing PCIe
(``Engine.snapshot_png``).  Only the camera set-up below (io.py:249-258, a
handful of float64 scalars) runs on the host, in numpy, exactly as the
reference writes it; the PNG container is encoded by Pillow as there.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

from . import _native as N

# io.py:180 -- (u, v, depth) coordinate indices per viewing axis
VIEW_AXES = {"x": (1, 2, 0), "y": (0, 2, 1), "z": (0, 1, 2)}


def _check_args(size, axis):
    if axis not in VIEW_AXES:
        raise ValueError(f"axis must be one of {sorted(VIEW_AXES)}, got {axis!r}")
    width, height = int(size[0]), int(size[1])
    if width < 8 or height < 8:
        raise ValueError(f"snapshot size too small: {size!r}")
    return width, height


def camera(lo, hi, width, height, axis):
    """(lo_u, lo_v, scale) from the scene bounds, io.py:249-258 verbatim in
    float64 numpy (the same rounding as the reference)."""
    ax_u, ax_v, _ = VIEW_AXES[axis]
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    span = np.maximum(hi - lo, 1e-9)
    pad = 0.05 * span
    lo = lo - pad
    hi = hi + pad
    span = hi - lo
    scale = min((width - 1) / span[ax_u], (height - 1) / span[ax_v])
    return float(lo[ax_u]), float(lo[ax_v]), float(scale)


def _render(verts, tris, n_cloth_tris, width, height, axis, stream):
    """verts: cuda f64 (n, 3); tris: cuda int32 (t, 3) -> host uint8 (H, W, 3)."""
    import torch

    lib = N.load()
    bounds = (ctypes.c_double * 6)()
    N.check(lib.cs_snapshot_bounds(ctypes.c_void_p(verts.data_ptr()), int(verts.shape[0]), bounds,
                                   ctypes.c_void_p(stream)))
    lo_u, lo_v, scale = camera(bounds[0:3], bounds[3:6], width, height, axis)
    view = (ctypes.c_double * 3)(lo_u, lo_v, scale)
    axes = (ctypes.c_int32 * 3)(*VIEW_AXES[axis])
    rgb = torch.empty((height, width, 3), dtype=torch.uint8, device=verts.device)
    scratch = torch.empty(2 * width * height + 2, dtype=torch.int64, device=verts.device)
    N.check(lib.cs_snapshot_render(ctypes.c_void_p(verts.data_ptr()),
                                   ctypes.c_void_p(tris.data_ptr() if tris.numel() else 0),
                                   int(tris.shape[0]), int(n_cloth_tris), view, axes, width, height,
                                   ctypes.c_void_p(rgb.data_ptr()),
                                   ctypes.c_void_p(scratch.data_ptr()), ctypes.c_void_p(stream)))
    return rgb.cpu().numpy()


def _device_inputs(positions, triangles, obstacle_vertices, obstacle_triangles, device):
    """Concatenate cloth + obstacle into one device vertex / triangle set
    (obstacle indices offset by the cloth's vertex count)."""
    import torch

    def dev(a, dtype):
        if isinstance(a, torch.Tensor):
            return a.to(device=device, dtype=dtype)
        return torch.as_tensor(np.ascontiguousarray(np.asarray(a)), device=device).to(dtype)

    verts = [dev(positions, torch.float64).reshape(-1, 3)]
    tris = [dev(triangles, torch.int32).reshape(-1, 3)]
    n_cloth = tris[0].shape[0]
    if obstacle_vertices is not None:
        verts.append(dev(obstacle_vertices, torch.float64).reshape(-1, 3))
        if obstacle_triangles is not None:
            tris.append(dev(obstacle_triangles, torch.int32).reshape(-1, 3) + verts[0].shape[0])
    return torch.cat(verts).contiguous(), torch.cat(tris).contiguous(), n_cloth


def render_snapshot(positions, triangles, *, obstacle_vertices=None, obstacle_triangles=None,
                    size=(320, 240), axis: str = "y", device=None) -> np.ndarray:
    """The snapshot's pixels, uint8 (height, width, 3) -- what snapshot_png
    encodes.  Inputs may be host arrays or CUDA tensors."""
    width, height = _check_args(size, axis)
    import torch

    if not torch.cuda.is_available():
        raise N.AdapterUnavailable("snapshot rendering needs a CUDA device")
    device = torch.device(device or "cuda")
    verts, tris, n_cloth = _device_inputs(positions, triangles, obstacle_vertices,
                                          obstacle_triangles, device)
    with torch.cuda.device(device):
        stream = torch.cuda.current_stream().cuda_stream
        return _render(verts, tris, n_cloth, width, height, axis, stream)


def _save_png(path, pixels) -> None:
    from PIL import Image

    Image.fromarray(pixels, mode="RGB").save(Path(path), format="PNG")


def snapshot_png(path, positions, triangles, *, obstacle_vertices=None, obstacle_triangles=None,
                 size=(320, 240), axis: str = "y") -> None:
    """Render an orthographic depth-shaded snapshot to PNG (io.py:225-287):
    the camera looks along -axis, cloth off-white, obstacle blue, nearer is
    brighter; byte-deterministic for identical inputs."""
    _check_args(size, axis)
    _save_png(path, render_snapshot(positions, triangles, obstacle_vertices=obstacle_vertices,
                                    obstacle_triangles=obstacle_triangles, size=size, axis=axis))


def engine_snapshot(engine, *, size=(320, 240), axis: str = "y", obstacle: bool = True) -> np.ndarray:
    """Pixels of the engine's CURRENT frame, straight from device memory:
    the positions are widened to float64 on the device (cs_positions_device)
    and only the image is read back."""
    width, height = _check_args(size, axis)
    import torch

    cache = engine.__dict__.setdefault("_snapshot_cache", {})
    device = torch.device("cuda", torch.cuda.current_device())
    key = ("inputs", bool(obstacle))
    if key not in cache:
        ob = engine.obstacle if obstacle else None
        nv = engine.num_nodes
        tris = torch.as_tensor(np.ascontiguousarray(engine.mesh.triangles, dtype=np.int32),
                               device=device).reshape(-1, 3)
        parts = [tris]
        ov = None
        if ob is not None:
            ov = torch.as_tensor(np.ascontiguousarray(ob.vertices, dtype=np.float64), device=device)
            parts.append(torch.as_tensor(np.ascontiguousarray(ob.triangles, dtype=np.int32),
                                         device=device).reshape(-1, 3) + nv)
        torch.cuda.current_stream().synchronize()  # uploads land before the engine stream reads
        cache[key] = (torch.cat(parts).contiguous(), tris.shape[0], ov)
    tris, n_cloth, ov = cache[key]
    nv = engine.num_nodes
    verts = torch.empty((nv + (0 if ov is None else ov.shape[0]), 3), dtype=torch.float64,
                        device=device)
    if ov is not None:
        verts[nv:] = ov
        torch.cuda.current_stream().synchronize()
    N.check(engine._lib.cs_positions_device(engine._handle, ctypes.c_void_p(verts.data_ptr())))
    return _render(verts, tris, n_cloth, width, height, axis, engine.stream_handle)
