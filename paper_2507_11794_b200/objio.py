"""Minimal Wavefront OBJ reader/writer for obstacle meshes (io.py:127-177).

Only ``v`` and ``f`` records matter for the hot path; polygons are fanned into
triangles, ``a/b/c`` references keep the vertex index, negative indices count
from the end.  ``write_obj`` emits ``%.17g`` so a round trip is exact.
"""

from __future__ import annotations

import numpy as np


def load_obj(path):
    verts, tris = [], []
    with open(path, "r", encoding="utf-8") as fh:
        for line in fh:
            parts = line.split()
            if not parts:
                continue
            if parts[0] == "v":
                verts.append([float(x) for x in parts[1:4]])
            elif parts[0] == "f":
                idx = []
                for tok in parts[1:]:
                    k = int(tok.split("/")[0])
                    idx.append(k - 1 if k > 0 else len(verts) + k)
                for q in range(1, len(idx) - 1):
                    tris.append((idx[0], idx[q], idx[q + 1]))
    if not verts or not tris:
        raise ValueError(f"{path}: no vertices or faces")
    return np.asarray(verts, dtype=np.float64), np.asarray(tris, dtype=np.int32)


def write_obj(path, vertices, triangles):
    with open(path, "w", encoding="utf-8") as fh:
        for v in np.asarray(vertices, dtype=np.float64):
            fh.write("v %.17g %.17g %.17g\n" % tuple(v))
        for t in np.asarray(triangles, dtype=np.int64):
            fh.write("f %d %d %d\n" % (t[0] + 1, t[1] + 1, t[2] + 1))
