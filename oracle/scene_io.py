"""CPU oracle of the reference's OBJ reader -- TEST INFRASTRUCTURE ONLY.

A plain-Python restatement of _parse_obj (reference scene.py:255-280):
positions only, str.split() tokens, '#' comments, the current g / o / usemtl
name per triangle, 1-based / negative indices, fan triangulation, Python
float() / int() number syntax.  tests/test_mesh_ingest.py checks the native
reader (ef_obj_parse) against it bit-for-bit."""
from __future__ import annotations

import numpy as np


def parse_obj(path):
    verts, tris, groups = [], [], []
    current = ""
    with open(path, "r", encoding="utf-8") as f:
        for line in f:
            parts = line.split()
            if not parts or parts[0].startswith("#"):
                continue
            tag = parts[0]
            if tag == "v":
                verts.append([float(x) for x in parts[1:4]])
            elif tag in ("g", "o", "usemtl"):
                current = parts[1] if len(parts) > 1 else ""
            elif tag == "f":
                idx = []
                for token in parts[1:]:
                    i = int(token.split("/")[0])
                    idx.append(i - 1 if i > 0 else len(verts) + i)
                for k in range(1, len(idx) - 1):
                    tris.append((idx[0], idx[k], idx[k + 1]))
                    groups.append(current)
    return np.asarray(verts, dtype=np.float64), tris, groups
