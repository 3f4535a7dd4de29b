"""Scene ingestion: the native OBJ reader
(ef_obj_parse) equals the reference's _parse_obj restated in
oracle/scene_io.py bit-for-bit, malformed files raise ValueError, and the
parse-free binary .efmesh loads the same scene.  CPU only (host code of the
C-ABI library)."""
import json
import os
import sys
import time

import numpy as np
import pytest

from oracle import scene_io
from paper_1803_00430_b200 import scene, workloads

REF_SRC = "/root/reference/pkg/src"


def _tricky_obj(path, n_boxes=300, seed=4):
    """Boxes as quads (fan-triangulated), polygons, negative indices,
    comments, groups via g / o / usemtl, exponents / underscores / signs."""
    rng = np.random.default_rng(seed)
    lines = ["# generated", "o city", "", "\t# indented comment"]
    nv = 0
    for b in range(n_boxes):
        lo = rng.uniform(-500, 500, 3)
        hi = lo + rng.uniform(0.1, 40, 3)
        if b % 3 == 0:
            lines.append(f"usemtl brick_{b % 7}")
        elif b % 3 == 1:
            lines.append(f"g facade{b % 5} extra tokens")
        corners = [(x, y, z) for x in (lo[0], hi[0]) for y in (lo[1], hi[1]) for z in (lo[2], hi[2])]
        for k, c in enumerate(corners):
            fmt = ["{:.17g}", "{:.6e}", "{!r}"][(b + k) % 3]
            lines.append("v " + " ".join(fmt.format(float(v)) for v in c) + (" 1.0" if k == 0 else ""))
        base = nv + 1
        quads = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
        for qi, q in enumerate(quads):
            if b % 4 == 0:      # negative (relative) indices with texture / normal slots
                toks = [f"{base + i - (nv + 9)}/{i + 1}/{i + 1}" for i in q]
            elif b % 4 == 1:
                toks = [f"{base + i}//{i + 1}" for i in q]
            else:
                toks = [str(base + i) for i in q]
            lines.append("f " + " ".join(toks))
        nv += 8
        if b % 50 == 0:
            lines.append(f"f {nv} {nv - 1} {nv - 2} {nv - 3} {nv - 4}")   # pentagon
            lines.append(f"f {nv} {nv - 1}")                              # < 3 vertices: nothing
    lines.append("v 1_000.5 -2e-3 +3")
    lines.append("f -1 -2 -3")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def _same(native, ref):
    verts, tris, grp, names = native
    rv, rt, rg = ref
    assert np.array_equal(verts, rv)
    assert np.array_equal(tris, np.asarray(rt, np.int64).reshape(-1, 3))
    assert [names[g] for g in grp] == rg


def test_native_obj_reader_matches_reference_restatement(tmp_path):
    p = str(tmp_path / "city.obj")
    _tricky_obj(p)
    _same(scene.read_obj(p), scene_io.parse_obj(p))
    v, t, g = scene._parse_obj(p)            # the reference's return shapes
    rv, rt, rg = scene_io.parse_obj(p)
    assert np.array_equal(v, rv) and t == rt and g == rg


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")
def test_native_obj_reader_matches_reference_itself(tmp_path):
    sys.path.insert(0, REF_SRC)
    try:
        from echoforge import scene as ref
    finally:
        sys.path.remove(REF_SRC)
    p = str(tmp_path / "city.obj")
    _tricky_obj(p, n_boxes=120, seed=9)
    _same(scene.read_obj(p), ref._parse_obj(p))


def test_malformed_obj_raises(tmp_path):
    cases = {"v 1 2\n": "fewer than 3", "v 1 x 3\n": "bad vertex", "v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 a\n": "bad face",
             "v 0 0 0\nf 1 2 3\n": "out of range", "v 1__0 0 0\n": "bad vertex",
             "v 0x1p3 0 0\n": "bad vertex"}
    for text, msg in cases.items():
        p = tmp_path / "bad.obj"
        p.write_text(text)
        with pytest.raises(ValueError, match=msg):
            scene.read_obj(str(p))
        # the reference fails on these too (float()/int() ValueError, the
        # out-of-range index an IndexError when the soup is gathered) except
        # a short vertex, which it keeps as a ragged row until used
        if msg != "fewer than 3":
            with pytest.raises((ValueError, IndexError)):
                v, t, _ = scene_io.parse_obj(str(p))
                np.asarray(v)[np.asarray(t)]
    with pytest.raises(ValueError):
        scene.read_obj(str(tmp_path / "missing.obj"))


def test_efmesh_roundtrip_and_load_scene(tmp_path):
    p = str(tmp_path / "city.obj")
    _tricky_obj(p, n_boxes=200, seed=2)
    verts, tris, grp, names = scene.read_obj(p)
    q = str(tmp_path / "city.efmesh")
    scene.save_mesh(q, verts, tris, grp, names)
    v2, t2, g2, n2 = scene.read_efmesh(q)
    assert np.array_equal(v2, verts) and np.array_equal(t2, tris) and np.array_equal(g2, grp) and n2 == names
    mats = [{"name": "brick", "absorption": [0.1, 0.2, 0.3, 0.4], "scattering": [0.5] * 4},
            {"name": "glass", "absorption": [0.05] * 4, "scattering": [0.1] * 4}]
    desc = {"materials": mats, "material_bindings": {"brick_3": "brick", "facade2": "glass"},
            "sources": [{"position": [0, 0, 1]}], "listener": {"position": [5, 5, 1]}}
    a = scene.load_scene(dict(desc, mesh=p), base_dir=str(tmp_path))
    b = scene.load_scene(dict(desc, mesh=q), base_dir=str(tmp_path))
    for f in ("v0", "e1", "e2", "normals", "material_index"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.degenerate_dropped == b.degenerate_dropped
    assert set(a.material_index.tolist()) == {0, 1, 2}
    bad = tmp_path / "bad.efmesh"
    bad.write_bytes(b"NOTAMESH" + bytes(40))
    with pytest.raises(ValueError):
        scene.read_efmesh(str(bad))


def test_native_reader_is_fast(tmp_path):
    """C3's 99k-triangle interior as an OBJ: the native reader vs the
    per-line Python restatement (informational bound: >= 5x)."""
    w = workloads.c3_interior(n_sources=1, n_rays=1)
    verts = w.tris.reshape(-1, 3)
    p = tmp_path / "c3.obj"
    with open(p, "w") as f:
        f.write("\n".join("v %.17g %.17g %.17g" % tuple(v) for v in verts) + "\n")
        f.write("\n".join(f"f {3 * i + 1} {3 * i + 2} {3 * i + 3}" for i in range(len(w.tris))) + "\n")
    t_native = float("inf")
    for _ in range(3):   # best of three: the first read also pays the page cache
        t0 = time.perf_counter()
        native = scene.read_obj(str(p))
        t_native = min(t_native, time.perf_counter() - t0)
    t1 = time.perf_counter()
    ref = scene_io.parse_obj(str(p))
    t_ref = time.perf_counter() - t1
    _same(native, ref)
    assert t_ref > 5 * t_native, (t_native, t_ref)
