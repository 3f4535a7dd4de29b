"""Host side of the drop-in boundary on CPU (no device calls): scene
ingestion, materials, sources, trajectories -- the reference's scene.py
behaviour (scene.py:32-171, 282-380) -- checked against the reference
package itself when it is importable (this container), and against its
documented rules otherwise."""
import json
import os
import sys

import numpy as np
import pytest

from paper_1803_00430_b200 import scene

REF_SRC = "/root/reference/pkg/src"

# a unit cube as six quads (fan-triangulated into 12 triangles), one group
CUBE = "\n".join([
    "v 0 0 0", "v 1 0 0", "v 1 1 0", "v 0 1 0",
    "v 0 0 1", "v 1 0 1", "v 1 1 1", "v 0 1 1",
    "g shell",
    "f 1 4 3 2", "f 5 6 7 8", "f 1 2 6 5",
    "f 2 3 7 6", "f 3 4 8 7", "f 4 1 5 8",
]) + "\n"


def _write(tmp_path, mesh=CUBE, **extra):
    desc = {
        "materials": [{"name": "brick", "absorption": [0.05, 0.1, 0.2, 0.3],
                       "scattering": [0.4, 0.4, 0.5, 0.6]}],
        "material_bindings": {"shell": "brick"},
        "sources": [{"id": "a", "position": [0.4, 0.5, 0.5], "radius": 0.0, "gain": 1.0}],
        "listener": {"position": [0.6, 0.5, 0.5], "orientation_quat": [1, 0, 0, 0]},
        "speed_of_sound": 340.0,
    }
    if mesh is not None:
        (tmp_path / "room.obj").write_text(mesh)
        desc["mesh"] = "room.obj"
    desc.update(extra)
    p = tmp_path / "scene.json"
    p.write_text(json.dumps(desc))
    return p


def test_load_cube(tmp_path):
    m = scene.load_scene(_write(tmp_path))
    assert m.n_triangles == 12 and m.degenerate_dropped == 0
    assert m.speed_of_sound == 340.0 and len(m.sources) == 1
    assert {m.materials[i].name for i in m.material_index} == {"brick"}
    assert np.allclose(np.linalg.norm(m.normals, axis=1), 1.0)


def test_unbound_group_gets_default_material(tmp_path):
    m = scene.load_scene(_write(tmp_path, material_bindings={}))
    mat = m.materials[m.material_index[0]]
    assert mat.name == "default"
    assert np.allclose(mat.absorption, scene.DEFAULT_ABSORPTION)
    assert np.allclose(mat.scattering, scene.DEFAULT_SCATTERING)


def test_degenerate_triangles_dropped(tmp_path):
    m = scene.load_scene(_write(tmp_path, mesh=CUBE + "f 1 1 2\nf 3 3 3\n"))
    assert m.n_triangles == 12 and m.degenerate_dropped == 2


def test_free_field_and_validation(tmp_path):
    m = scene.load_scene(_write(tmp_path, mesh=None))
    assert m.n_triangles == 0
    assert m.intersect([0.0, 0, 0], [1.0, 0, 0]) is None      # host answer, no device call
    assert m.intersect_brute([0.0, 0, 0], [1.0, 0, 0]) == (np.inf, -1)
    with pytest.raises(ValueError):
        scene.load_scene(_write(tmp_path, sources=[]))
    with pytest.raises(ValueError):
        scene.Material("bad", [1.2, 0, 0, 0], [0.5] * 4)
    with pytest.raises(ValueError):
        scene.Material("bad", [0.5] * 4, [0.5] * 3)


def test_trajectory_and_rotation(tmp_path):
    csv = tmp_path / "path.csv"
    csv.write_text("0.0,0,0,0,1,0,0,0\n4.0,8,0,0,0,0,0,1\n")
    tr = scene.Trajectory.from_csv(csv)
    pos, quat = tr.pose(2.0)
    assert np.allclose(pos, [4.0, 0.0, 0.0])
    assert abs(np.linalg.norm(quat) - 1.0) < 1e-12
    R = scene.quat_to_matrix(quat)
    assert np.allclose(R @ R.T, np.eye(3), atol=1e-12)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")
def test_ingestion_matches_reference(tmp_path):
    """The same scene through the reference's load_scene and ours: identical
    triangle arrays, normals, material assignment and degenerate count."""
    sys.path.insert(0, REF_SRC)
    try:
        from echoforge import scene as ref
    finally:
        sys.path.remove(REF_SRC)
    path = _write(tmp_path, mesh=CUBE + "f 1 1 2\n")
    a, b = ref.load_scene(path), scene.load_scene(path)
    for f in ("v0", "e1", "e2", "normals"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.degenerate_dropped == b.degenerate_dropped
    assert [a.materials[i].name for i in a.material_index] == \
        [b.materials[i].name for i in b.material_index]
    box_a, box_b = ref.make_box_scene(size=6.0), scene.make_box_scene(size=6.0)
    for f in ("v0", "e1", "e2", "normals"):
        assert np.array_equal(getattr(box_a, f), getattr(box_b, f)), f
