"""Host BVH builder on CPU (no GPU): the 4-wide tree with spatial splits
(triangles shared between leaves through clipped reference boxes) references
every triangle and its conservative f32 boxes never lose a closest hit --
tree answers == brute force over all triangles for random rays, on the C2
city, a C3-like interior and a random soup, with splits on and off."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1803_00430_b200", "csrc")


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("bvh") / "bvh_check")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-I", CSRC,
                           os.path.join(ROOT, "tools", "bvh_check.cpp"),
                           os.path.join(CSRC, "bvh_build.cpp"), "-o", out])
    return out


def _write(path, tris):
    A, B, C = tris[:, 0], tris[:, 1], tris[:, 2]
    with open(path, "wb") as f:
        np.array([len(tris)], np.int64).tofile(f)
        for a in (A, B - A, C - A):
            np.ascontiguousarray(a, np.float64).tofile(f)


def _soup(n, seed):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-10, 10, size=(n, 1, 3))
    return c + rng.normal(scale=1.5, size=(n, 3, 3))


@pytest.mark.parametrize("splits", ["0", "0.5"])
@pytest.mark.parametrize("name", ["c2", "c3", "soup"])
def test_tree_answers_equal_brute_force(checker, tmp_path, name, splits):
    from paper_1803_00430_b200 import workloads
    if name == "c2":
        tris, rays = workloads.c2_city().tris, 3000
    elif name == "c3":
        tris, rays = workloads.c3_interior().tris[:20000], 300
    else:
        tris, rays = _soup(3000, 4), 3000
    path = str(tmp_path / "tris.bin")
    _write(path, tris)
    r = subprocess.run([checker, path, str(rays), "7"], capture_output=True, text=True,
                       env={**os.environ, "EF_BVH_SPLITS": splits}, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    fields = dict(zip(r.stdout.split()[::2], r.stdout.split()[1::2]))
    assert int(fields["hits"]) > rays // 10
    if splits == "0":
        assert int(fields["refs"]) == len(tris)
