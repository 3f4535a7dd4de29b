"""Pin the CPU oracle against golden vectors produced by the reference itself
(oracle/gen_golden.py).  Intersection, BVH build/traversal and SH must be
bit-exact; the bounce loop is compared with the numpy restatement whose every
closest hit came from the reference's SceneModel.intersect_batch."""
import numpy as np
import pytest

from oracle import oracle as O


def _scene(g):
    return O.OracleScene(g["v0"], g["e1"], g["e2"], g["normals"], g["material_index"],
                         g["absorption"], g["scattering"])


BVH_KEYS = ("node_min", "node_max", "node_left", "node_start", "node_count", "tri_order")


@pytest.mark.parametrize("name", ["box", "soup700", "c2_city", "c1_trace"])
def test_bvh_build_identical(golden, name):
    """bvh.py:51-128 restated: identical node arrays and tri_order."""
    g = golden(name)
    arr = _scene(g).bvh_arrays()
    for k in BVH_KEYS:
        assert arr[k].shape == g[k].shape, k
        assert np.array_equal(arr[k], g[k]), k


def test_box_batch_bit_exact(golden):
    """intersect_batch brute path (scene.py:216-223) on the 10 m box."""
    g = golden("box")
    t, tri, hit = _scene(g).intersect_batch(g["origins"], g["dirs"])
    assert np.array_equal(t, g["t"])
    assert np.array_equal(tri, g["tri"])
    assert np.array_equal(hit, g["hit"])


def test_box_scalar_bvh(golden):
    """SceneModel.intersect -> BVH.intersect (scene.py:184, bvh.py:130)."""
    g = golden("box")
    s = _scene(g)
    t, tri, _ = s.intersect_batch(g["origins"], g["dirs"], mode=2, blas_v=True)
    assert np.array_equal(t, g["scalar_t"])
    assert np.array_equal(tri, g["scalar_tri"])
    t, tri, _ = s.intersect_batch(g["special_o"], g["special_d"], mode=2, blas_v=True)
    assert np.array_equal(tri, g["special_tri"])
    assert np.array_equal(t, g["special_t"])
    assert abs(t[0] - 5.0) < 1e-6 and tri[1] == -1     # test_scene.py:107-120


def test_soup_brute_and_bvh(golden):
    """test_random_soup (test_scene.py:145-169) fixtures, bit-exact."""
    g = golden("soup700")
    s = _scene(g)
    t, tri, _ = s.intersect_batch(g["origins"], g["dirs"], mode=1)
    assert np.array_equal(tri, g["brute_tri"])
    assert np.array_equal(t[tri >= 0], g["brute_t"][tri >= 0])
    t, tri, _ = s.intersect_batch(g["origins"], g["dirs"], mode=2, blas_v=True)
    assert np.array_equal(tri, g["bvh_tri"])
    assert np.array_equal(t, g["bvh_t"])
    # numpy-einsum v (the product's formula) differs only at near-edge hits
    t2, tri2, _ = s.intersect_batch(g["origins"], g["dirs"], mode=2, blas_v=False)
    assert (tri2 != tri).sum() <= 2
    # all-pairs kernel (bvh.py:31-45) on the first 2000 rays
    t, tri, _ = s.intersect_batch(g["origins"][:2000], g["dirs"][:2000], mode=1)
    assert np.array_equal(tri, g["allpairs_tri"])
    assert np.array_equal(t, g["allpairs_t"])


def test_city_bvh_queries(golden):
    """C2 city (2,402 tris > 512): intersect_batch takes the BVH path."""
    g = golden("c2_city")
    t, tri, hit = _scene(g).intersect_batch(g["q_o"], g["q_d"], blas_v=True)
    assert np.array_equal(tri, g["q_tri"])
    assert np.array_equal(t, g["q_t"])


def test_eval_sh_bit_exact(golden):
    g = golden("sh")
    for o in range(5):
        assert np.array_equal(O.eval_sh_batch(g["dirs"], o), g[f"Y{o}"])


def _trace_cfg(w_arrays, **kw):
    return kw


def test_c1_trace_matches_reference_hits(golden):
    """C1 bounce loop: C oracle vs numpy loop driven by the reference's
    intersect_batch.  Hit-id sequences and segment counts exact."""
    from paper_1803_00430_b200 import workloads
    g = golden("c1_trace")
    w = workloads.c1_shoebox()
    s = _scene(g)
    res = O.trace(s, src_key=0, src_pos=w.sources[0], listener=w.listener, radius=w.radius,
                  seed=w.seed, order=w.order, n_bins=w.n_bins, bin_len=343.0 * 1e-3,
                  max_bounces=w.max_bounces, e0=g["e0"], rays=g["rays"], record=True)
    assert np.array_equal(res.nseg, g["nseg"])
    assert np.array_equal(res.ids, g["ids"])
    assert res.stats["segments"] == int(g["nseg"].sum())
    np.testing.assert_allclose(res.H, g["H"], rtol=1e-9, atol=1e-12 * g["H"].max())
    np.testing.assert_allclose(res.Dir, g["Dir"], rtol=1e-9, atol=1e-15)
    assert res.stats["escaped"] >= 1      # corner escapes through RAY_EPS


def test_c2_trace_subsample_matches_reference_hits(golden):
    from paper_1803_00430_b200 import workloads
    g = golden("c2_city")
    w = workloads.c2_city()
    s = _scene(g)
    res = O.trace(s, src_key=0, src_pos=w.sources[0], listener=w.listener, radius=w.radius,
                  seed=w.seed, order=w.order, n_bins=w.n_bins, bin_len=343.0 * 1e-3,
                  max_bounces=w.max_bounces, e0=g["trace_e0"], rays=g["rays"], record=True,
                  blas_v=True)
    assert np.array_equal(res.nseg, g["trace_nseg"])
    assert np.array_equal(res.ids, g["trace_ids"])


def test_philox_known_answers():
    """Random123 Philox4x32-10 known-answer vectors."""
    assert list(O.philox([0, 0, 0, 0], [0, 0])) == [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]
    f = 0xffffffff
    assert list(O.philox([f, f, f, f], [f, f])) == [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]
    assert list(O.philox([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344],
                         [0xa4093822, 0x299f31d0])) == [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]


def test_sphere_samples_unit_and_uniform():
    d = np.array([O.sample_sphere(0, 0, r) for r in range(4000)])
    assert np.abs(np.linalg.norm(d, axis=1) - 1.0).max() < 1e-14
    assert np.abs(d.mean(axis=0)).max() < 0.05
