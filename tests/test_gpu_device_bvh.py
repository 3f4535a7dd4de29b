"""GPU BVH builder (csrc/bvh_device.cu): trees built on the device answer
every query exactly as the host SAH tree does (hit results are
tree-independent by construction), from 1 triangle up to the
964k-triangle C5 city, through a full bounce loop, and after
ef_scene_rebuild of moved geometry.  Run on a B200 with ``-m gpu``."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import oracle as O  # noqa: E402
from paper_1803_00430_b200 import propagation, scene, workloads  # noqa: E402


def _scene(tris, mat, absorption, scattering, build):
    A, B, C = tris[:, 0], tris[:, 1], tris[:, 2]
    mats = [scene.Material(f"m{i}", absorption[i], scattering[i]) for i in range(len(absorption))]
    return scene.SceneModel(A, B - A, C - A, mat, mats, [scene.Source(id="s", position=np.zeros(3))],
                            scene.Listener(position=np.zeros(3)), bvh_build=build)


def _rays(lo, hi, n, seed):
    rng = np.random.default_rng(seed)
    o = rng.uniform(lo, hi, size=(n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1)[:, None]
    return o, d


def _same_answers(s_host, s_dev, o, d):
    th, ih, hh = s_host._query(o, d, 1e-4, None, 2)
    td, idv, hd = s_dev._query(o, d, 1e-4, None, 2)
    assert np.array_equal(ih, idv) and np.array_equal(hh, hd)
    assert np.array_equal(th, td)
    return hh


@pytest.mark.parametrize("name", ["c2", "c3", "c5"])
def test_device_tree_answers_like_host_tree(name):
    w = workloads.WORKLOADS[name]()
    s_host = _scene(w.tris, w.material_index, w.absorption, w.scattering, "host")
    s_dev = _scene(w.tris, w.material_index, w.absorption, w.scattering, "device")
    info = s_dev.device_info()
    assert info["n_nodes"] > 0 and 1 <= info["max_leaf"] <= 4 and info["max_depth"] <= 31
    lo, hi = w.tris.reshape(-1, 3).min(0), w.tris.reshape(-1, 3).max(0)
    o, d = _rays(lo, hi, 20000, 3)
    hit = _same_answers(s_host, s_dev, o, d)
    assert hit.mean() > 0.3
    # the brute-force answer on a slice (all triangles, no tree at all)
    k = 64 if name == "c5" else 512
    tb, ib, _ = s_dev._query(o[:k], d[:k], 1e-4, None, 1)
    td, idv, _ = s_dev._query(o[:k], d[:k], 1e-4, None, 2)
    assert np.array_equal(ib, idv) and np.array_equal(tb, td)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 9, 33, 700])
def test_device_tree_small_and_degenerate_counts(n):
    """Tiny trees (a single leaf root, 1..4 triangles) and clustered
    centroids (duplicate Morton codes: many triangles sharing a centre)."""
    rng = np.random.default_rng(n)
    c = rng.uniform(-3, 3, size=(n, 1, 3))
    if n >= 9:
        c[: n // 2] = c[0]          # duplicate centroids -> equal codes
    tris = c + rng.normal(scale=0.8, size=(n, 3, 3))
    mat = np.zeros(n, np.int64)
    s_dev = _scene(tris, mat, [[0.1] * 4], [[0.2] * 4], "device")
    o, d = _rays(-4, 4, 4000, n)
    tb, ib, hb = s_dev._query(o, d, 1e-4, None, 1)
    td, idv, hd = s_dev._query(o, d, 1e-4, None, 2)
    assert np.array_equal(ib, idv) and np.array_equal(hb, hd) and np.array_equal(tb, td)
    assert hb.any()


def test_bounce_loop_on_device_tree_matches_host_tree():
    """C2 frame slice (diffuse rain on, so the histograms carry energy)
    through ef_trace: identical paths on both trees; the histograms agree to
    float-atomic ordering."""
    w = workloads.c2_city()
    out = {}
    for build in ("host", "device"):
        sc = _scene(w.tris, w.material_index, w.absorption, w.scattering, build)
        cfg = propagation.TraceConfig(primary_rays=w.n_rays, max_order=w.max_bounces, sh_order=w.order,
                                      bin_s=w.bin_s, n_bins=w.n_bins, listener_radius=w.radius,
                                      seed=w.seed, diffuse_rain=True)
        tr = propagation.FrameTracer(sc, len(w.sources), cfg, record=True)
        tr.set_sources(w.sources)
        tr.trace(w.listener, n_rays=4096)
        torch.cuda.synchronize()
        out[build] = (tr.path_ids.cpu().numpy(), tr.path_nseg.cpu().numpy(), tr.H.cpu().numpy(),
                      tr.trace_stats())
    assert np.array_equal(out["host"][0], out["device"][0])
    assert np.array_equal(out["host"][1], out["device"][1])
    Hh, Hd = out["host"][2], out["device"][2]
    assert sum(st.arrivals for st in out["host"][3]) > 0 and np.abs(Hh).sum() > 0 and np.abs(Hd).sum() > 0
    assert np.allclose(Hh, Hd, rtol=1e-5, atol=1e-6 * np.abs(Hh).max())
    assert out["host"][3][0].total_segments == out["device"][3][0].total_segments


def test_rebuild_after_large_motion():
    """Move a third of the C2 city by tens of metres (a refit would keep the
    old, now loose topology), rebuild on the device and compare with a fresh
    host-built scene and the oracle; a refit of the rebuilt tree then tracks
    a second motion."""
    w = workloads.c2_city()
    s = _scene(w.tris, w.material_index, w.absorption, w.scattering, "host")
    lo, hi = w.tris.reshape(-1, 3).min(0), w.tris.reshape(-1, 3).max(0)
    o, d = _rays(lo, hi, 8000, 11)
    s.intersect_batch(o[:8], d[:8])                              # create the device scene
    moved = w.tris.copy()
    moved[2::3] += np.array([35.0, -20.0, 0.0])
    A, B, C = moved[:, 0], moved[:, 1], moved[:, 2]
    s.update_geometry(A, B - A, C - A, rebuild=True)
    fresh = _scene(moved, w.material_index, w.absorption, w.scattering, "host")
    _same_answers(fresh, s, o, d)
    os_ = O.OracleScene(A, B - A, C - A, fresh.normals, w.material_index, w.absorption, w.scattering)
    # oracle all-pairs (ray_triangles_batch + argmin, bvh.py:31-45): lowest id
    # on exact ties, like the device trees
    to, io, _ = os_.intersect_batch(o[:2000], d[:2000], mode=1)
    tg, ig, _ = s._query(o[:2000], d[:2000], 1e-4, None, 2)
    assert np.array_equal(io, ig)
    assert np.array_equal(to[ig >= 0], tg[ig >= 0])
    # second motion by refit of the device-built tree
    moved2 = moved.copy()
    moved2[5::7] += np.array([0.0, 3.0, 1.0])
    A2, B2, C2 = moved2[:, 0], moved2[:, 1], moved2[:, 2]
    s.update_geometry(A2, B2 - A2, C2 - A2)
    fresh2 = _scene(moved2, w.material_index, w.absorption, w.scattering, "host")
    _same_answers(fresh2, s, o, d)
