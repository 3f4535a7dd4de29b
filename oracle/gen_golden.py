"""Generate golden fixtures from the REFERENCE itself (run in the build
container only; /root/reference does not exist on the GPU box).

    python oracle/gen_golden.py

Writes tests/golden/*.npz (committed) and the t-design tables used by the
product (paper_1803_00430_b200/data/tdesigns.npz).  Everything here calls the
unmodified reference package (/root/reference/pkg/src/echoforge) for the
quantities it implements (intersection, BVH, SH, loudness); the bounce loop
(SPEC-only, no reference code) is restated in numpy with every closest-hit
query answered by the reference's own ``SceneModel.intersect_batch``
("hit IDs are ground truth, not a restatement").
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = os.environ.get("ECHOFORGE_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from echoforge import bvh as ref_bvh  # noqa: E402
from echoforge import scene as ref_scene  # noqa: E402
from echoforge import sh as ref_sh  # noqa: E402
from echoforge import tdesigns as ref_td  # noqa: E402

from paper_1803_00430_b200 import workloads  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def _model_from_workload(w):
    v0, e1, e2 = w.soup()
    mats = [ref_scene.Material(f"m{i}", np.clip(w.absorption[i], 0, 1)[:4],
                               np.clip(w.scattering[i], 0, 1)[:4])
            for i in range(len(w.absorption))]
    src = [ref_scene.Source(id=str(i), position=p) for i, p in enumerate(w.sources)]
    return ref_scene.SceneModel(v0, e1, e2, w.material_index, mats, src,
                                ref_scene.Listener(position=w.listener))


def _bvh_arrays(model):
    b = model.bvh
    return dict(node_min=b.node_min, node_max=b.node_max, node_left=b.node_left,
                node_start=b.node_start, node_count=b.node_count, tri_order=b.tri_order)


# ---------------------------------------------------------------- numpy RNG
M0, M1, W0, W1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57), np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)


def philox_np(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 (uint32 arrays)."""
    c0, c1, c2, c3 = (np.asarray(x, np.uint32).copy() for x in (c0, c1, c2, c3))
    k0 = np.asarray(k0, np.uint32).copy()
    k1 = np.asarray(k1, np.uint32).copy()
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = M0 * c0.astype(np.uint64)
            p1 = M1 * c2.astype(np.uint64)
            hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
            lo0 = p0.astype(np.uint32)
            hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
            lo1 = p1.astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0 = k0 + W0
            k1 = k1 + W1
    return c0, c1, c2, c3


def u53_np(a, b):
    return ((a >> np.uint32(5)).astype(np.float64) * 67108864.0 +
            (b >> np.uint32(6)).astype(np.float64)) * (1.0 / 9007199254740992.0)


def draw2_np(ray, bounce, draw, frame, seed, src):
    n = len(ray)
    x = philox_np(ray, np.full(n, bounce, np.uint32) if np.isscalar(bounce) else bounce,
                  np.full(n, draw, np.uint32), np.full(n, frame, np.uint32),
                  np.full(n, seed, np.uint32), np.full(n, src, np.uint32))
    return u53_np(x[0], x[1]), u53_np(x[2], x[3])


def sample_sphere_np(seed, src, rays, frame):
    n = len(rays)
    d = np.zeros((n, 3))
    todo = np.ones(n, bool)
    for j in range(64):
        idx = np.nonzero(todo)[0]
        if len(idx) == 0:
            break
        u1, u2 = draw2_np(rays[idx], 0, j, frame, seed, src)
        a = 2.0 * u1 - 1.0
        b = 2.0 * u2 - 1.0
        s = a * a + b * b
        ok = s < 1.0
        f = 2.0 * np.sqrt(1.0 - s[ok])
        d[idx[ok], 0] = a[ok] * f
        d[idx[ok], 1] = b[ok] * f
        d[idx[ok], 2] = 1.0 - 2.0 * s[ok]
        todo[idx[ok]] = False
    d[todo] = [0.0, 0.0, 1.0]
    return d


def sample_cosine_np(seed, src, rays, bounce, frame, n):
    m = len(rays)
    d = n.copy()
    todo = np.ones(m, bool)
    for j in range(64):
        idx = np.nonzero(todo)[0]
        if len(idx) == 0:
            break
        u1, u2 = draw2_np(rays[idx], bounce[idx], 1 + j, frame, seed, src)
        a = 2.0 * u1 - 1.0
        b = 2.0 * u2 - 1.0
        s = a * a + b * b
        ok = s < 1.0
        k = idx[ok]
        a, b, s = a[ok], b[ok], s[ok]
        z = np.sqrt(1.0 - s)
        nx, ny, nz = n[k, 0], n[k, 1], n[k, 2]
        sg = np.copysign(1.0, nz)
        aa = -1.0 / (sg + nz)
        bb = nx * ny * aa
        t1x, t1y, t1z = 1.0 + sg * nx * nx * aa, sg * bb, -sg * nx
        t2x, t2y, t2z = bb, sg + ny * ny * aa, -ny
        d[k, 0] = (a * t1x + b * t2x) + z * nx
        d[k, 1] = (a * t1y + b * t2y) + z * ny
        d[k, 2] = (a * t1z + b * t2z) + z * nz
        todo[k] = False
    return d


def dot_np(a, b):
    return (a[:, 0] * b[:, 0] + a[:, 2] * b[:, 2]) + a[:, 1] * b[:, 1]


def material_tables_np(absorption, scattering):
    m, nb = absorption.shape
    fd = np.zeros((m, nb), np.float32)
    fs = np.zeros((m, nb), np.float32)
    pd = np.zeros(m)
    for i in range(m):
        p = 0.0
        for b in range(nb):
            p += float(scattering[i, b])
        p = p / nb
        pd[i] = p
        for b in range(nb):
            keep = 1.0 - float(absorption[i, b])
            sb = float(scattering[i, b])
            fd[i, b] = np.float32(keep * (sb / p)) if p > 0.0 else 0.0
            fs[i, b] = np.float32(keep * ((1.0 - sb) / (1.0 - p))) if p < 1.0 else 0.0
    return fd, fs, pd


def trace_reference(model, w, src_index, rays, frame=0):
    """Pinned bounce loop with the reference answering every
    closest-hit query through SceneModel.intersect_batch (scene.py:208)."""
    nb = w.n_bands
    order = w.order
    nk = (order + 1) ** 2
    n = len(rays)
    fd, fs, pd = material_tables_np(w.absorption, w.scattering)
    e0 = np.float32(1.0 / (w.n_rays * np.pi * w.radius * w.radius))
    bin_len = w.speed_of_sound * w.bin_s
    L = w.listener
    r2 = w.radius * w.radius
    d = sample_sphere_np(w.seed, src_index, rays, frame)
    o = np.repeat(w.sources[src_index][None, :], n, axis=0)
    E = np.full((n, nb), e0, np.float32)
    plen = np.zeros(n)
    nrefl = np.zeros(n, np.int64)
    nseg = np.zeros(n, np.int32)
    ids = np.full((n, w.max_bounces), -2, np.int32)
    H = np.zeros((w.n_bins, nb, nk))
    Dir = np.zeros((nb, nk))
    active = np.ones(n, bool)
    while active.any():
        a = np.nonzero(active)[0]
        t, tri, hit = model.intersect_batch(o[a], d[a])
        ids[a, nseg[a]] = np.where(hit, tri, -1)
        Lo = L[None, :] - o[a]
        tc = dot_np(Lo, d[a])
        tlim = np.where(hit, t, np.inf)
        cand = (tc > 0.0) & (tc < tlim)
        dist2 = dot_np(Lo, Lo)
        perp2 = dist2 - tc * tc
        arr = cand & (perp2 <= r2)
        if arr.any():
            k = a[arr]
            Y = ref_sh.eval_sh_batch(-d[k], order).astype(np.float32)
            contrib = (E[k][:, :, None] * Y[:, None, :]).astype(np.float64)
            direct = nrefl[k] == 0
            Dir += contrib[direct].sum(axis=0)
            q = (plen[k] + tc[arr]) / bin_len
            keep = (~direct) & (q < w.n_bins)
            np.add.at(H, q[keep].astype(np.int64), contrib[keep])
        nseg[a] += 1
        miss = a[~hit]
        active[miss] = False
        h = a[hit]
        th = t[hit]
        plen[h] += th
        o[h] = o[h] + th[:, None] * d[h]
        nrefl[h] += 1
        tri_h = tri[hit]
        m = w.material_index[tri_h]
        nrm = model.normals[tri_h]
        u1, _ = draw2_np(rays[h], nrefl[h].astype(np.uint32), 0, frame, w.seed, src_index)
        diffuse = u1 < pd[m]
        f = np.where(diffuse[:, None], fd[m], fs[m])
        E[h] = E[h] * f
        nd = dot_np(nrm, d[h])
        newd = d[h].copy()
        spec = ~diffuse
        k2 = 2.0 * nd[spec]
        newd[spec] = d[h][spec] - k2[:, None] * nrm[spec]
        if diffuse.any():
            nn = nrm[diffuse].copy()
            flip = nd[diffuse] > 0.0
            nn[flip] = -nn[flip]
            newd[diffuse] = sample_cosine_np(w.seed, src_index, rays[h][diffuse],
                                             nrefl[h][diffuse].astype(np.uint32), frame, nn)
        d[h] = newd
        active[h[nrefl[h] >= w.max_bounces]] = False
    return dict(H=H, Dir=Dir, nseg=nseg, ids=ids, e0=np.float32(e0))


def main():
    os.makedirs(GOLD, exist_ok=True)
    # --- t-designs (data tables, also shipped to the product) -----------------
    td = {f"t{d}": np.array(ref_td._TABLES[d]) for d in ref_td.AVAILABLE_DEGREES}
    np.savez_compressed(os.path.join(GOLD, "tdesigns.npz"), **td)
    datadir = os.path.join(ROOT, "paper_1803_00430_b200", "data")
    os.makedirs(datadir, exist_ok=True)
    np.savez_compressed(os.path.join(datadir, "tdesigns.npz"), **td)

    # --- box scene (test_scene.py:107-142) ------------------------------------
    box = ref_scene.make_box_scene(size=10.0)
    rng = np.random.default_rng(0)
    dirs = rng.normal(size=(100, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    origins = rng.uniform(-4, 4, size=(100, 3))
    t, tri, hit = box.intersect_batch(origins, dirs)
    st = np.zeros(100); stri = np.zeros(100, np.int64)
    for i in range(100):
        h = box.intersect(origins[i], dirs[i])
        st[i], stri[i] = h.distance, h.triangle
    rt_t, rt_v = ref_bvh.ray_triangles_batch(origins, dirs, box.v0, box.e1, box.e2, 1e-4)
    rs_t, rs_v = ref_bvh.ray_triangles(origins[3], dirs[3], box.v0, box.e1, box.e2, 1e-4, 7.5)
    special_o = np.array([[0.0, 0, 0], [5.0, 0, 0], [0.0, 0, 0]])
    special_d = np.array([[1.0, 0, 0], [1.0, 0, 0], [0.0, 0, 1.0]])
    sp = [box.bvh.intersect(special_o[i], special_d[i], 1e-4, np.inf) for i in range(3)]
    np.savez_compressed(os.path.join(GOLD, "box.npz"), v0=box.v0, e1=box.e1, e2=box.e2,
             normals=box.normals, material_index=box.material_index,
             absorption=box.absorption, scattering=box.scattering,
             origins=origins, dirs=dirs, t=t, tri=tri, hit=hit, scalar_t=st, scalar_tri=stri,
             special_o=special_o, special_d=special_d,
             special_t=np.array([s[0] for s in sp]), special_tri=np.array([s[1] for s in sp]),
             rt_t=rt_t, rt_valid=rt_v, rs_t=rs_t, rs_valid=rs_v, **_bvh_arrays(box))

    # --- 700-triangle soup, seed 7 (test_scene.py:145-169) ---------------------
    rng = np.random.default_rng(7)
    n_tris = 700
    centers = rng.uniform(-5, 5, size=(n_tris, 3))
    a = centers + rng.normal(scale=0.4, size=(n_tris, 3))
    b = centers + rng.normal(scale=0.4, size=(n_tris, 3))
    c = centers + rng.normal(scale=0.4, size=(n_tris, 3))
    mat = ref_scene.Material("m", [0.1] * 4, [0.5] * 4)
    soup = ref_scene.SceneModel(a, b - a, c - a, np.zeros(n_tris, dtype=np.int64), [mat],
                                [ref_scene.Source(id="s", position=np.zeros(3))],
                                ref_scene.Listener(position=np.zeros(3)))
    n_rays = 10_000
    origins = rng.uniform(-6, 6, size=(n_rays, 3))
    dirs = rng.normal(size=(n_rays, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    bt = np.zeros(n_rays); btri = np.zeros(n_rays, np.int64)
    vt = np.zeros(n_rays); vtri = np.zeros(n_rays, np.int64)
    for i in range(n_rays):
        bt[i], btri[i] = soup.intersect_brute(origins[i], dirs[i])
        vt[i], vtri[i] = soup.bvh.intersect(origins[i], dirs[i], 1e-4, np.inf)
    allt, alltri, allhit = ref_scene.SceneModel.intersect_batch(soup, origins[:2000], dirs[:2000])
    # brute batch path on the same soup (forced: call the all-pairs kernel)
    tb, vb = ref_bvh.ray_triangles_batch(origins[:2000], dirs[:2000], soup.v0, soup.e1, soup.e2, 1e-4)
    tb = np.where(vb, tb, np.inf)
    k = np.argmin(tb, axis=1)
    bb = tb[np.arange(2000), k]
    np.savez_compressed(os.path.join(GOLD, "soup700.npz"), v0=soup.v0, e1=soup.e1, e2=soup.e2,
             normals=soup.normals, material_index=soup.material_index,
             absorption=soup.absorption, scattering=soup.scattering,
             origins=origins, dirs=dirs, brute_t=bt, brute_tri=btri, bvh_t=vt, bvh_tri=vtri,
             batch_t=allt, batch_tri=alltri, allpairs_t=bb,
             allpairs_tri=np.where(np.isfinite(bb), k, -1), **_bvh_arrays(soup))

    # --- SH (sh.py) -----------------------------------------------------------
    rng = np.random.default_rng(11)
    d = rng.normal(size=(500, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    shd = {f"Y{o}": ref_sh.eval_sh_batch(d, o) for o in range(5)}
    avgs = {}
    for o in (1, 2, 3, 4):
        nc = (o + 1) ** 2
        for j in range(4):
            v = rng.normal(size=nc) * 0.1
            v[0] = abs(v[0]) + 0.05 * j
            avgs[f"avg{o}_{j}"] = v
            avgs[f"D{o}_{j}"] = ref_sh.directional_loudness_matrix(v, o)
        iso = np.zeros(nc); iso[0] = ref_sh.SH_C0
        avgs[f"avg{o}_iso"] = iso
        avgs[f"D{o}_iso"] = ref_sh.directional_loudness_matrix(iso, o)
    rots = []
    for j in range(5):
        q = rng.normal(size=4)
        R = ref_scene.quat_to_matrix(q)
        rots.append(R)
        avgs[f"J{j}"] = ref_sh.sh_rotation(R, 4).matrix
    np.savez_compressed(os.path.join(GOLD, "sh.npz"), dirs=d, R=np.array(rots), **shd, **avgs)

    # --- C1 shoebox bounce loop, every hit answered by the reference -----------
    w = workloads.c1_shoebox()
    model = _model_from_workload(w)
    rays = np.arange(w.n_rays, dtype=np.uint32)
    res = trace_reference(model, w, 0, rays)
    np.savez_compressed(os.path.join(GOLD, "c1_trace.npz"), rays=rays, **res, **w.arrays(),
             **_bvh_arrays(model))

    # --- C2 city: reference BVH + BVH-path queries + a traced subsample --------
    w = workloads.c2_city()
    model = _model_from_workload(w)
    rng = np.random.default_rng(21)
    q_o = np.concatenate([np.repeat(w.sources[:1], 600, axis=0),
                          rng.uniform([0, 0, 0.5], [500, 500, 80], size=(600, 3))])
    q_d = rng.normal(size=(1200, 3))
    q_d /= np.linalg.norm(q_d, axis=1, keepdims=True)
    ct, ctri, chit = model.intersect_batch(q_o, q_d)
    rays = np.arange(256, dtype=np.uint32)
    res = trace_reference(model, w, 0, rays)
    np.savez_compressed(os.path.join(GOLD, "c2_city.npz"), q_o=q_o, q_d=q_d, q_t=ct, q_tri=ctri,
             rays=rays, **{f"trace_{k}": v for k, v in res.items()}, **w.arrays(),
             **_bvh_arrays(model))
    print("golden fixtures written to", GOLD)


if __name__ == "__main__":
    main()
