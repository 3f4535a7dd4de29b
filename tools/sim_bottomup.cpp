// CPU simulation of node-visit counts (not a timing tool): the trace
// kernel's top-down closest-hit traversal of the host-built 4-wide tree vs a
// bottom-up traversal that starts at the leaf of the triangle a bounce ray
// leaves and stops climbing once the segment [origin, closest hit] lies in
// the current ancestor's "safe box" (a sub-box of the node's box that no
// box outside its subtree touches).  Paths are simulated geometrically
// (cosine-lobe bounces from the sources, max_bounces), which reproduces the
// segment mix (primary / bounce / escape) of the real frames.
//   sim_bottomup <scene.bin> <paths> <max_bounces> <seed>
// scene.bin: int64 n, v0 (n,3), e1 (n,3), e2 (n,3) f64, int64 n_src, src (n_src,3) f64
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "ef_internal.h"

using namespace ef;

static bool mt(const double* o, const double* d, const double* v, double tmax, double& t) {
    const double *v0 = v, *e1 = v + 3, *e2 = v + 6;
    const double p[3] = {d[1] * e2[2] - d[2] * e2[1], d[2] * e2[0] - d[0] * e2[2], d[0] * e2[1] - d[1] * e2[0]};
    const double det = e1[0] * p[0] + e1[1] * p[1] + e1[2] * p[2];
    if (std::fabs(det) < 1e-14) return false;
    const double inv = 1.0 / det;
    const double s[3] = {o[0] - v0[0], o[1] - v0[1], o[2] - v0[2]};
    const double u = (s[0] * p[0] + s[1] * p[1] + s[2] * p[2]) * inv;
    if (u < -1e-10) return false;
    const double q[3] = {s[1] * e1[2] - s[2] * e1[1], s[2] * e1[0] - s[0] * e1[2], s[0] * e1[1] - s[1] * e1[0]};
    const double w = (d[0] * q[0] + d[1] * q[1] + d[2] * q[2]) * inv;
    if (w < -1e-10 || u + w > 1.0 + 1e-10) return false;
    t = (e2[0] * q[0] + e2[1] * q[1] + e2[2] * q[2]) * inv;
    return t > 1e-4 && t <= tmax;
}

struct Box6 { float lo[3], hi[3]; };

struct Tree {
    HostBvh b;
    std::vector<double> tri;            // leaf order, 9 per ref
    std::vector<int32_t> parent, pslot; // per node
    std::vector<int32_t> leaf_parent, leaf_slot;   // per leaf start position
    std::vector<Box6> safe;             // per node
    std::vector<int64_t> ref_of_tri;    // one reference (leaf position) per triangle id
};

static Box6 child_box(const GpuNode& g, int c) {
    Box6 b;
    b.lo[0] = g.lox[c]; b.hi[0] = g.hix[c];
    b.lo[1] = g.loy[c]; b.hi[1] = g.hiy[c];
    b.lo[2] = g.loz[c]; b.hi[2] = g.hiz[c];
    return b;
}

// shrink `s` so it no longer overlaps `o` (cut along the axis losing the least volume)
static void cut(Box6& s, const Box6& o, float margin) {
    for (int k = 0; k < 3; ++k)
        if (o.hi[k] + margin <= s.lo[k] || o.lo[k] - margin >= s.hi[k]) return;   // disjoint already
    double best = -1.0;
    int bk = 0, bside = 0;
    double ext[3];
    for (int k = 0; k < 3; ++k) ext[k] = std::max(0.0, (double)s.hi[k] - s.lo[k]);
    for (int k = 0; k < 3; ++k) {
        // keep [s.lo, o.lo - margin] or [o.hi + margin, s.hi]
        const double keep_lo = std::max(0.0, (double)(o.lo[k] - margin) - s.lo[k]);
        const double keep_hi = std::max(0.0, (double)s.hi[k] - (o.hi[k] + margin));
        const double other = ext[(k + 1) % 3] * ext[(k + 2) % 3];
        if (keep_lo * other > best) { best = keep_lo * other; bk = k; bside = 0; }
        if (keep_hi * other > best) { best = keep_hi * other; bk = k; bside = 1; }
    }
    if (bside == 0) s.hi[bk] = std::min(s.hi[bk], o.lo[bk] - margin);
    else s.lo[bk] = std::max(s.lo[bk], o.hi[bk] + margin);
    if (s.hi[bk] < s.lo[bk]) s.hi[bk] = s.lo[bk] = 0.f, s.hi[0] = s.lo[0] - 1.f;   // empty
}

static bool empty(const Box6& s) { return s.hi[0] < s.lo[0] || s.hi[1] < s.lo[1] || s.hi[2] < s.lo[2]; }
static bool inside(const Box6& s, const double* p) {
    for (int k = 0; k < 3; ++k)
        if (!(p[k] >= s.lo[k] && p[k] <= s.hi[k])) return false;
    return true;
}

struct Counters {
    double visits = 0, leaves = 0, tests = 0, climbs = 0, early = 0, segs = 0;
};

// key of a child box for ray (o, inv), [tmin, tmax]
static bool slab(const Box6& b, const double* o, const double* inv, float tmin, float tmax, float& tn) {
    float n = tmin, f = tmax;
    for (int k = 0; k < 3; ++k) {
        float a = (float)((b.lo[k] - o[k]) * inv[k]), c = (float)((b.hi[k] - o[k]) * inv[k]);
        if (a > c) std::swap(a, c);
        n = std::max(n, a);
        f = std::min(f, c);
    }
    tn = n;
    return n <= f;
}

struct Hit { double t = INFINITY; int64_t id = INT32_MAX; int32_t leaf = 0; };

// traverse the subtree entered at `node` (inner index >= 0 or leaf enc < 0); skips child `skip`
static void traverse(const Tree& T, int32_t node, int32_t skip, const double* o, const double* d, const double* inv,
                     Hit& h, Counters& C) {
    struct E { int32_t n; float t; };
    E stack[128];
    int sp = 0;
    float tb = (float)std::min(h.t * (1.0 + 1e-6), 1e38);
    for (;;) {
        while (node >= 0) {
            C.visits++;
            const GpuNode& g = T.b.nodes[node];
            E k[4];
            int nh = 0;
            for (int c = 0; c < 4; ++c) {
                if (g.child[c] == kEmptyChild || g.child[c] == skip) continue;
                float tn;
                if (slab(child_box(g, c), o, inv, 1e-4f, tb, tn)) k[nh++] = {g.child[c], tn};
            }
            std::sort(k, k + nh, [](const E& a, const E& b) { return a.t < b.t; });
            for (int i = nh - 1; i >= 1; --i) stack[sp++] = k[i];
            if (nh) { node = k[0].n; continue; }
            bool got = false;
            while (sp) {
                E e = stack[--sp];
                if (e.t <= tb) { node = e.n; got = true; break; }
            }
            if (!got) return;
        }
        // leaf
        C.leaves++;
        const uint32_t e = ~(uint32_t)node;
        const uint32_t start = e >> 3, cnt = (e & 7u) + 1u;
        for (uint32_t i = 0; i < cnt; ++i) {
            C.tests++;
            double t;
            const int64_t id = T.b.order[start + i];
            if (mt(o, d, &T.tri[9 * (start + i)], h.t, t) && (t < h.t || id < h.id)) {
                h.t = t; h.id = id; h.leaf = node;
                tb = (float)std::min(t * (1.0 + 1e-6), 1e38);
            }
        }
        bool got = false;
        while (sp) {
            E e2 = stack[--sp];
            if (e2.t <= tb) { node = e2.n; got = true; break; }
        }
        if (!got) return;
    }
}

int main(int argc, char** argv) {
    if (argc < 5) return 2;
    FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 2;
    int64_t n = 0, ns = 0;
    if (std::fread(&n, 8, 1, f) != 1) return 2;
    std::vector<double> v0(3 * n), e1(3 * n), e2(3 * n);
    if (std::fread(v0.data(), 8, 3 * n, f) != (size_t)(3 * n) || std::fread(e1.data(), 8, 3 * n, f) != (size_t)(3 * n) ||
        std::fread(e2.data(), 8, 3 * n, f) != (size_t)(3 * n))
        return 2;
    if (std::fread(&ns, 8, 1, f) != 1) return 2;
    std::vector<double> src(3 * ns);
    if (std::fread(src.data(), 8, 3 * ns, f) != (size_t)(3 * ns)) return 2;
    std::fclose(f);
    Tree T;
    build_bvh(v0.data(), e1.data(), e2.data(), n, T.b);
    const size_t nn = T.b.nodes.size(), nr = T.b.order.size();
    std::printf("triangles %lld refs %zu nodes %zu depth %d\n", (long long)n, nr, nn, T.b.max_depth);
    T.tri.resize(9 * nr);
    T.ref_of_tri.assign(n, -1);
    for (size_t i = 0; i < nr; ++i) {
        const int64_t id = T.b.order[i];
        for (int k = 0; k < 3; ++k) {
            T.tri[9 * i + k] = v0[3 * id + k];
            T.tri[9 * i + 3 + k] = e1[3 * id + k];
            T.tri[9 * i + 6 + k] = e2[3 * id + k];
        }
    }
    T.parent.assign(nn, -1);
    T.pslot.assign(nn, 0);
    T.leaf_parent.assign(nr, -1);
    T.leaf_slot.assign(nr, 0);
    for (size_t i = 0; i < nn; ++i)
        for (int c = 0; c < 4; ++c) {
            const int32_t ch = T.b.nodes[i].child[c];
            if (ch == kEmptyChild) continue;
            if (ch >= 0) { T.parent[ch] = (int32_t)i; T.pslot[ch] = c; }
            else { const uint32_t e = ~(uint32_t)ch; T.leaf_parent[e >> 3] = (int32_t)i; T.leaf_slot[e >> 3] = c; }
        }
    // safe boxes, top-down (children are numbered after their parents)
    const float margin = (float)(2.0 * T.b.pad);
    T.safe.resize(nn);
    for (int k = 0; k < 3; ++k) { T.safe[0].lo[k] = -INFINITY; T.safe[0].hi[k] = INFINITY; }
    double vol_ratio = 0; long vr_n = 0, n_empty = 0;
    for (size_t i = 0; i < nn; ++i) {
        const GpuNode& g = T.b.nodes[i];
        for (int c = 0; c < 4; ++c) {
            if (g.child[c] < 0) continue;   // leaves and empty slots carry no safe box
            Box6 s = child_box(g, c);
            const Box6 full = s;
            for (int k = 0; k < 3; ++k) {
                s.lo[k] = std::max(s.lo[k], T.safe[i].lo[k]);
                s.hi[k] = std::min(s.hi[k], T.safe[i].hi[k]);
            }
            for (int c2 = 0; c2 < 4 && !empty(s); ++c2)
                if (c2 != c && g.child[c2] != kEmptyChild) cut(s, child_box(g, c2), margin);
            if (empty(s)) { n_empty++; s.lo[0] = 1.f; s.hi[0] = 0.f; }
            else {
                double a = 1, b = 1;
                for (int k = 0; k < 3; ++k) { a *= (double)s.hi[k] - s.lo[k]; b *= (double)full.hi[k] - full.lo[k]; }
                if (b > 0) { vol_ratio += a / b; vr_n++; }
            }
            T.safe[g.child[c]] = s;
        }
    }
    std::printf("safe boxes: %ld empty of %zu, mean volume ratio %.3f\n", n_empty, nn, vol_ratio / std::max(1L, vr_n));

    const long paths = std::atol(argv[2]);
    const int max_b = std::atoi(argv[3]);
    std::mt19937_64 rng(std::atol(argv[4]));
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::normal_distribution<double> N(0.0, 1.0);
    Counters td, bu_hit, bu_esc, td_prim, td_hit, td_esc;
    long mism = 0;
    double climb_hist[40] = {0};
    for (long p = 0; p < paths; ++p) {
        double o[3], d[3];
        const int s = (int)(p % ns);
        for (int k = 0; k < 3; ++k) o[k] = src[3 * s + k];
        double nrm = 0;
        for (int k = 0; k < 3; ++k) { d[k] = N(rng); nrm += d[k] * d[k]; }
        for (int k = 0; k < 3; ++k) d[k] /= std::sqrt(nrm);
        int32_t from_leaf = 0;   // leaf enc of the triangle the ray leaves (0: none, primary)
        for (int bnc = 0; bnc < max_b; ++bnc) {
            double inv[3];
            for (int k = 0; k < 3; ++k) inv[k] = 1.0 / (std::fabs(d[k]) < 1e-20 ? 1e-20 : d[k]);
            // top-down (the kernel's traversal)
            Hit h;
            Counters c0;
            traverse(T, 0, kEmptyChild, o, d, inv, h, c0);
            const bool hit = h.id != INT32_MAX;
            Counters& cls = from_leaf == 0 ? td_prim : (hit ? td_hit : td_esc);
            cls.visits += c0.visits; cls.leaves += c0.leaves; cls.tests += c0.tests; cls.segs++;
            td.visits += c0.visits; td.tests += c0.tests; td.segs++;
            // bottom-up from the previous hit's leaf
            if (from_leaf != 0) {
                Hit hb;
                Counters c1;
                int32_t node = from_leaf;
                const uint32_t e = ~(uint32_t)from_leaf;
                int32_t up = T.leaf_parent[e >> 3];
                int32_t skip = kEmptyChild;
                int climbs = 0;
                bool early = false;
                // the starting leaf itself
                traverse(T, node, kEmptyChild, o, d, inv, hb, c1);
                skip = from_leaf;
                while (up >= 0) {
                    // subtree(up) minus `skip`
                    traverse(T, up, skip, o, d, inv, hb, c1);
                    climbs++;
                    // early-out: segment inside safe(up)?
                    if (hb.id != INT32_MAX) {
                        double e2[3];
                        for (int k = 0; k < 3; ++k) e2[k] = o[k] + hb.t * d[k];
                        if (inside(T.safe[up], o) && inside(T.safe[up], e2)) { early = true; break; }
                    }
                    skip = up;
                    up = T.parent[up];
                }
                if (hb.id != h.id || hb.t != h.t) mism++;
                Counters& cb = hit ? bu_hit : bu_esc;
                cb.visits += c1.visits; cb.leaves += c1.leaves; cb.tests += c1.tests; cb.segs++;
                cb.climbs += climbs; cb.early += early;
                if (hit) climb_hist[std::min(climbs, 39)]++;
            }
            if (!hit) break;
            // bounce: cosine lobe about the normal facing the incoming side
            const double* v = &T.tri[0];
            (void)v;
            const int64_t id = h.id;
            double nx = e1[3 * id + 1] * e2[3 * id + 2] - e1[3 * id + 2] * e2[3 * id + 1];
            double ny = e1[3 * id + 2] * e2[3 * id + 0] - e1[3 * id + 0] * e2[3 * id + 2];
            double nz = e1[3 * id + 0] * e2[3 * id + 1] - e1[3 * id + 1] * e2[3 * id + 0];
            const double nl = std::sqrt(nx * nx + ny * ny + nz * nz);
            nx /= nl; ny /= nl; nz /= nl;
            if (nx * d[0] + ny * d[1] + nz * d[2] > 0) { nx = -nx; ny = -ny; nz = -nz; }
            for (int k = 0; k < 3; ++k) o[k] += h.t * d[k];
            if (U(rng) < 0.5) {   // specular
                const double k2 = 2.0 * (nx * d[0] + ny * d[1] + nz * d[2]);
                d[0] -= k2 * nx; d[1] -= k2 * ny; d[2] -= k2 * nz;
            } else {
                double a, b2, ss;
                do { a = 2 * U(rng) - 1; b2 = 2 * U(rng) - 1; ss = a * a + b2 * b2; } while (ss >= 1.0);
                double t1[3], t2[3];
                const double sg = std::copysign(1.0, nz), aa = -1.0 / (sg + nz), bb = nx * ny * aa;
                t1[0] = 1.0 + sg * nx * nx * aa; t1[1] = sg * bb; t1[2] = -sg * nx;
                t2[0] = bb; t2[1] = sg + ny * ny * aa; t2[2] = -ny;
                const double z = std::sqrt(1.0 - ss);
                d[0] = a * t1[0] + b2 * t2[0] + z * nx;
                d[1] = a * t1[1] + b2 * t2[1] + z * ny;
                d[2] = a * t1[2] + b2 * t2[2] + z * nz;
            }
            from_leaf = h.leaf;
        }
    }
    auto pr = [](const char* name, const Counters& c) {
        if (c.segs == 0) return;
        std::printf("%-28s segs %10.0f visits/seg %6.2f leaves/seg %5.2f tests/seg %5.2f climbs/seg %5.2f early %.3f\n", name,
                    c.segs, c.visits / c.segs, c.leaves / c.segs, c.tests / c.segs, c.climbs / c.segs, c.early / c.segs);
    };
    pr("top-down all", td);
    pr("top-down primary", td_prim);
    pr("top-down bounce->hit", td_hit);
    pr("top-down bounce->escape", td_esc);
    pr("bottom-up bounce->hit", bu_hit);
    pr("bottom-up bounce->escape", bu_esc);
    std::printf("mismatches %ld\n", mism);
    std::printf("climb histogram (bounce->hit): ");
    for (int i = 0; i < 24; ++i) std::printf("%d:%.3f ", i, climb_hist[i] / std::max(1.0, bu_hit.segs));
    std::printf("\n");
    const double new_total = td_prim.visits + bu_hit.visits + bu_esc.visits;
    std::printf("visits per segment: top-down %.2f -> bottom-up for bounce rays %.2f\n", td.visits / td.segs,
                new_total / td.segs);
    return 0;
}
