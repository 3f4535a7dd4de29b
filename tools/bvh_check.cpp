// CPU check of the host BVH builder (bvh_build.cpp), including spatial
// splits: every triangle is referenced, and closest hits found through the
// 4-wide tree's f32 boxes equal brute force over all triangles for random
// rays (same f64 test, lowest id on equal t).  Built and run by
// tests/test_bvh_host.py:  bvh_check <triangles.bin> <n_rays> <seed>
#include <cmath>
#include <cstdio>
#include <cstdlib>
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
    if (u < 0.0 || u > 1.0) return false;
    const double q[3] = {s[1] * e1[2] - s[2] * e1[1], s[2] * e1[0] - s[0] * e1[2], s[0] * e1[1] - s[1] * e1[0]};
    const double w = (d[0] * q[0] + d[1] * q[1] + d[2] * q[2]) * inv;
    if (w < 0.0 || u + w > 1.0) return false;
    t = (e2[0] * q[0] + e2[1] * q[1] + e2[2] * q[2]) * inv;
    return t > 1e-4 && t < tmax;
}

int main(int argc, char** argv) {
    if (argc < 4) return 2;
    FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 2;
    int64_t n = 0;
    if (std::fread(&n, 8, 1, f) != 1) return 2;
    std::vector<double> v0(3 * n), e1(3 * n), e2(3 * n);
    if (std::fread(v0.data(), 8, 3 * n, f) != (size_t)(3 * n) || std::fread(e1.data(), 8, 3 * n, f) != (size_t)(3 * n) ||
        std::fread(e2.data(), 8, 3 * n, f) != (size_t)(3 * n))
        return 2;
    std::fclose(f);
    HostBvh b;
    build_bvh(v0.data(), e1.data(), e2.data(), n, b);
    std::vector<int> seen(n, 0);
    for (int64_t id : b.order) seen[id]++;
    for (int64_t t = 0; t < n; ++t)
        if (!seen[t]) { std::printf("FAIL triangle %lld not referenced\n", (long long)t); return 1; }
    std::vector<double> tri(9 * b.order.size());
    for (size_t i = 0; i < b.order.size(); ++i)
        for (int k = 0; k < 3; ++k) {
            const int64_t id = b.order[i];
            tri[9 * i + k] = v0[3 * id + k];
            tri[9 * i + 3 + k] = e1[3 * id + k];
            tri[9 * i + 6 + k] = e2[3 * id + k];
        }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int64_t t = 0; t < n; ++t)
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], v0[3 * t + k]);
            hi[k] = std::max(hi[k], v0[3 * t + k]);
        }
    const long rays = std::atol(argv[2]);
    std::mt19937_64 rng(std::atol(argv[3]));
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::normal_distribution<double> N(0.0, 1.0);
    long bad = 0, hits = 0;
    double visits = 0;
    for (long r = 0; r < rays; ++r) {
        double o[3], d[3];
        for (int k = 0; k < 3; ++k) o[k] = lo[k] + (hi[k] - lo[k]) * U(rng);
        double nn = 0;
        for (int k = 0; k < 3; ++k) { d[k] = N(rng); nn += d[k] * d[k]; }
        for (int k = 0; k < 3; ++k) d[k] /= std::sqrt(nn);
        // brute force
        double bt = INFINITY; int64_t bid = -1;
        for (int64_t t = 0; t < n; ++t) {
            double tt;
            double v[9];
            for (int k = 0; k < 3; ++k) { v[k] = v0[3 * t + k]; v[3 + k] = e1[3 * t + k]; v[6 + k] = e2[3 * t + k]; }
            if (mt(o, d, v, INFINITY, tt) && (tt < bt || (tt == bt && t < bid))) { bt = tt; bid = t; }
        }
        // tree (f64 slab test on the f32 boxes, any order, prune by t)
        double tt_best = INFINITY; int64_t tid = -1;
        std::vector<int32_t> stack = {0};
        while (!stack.empty()) {
            const GpuNode& g = b.nodes[stack.back()];
            stack.pop_back();
            visits += 1;
            for (int c = 0; c < 4; ++c) {
                if (g.child[c] == kEmptyChild) continue;
                const double bl[3] = {g.lox[c], g.loy[c], g.loz[c]}, bh[3] = {g.hix[c], g.hiy[c], g.hiz[c]};
                double t0 = 0.0, t1 = tt_best;
                for (int k = 0; k < 3 && t0 <= t1; ++k) {
                    if (d[k] == 0.0) { if (o[k] < bl[k] || o[k] > bh[k]) t0 = INFINITY; continue; }
                    double a = (bl[k] - o[k]) / d[k], z = (bh[k] - o[k]) / d[k];
                    if (a > z) std::swap(a, z);
                    t0 = std::max(t0, a);
                    t1 = std::min(t1, z);
                }
                if (!(t0 <= t1)) continue;
                if (g.child[c] >= 0) { stack.push_back(g.child[c]); continue; }
                const uint32_t e = ~(uint32_t)g.child[c];
                const uint32_t start = e >> 3, cnt = (e & 7u) + 1u;
                for (uint32_t j = 0; j < cnt; ++j) {
                    double tt;
                    const int64_t id = b.order[start + j];
                    if (mt(o, d, &tri[9 * (start + j)], INFINITY, tt) && (tt < tt_best || (tt == tt_best && id < tid))) {
                        tt_best = tt; tid = id;
                    }
                }
            }
        }
        if (bid >= 0) ++hits;
        if (bid != tid || (bid >= 0 && bt != tt_best)) {
            if (++bad <= 5) std::printf("MISMATCH ray %ld brute %lld %.17g tree %lld %.17g\n", r, (long long)bid, bt, (long long)tid, tt_best);
        }
    }
    std::printf("n_tri %lld refs %zu nodes %zu depth %d max_leaf %d rays %ld hits %ld bad %ld visits/ray %.2f\n",
                (long long)n, b.order.size(), b.nodes.size(), b.max_depth, b.max_leaf, rays, hits, bad, visits / rays);
    return bad ? 1 : 0;
}
