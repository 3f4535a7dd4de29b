// CPU simulation of node-visit counts for W-wide collapses of the host
// builder's binary tree (W = 4 is the device tree; 8 / 16 are what a wider
// node would visit), on geometrically simulated paths like sim_bottomup.cpp.
// Prints visits, box tests and dependent steps per segment.
//   sim_width <scene.bin> <paths> <max_bounces> <seed> <W> [mode]
// mode 0: open the largest-area inner child (the builder's rule)
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

struct WChild { float lo[3], hi[3]; int32_t ref; };   // ref >= 0 inner, < 0 leaf ~((start << 3) | (count - 1))
struct WNode { int first, n; };

struct Tree {
    HostBvh b;
    std::vector<WNode> nodes;
    std::vector<WChild> kids;
    std::vector<double> tri;
    int depth = 0;
};

static double harea(const HostBinNode& n) {
    const double dx = n.hi[0] - n.lo[0], dy = n.hi[1] - n.lo[1], dz = n.hi[2] - n.lo[2];
    return dx * dy + dy * dz + dz * dx;
}

// SAH-optimal collapse (dynamic programme of Ylitie, Karras & Laine 2017,
// section 3.1, with the builder's leaves kept): cost[n][i] = least sum of
// wide-node areas for the subtree of binary node n represented by at most
// i + 1 roots; a wide node's W children are the best W-root forest.
static void collapse_dp(Tree& T, int W) {
    const auto& B = T.b.binary;
    const size_t nb = B.size();
    std::vector<double> cost(nb * W, 0.0);       // [n][i], i = 0..W-1 -> at most i+1 roots
    std::vector<int8_t> split(nb * W, 0);        // k (roots given to the left child), 0: use [i-1]
    std::vector<double> dist(nb * (W + 1), 0.0); // distribute cost for j = 2..W roots
    std::vector<int8_t> dsplit(nb * (W + 1), 0);
    // post-order over the binary tree
    std::vector<int32_t> order, st = {T.b.binary_root};
    while (!st.empty()) {
        const int32_t n = st.back();
        st.pop_back();
        order.push_back(n);
        if (B[n].left >= 0) { st.push_back(B[n].left); st.push_back(B[n].right); }
    }
    for (size_t q = order.size(); q-- > 0;) {
        const int32_t n = order[q];
        if (B[n].left < 0) {
            for (int i = 0; i < W; ++i) cost[n * W + i] = 0.0;   // leaves cost the same in every collapse
            continue;
        }
        const int32_t l = B[n].left, r = B[n].right;
        for (int j = 2; j <= W; ++j) {
            double best = INFINITY;
            int bk = 1;
            for (int k = 1; k < j; ++k) {
                const double c = cost[l * W + (k - 1)] + cost[r * W + (j - k - 1)];
                if (c < best) { best = c; bk = k; }
            }
            dist[n * (W + 1) + j] = best;
            dsplit[n * (W + 1) + j] = (int8_t)bk;
        }
        cost[n * W + 0] = dist[n * (W + 1) + W] + harea(B[n]);   // one root: n is a wide node
        for (int i = 1; i < W; ++i) {
            const double d = dist[n * (W + 1) + (i + 1)];
            if (d < cost[n * W + i - 1]) { cost[n * W + i] = d; split[n * W + i] = 1; }
            else { cost[n * W + i] = cost[n * W + i - 1]; split[n * W + i] = 0; }
        }
    }
    // roots of the best (<= i+1)-root forest of subtree n
    struct F { int32_t n; int i; };
    auto forest = [&](int32_t n0, int j0, std::vector<int32_t>& out) {
        // distribute j0 roots over n0's children
        std::vector<F> fs;
        const int k0 = dsplit[n0 * (W + 1) + j0];
        fs.push_back({B[n0].left, k0 - 1});
        fs.push_back({B[n0].right, j0 - k0 - 1});
        while (!fs.empty()) {
            F f = fs.back();
            fs.pop_back();
            if (B[f.n].left < 0) { out.push_back(f.n); continue; }
            int i = f.i;
            while (i > 0 && split[f.n * W + i] == 0) --i;
            if (i == 0) { out.push_back(f.n); continue; }   // a single root: wide node (or leaf)
            const int j = i + 1, k = dsplit[f.n * (W + 1) + j];
            fs.push_back({B[f.n].left, k - 1});
            fs.push_back({B[f.n].right, j - k - 1});
        }
    };
    struct Item { int32_t bn; int32_t slot; int depth; };
    std::vector<Item> stack;
    T.nodes.push_back({0, 0});
    stack.push_back({T.b.binary_root, 0, 1});
    const float pad = (float)T.b.pad;
    while (!stack.empty()) {
        Item it = stack.back();
        stack.pop_back();
        T.depth = std::max(T.depth, it.depth);
        std::vector<int32_t> kids;
        forest(it.bn, W, kids);
        WNode nd{(int)T.kids.size(), (int)kids.size()};
        const size_t base = T.kids.size();
        T.kids.resize(base + kids.size());
        for (size_t c = 0; c < kids.size(); ++c) {
            const HostBinNode& ch = B[kids[c]];
            WChild k;
            for (int a = 0; a < 3; ++a) {
                k.lo[a] = std::nextafterf((float)(ch.lo[a] - pad), -INFINITY);
                k.hi[a] = std::nextafterf((float)(ch.hi[a] + pad), INFINITY);
            }
            if (ch.left < 0) k.ref = ~(int32_t)((ch.start << 3) | (ch.count - 1));
            else {
                k.ref = (int32_t)T.nodes.size();
                T.nodes.push_back({0, 0});
                stack.push_back({kids[c], k.ref, it.depth + 1});
            }
            T.kids[base + c] = k;
        }
        T.nodes[it.slot] = nd;
    }
}

static void collapse(Tree& T, int W) {
    const auto& B = T.b.binary;
    struct Item { int32_t bn; int32_t slot; int depth; };
    std::vector<Item> stack;
    T.nodes.push_back({0, 0});
    stack.push_back({T.b.binary_root, 0, 1});
    const float pad = (float)T.b.pad;
    while (!stack.empty()) {
        Item it = stack.back();
        stack.pop_back();
        T.depth = std::max(T.depth, it.depth);
        std::vector<int32_t> kids = {B[it.bn].left, B[it.bn].right};
        while ((int)kids.size() < W) {
            int best = -1;
            double ba = -1;
            for (size_t c = 0; c < kids.size(); ++c)
                if (B[kids[c]].left >= 0 && harea(B[kids[c]]) > ba) { ba = harea(B[kids[c]]); best = (int)c; }
            if (best < 0) break;
            const int32_t op = kids[best];
            kids[best] = B[op].left;
            kids.push_back(B[op].right);
        }
        WNode nd{(int)T.kids.size(), (int)kids.size()};
        const size_t base = T.kids.size();
        T.kids.resize(base + kids.size());
        for (size_t c = 0; c < kids.size(); ++c) {
            const HostBinNode& ch = B[kids[c]];
            WChild k;
            for (int a = 0; a < 3; ++a) {
                k.lo[a] = std::nextafterf((float)(ch.lo[a] - pad), -INFINITY);
                k.hi[a] = std::nextafterf((float)(ch.hi[a] + pad), INFINITY);
            }
            if (ch.left < 0) k.ref = ~(int32_t)((ch.start << 3) | (ch.count - 1));
            else {
                k.ref = (int32_t)T.nodes.size();
                T.nodes.push_back({0, 0});
                stack.push_back({kids[c], k.ref, it.depth + 1});
            }
            T.kids[base + c] = k;
        }
        T.nodes[it.slot] = nd;
    }
}

struct Counters { double visits = 0, boxes = 0, tests = 0, segs = 0, pushes = 0, hit1 = 0; };
struct Hit { double t = INFINITY; int64_t id = INT32_MAX; };

static void traverse(const Tree& T, const double* o, const double* d, const double* inv, Hit& h, Counters& C) {
    struct E { int32_t n; float t; };
    E stack[256];
    int sp = 0;
    float tb = 1e38f;
    int32_t node = 0;
    for (;;) {
        while (node >= 0) {
            C.visits++;
            const WNode& g = T.nodes[node];
            E k[32];
            int nh = 0;
            for (int c = 0; c < g.n; ++c) {
                const WChild& b = T.kids[g.first + c];
                C.boxes++;
                float n = 1e-4f, f = tb;
                for (int a = 0; a < 3; ++a) {
                    float x = (float)((b.lo[a] - o[a]) * inv[a]), y = (float)((b.hi[a] - o[a]) * inv[a]);
                    if (x > y) std::swap(x, y);
                    n = std::max(n, x);
                    f = std::min(f, y);
                }
                if (n <= f) k[nh++] = {b.ref, n};
            }
            if (nh == 1) C.hit1++;
            std::sort(k, k + nh, [](const E& a, const E& b) { return a.t < b.t; });
            for (int i = nh - 1; i >= 1; --i) { stack[sp++] = k[i]; C.pushes++; }
            if (nh) { node = k[0].n; continue; }
            bool got = false;
            while (sp) {
                E e = stack[--sp];
                if (e.t <= tb) { node = e.n; got = true; break; }
            }
            if (!got) return;
        }
        const uint32_t e = ~(uint32_t)node;
        const uint32_t start = e >> 3, cnt = (e & 7u) + 1u;
        for (uint32_t i = 0; i < cnt; ++i) {
            C.tests++;
            double t;
            const int64_t id = T.b.order[start + i];
            if (mt(o, d, &T.tri[9 * (start + i)], h.t, t) && (t < h.t || id < h.id)) {
                h.t = t; h.id = id;
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
    if (argc < 6) return 2;
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
    const int W = std::atoi(argv[5]);
    Tree T;
    T.b.keep_binary = true;
    build_bvh(v0.data(), e1.data(), e2.data(), n, T.b);
    if (argc > 6 && std::atoi(argv[6]) == 1) collapse_dp(T, W);
    else collapse(T, W);
    const size_t nr = T.b.order.size();
    T.tri.resize(9 * nr);
    for (size_t i = 0; i < nr; ++i) {
        const int64_t id = T.b.order[i];
        for (int k = 0; k < 3; ++k) {
            T.tri[9 * i + k] = v0[3 * id + k];
            T.tri[9 * i + 3 + k] = e1[3 * id + k];
            T.tri[9 * i + 6 + k] = e2[3 * id + k];
        }
    }
    std::printf("W %d: nodes %zu, children %zu (%.2f per node), depth %d\n", W, T.nodes.size(), T.kids.size(),
                (double)T.kids.size() / T.nodes.size(), T.depth);
    const long paths = std::atol(argv[2]);
    const int max_b = std::atoi(argv[3]);
    std::mt19937_64 rng(std::atol(argv[4]));
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::normal_distribution<double> N(0.0, 1.0);
    Counters C;
    for (long p = 0; p < paths; ++p) {
        double o[3], d[3];
        const int s = (int)(p % ns);
        for (int k = 0; k < 3; ++k) o[k] = src[3 * s + k];
        double nrm = 0;
        for (int k = 0; k < 3; ++k) { d[k] = N(rng); nrm += d[k] * d[k]; }
        for (int k = 0; k < 3; ++k) d[k] /= std::sqrt(nrm);
        for (int bnc = 0; bnc < max_b; ++bnc) {
            double inv[3];
            for (int k = 0; k < 3; ++k) inv[k] = 1.0 / (std::fabs(d[k]) < 1e-20 ? 1e-20 : d[k]);
            Hit h;
            traverse(T, o, d, inv, h, C);
            C.segs++;
            if (h.id == INT32_MAX) break;
            const int64_t id = h.id;
            double nx = e1[3 * id + 1] * e2[3 * id + 2] - e1[3 * id + 2] * e2[3 * id + 1];
            double ny = e1[3 * id + 2] * e2[3 * id + 0] - e1[3 * id + 0] * e2[3 * id + 2];
            double nz = e1[3 * id + 0] * e2[3 * id + 1] - e1[3 * id + 1] * e2[3 * id + 0];
            const double nl = std::sqrt(nx * nx + ny * ny + nz * nz);
            nx /= nl; ny /= nl; nz /= nl;
            if (nx * d[0] + ny * d[1] + nz * d[2] > 0) { nx = -nx; ny = -ny; nz = -nz; }
            for (int k = 0; k < 3; ++k) o[k] += h.t * d[k];
            if (U(rng) < 0.5) {
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
        }
    }
    std::printf("segments %.0f: visits/seg %.2f, box tests/seg %.1f, triangle tests/seg %.2f, pushes/seg %.2f, "
                "single-hit visits %.2f\n",
                C.segs, C.visits / C.segs, C.boxes / C.segs, C.tests / C.segs, C.pushes / C.segs, C.hit1 / C.segs);
    return 0;
}
