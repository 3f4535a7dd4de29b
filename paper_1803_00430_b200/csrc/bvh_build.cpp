// Host-side binned-SAH BVH2 builder for the device traversal (K2).
//
// Replaces the reference's recursive Python builder (bvh.py:51-128: 16 bins
// on the widest centroid axis, leaves <= 4, median fallback).  The device
// tree is deliberately NOT the reference's tree: hit ids do not depend on the
// tree because the leaf test is the reference's exact f64 arithmetic and
// equal-t ties resolve to the lowest id.  What changes is the
// layout: two-child nodes holding both child boxes in f32 (64 B, four 16-byte
// loads per visited node), boxes rounded outward and padded so the f32 slab
// test never culls a hit the f64 test would accept, SAH over all three axes
// with 32 bins, and nodes numbered in depth-first order for locality.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "ef_internal.h"

namespace ef {
namespace {

struct Box {
    double lo[3] = {INFINITY, INFINITY, INFINITY};
    double hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    void grow(const Box& b) {
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], b.lo[k]);
            hi[k] = std::max(hi[k], b.hi[k]);
        }
    }
    void grow_pt(const double* p) {
        for (int k = 0; k < 3; ++k) {
            lo[k] = std::min(lo[k], p[k]);
            hi[k] = std::max(hi[k], p[k]);
        }
    }
    double half_area() const {
        double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
        if (!(dx >= 0) || !(dy >= 0) || !(dz >= 0)) return 0.0;
        return dx * dy + dy * dz + dz * dx;
    }
};

struct BNode {
    Box box;
    int32_t left = -1, right = -1;  // build-node children (-1: leaf)
    int64_t start = 0, count = 0;
};

constexpr int kBins = 32;
constexpr double kTraverseCost = 1.0;
constexpr double kIntersectCost = 2.0;   // f64 Moeller-Trumbore vs an f32 box pair
constexpr int kForceMedianDepth = 40;

struct Builder {
    const std::vector<Box>& tb;
    const std::vector<double>& cen;  // (n,3)
    std::vector<int64_t>& idx;
    std::vector<BNode> nodes;
    int max_depth = 0;
    int max_leaf = 0;

    Builder(const std::vector<Box>& b, const std::vector<double>& c, std::vector<int64_t>& i)
        : tb(b), cen(c), idx(i) {}

    int32_t make_leaf(const Box& box, int64_t s, int64_t n) {
        BNode nd;
        nd.box = box;
        nd.start = s;
        nd.count = n;
        nodes.push_back(nd);
        max_leaf = std::max<int>(max_leaf, (int)n);
        return (int32_t)nodes.size() - 1;
    }

    int32_t build(int64_t s, int64_t e, int depth) {
        max_depth = std::max(max_depth, depth);
        Box box, cbox;
        for (int64_t i = s; i < e; ++i) {
            box.grow(tb[idx[i]]);
            cbox.grow_pt(&cen[3 * idx[i]]);
        }
        int64_t n = e - s;
        if (n == 1) return make_leaf(box, s, n);
        int64_t mid = -1;
        bool split_found = false;
        if (depth < kForceMedianDepth) {
            double best = INFINITY;
            int best_axis = -1, best_bin = -1;
            double parent = box.half_area();
            for (int ax = 0; ax < 3; ++ax) {
                double ext = cbox.hi[ax] - cbox.lo[ax];
                if (!(ext > 0.0)) continue;
                Box bb[kBins];
                int64_t bc[kBins] = {0};
                double scale = kBins / ext;
                for (int64_t i = s; i < e; ++i) {
                    int b = (int)((cen[3 * idx[i] + ax] - cbox.lo[ax]) * scale);
                    b = std::min(std::max(b, 0), kBins - 1);
                    bb[b].grow(tb[idx[i]]);
                    bc[b]++;
                }
                Box rb[kBins];
                int64_t rc[kBins];
                Box acc;
                int64_t cnt = 0;
                for (int b = kBins - 1; b >= 0; --b) {
                    acc.grow(bb[b]);
                    cnt += bc[b];
                    rb[b] = acc;
                    rc[b] = cnt;
                }
                acc = Box();
                cnt = 0;
                for (int b = 0; b < kBins - 1; ++b) {
                    acc.grow(bb[b]);
                    cnt += bc[b];
                    if (cnt == 0 || rc[b + 1] == 0) continue;
                    double cost = kTraverseCost + kIntersectCost *
                        (acc.half_area() * cnt + rb[b + 1].half_area() * rc[b + 1]) /
                        std::max(parent, 1e-300);
                    if (cost < best) { best = cost; best_axis = ax; best_bin = b; }
                }
            }
            double leaf_cost = kIntersectCost * (double)n;
            if (n <= kMaxLeaf && (best_axis < 0 || leaf_cost <= best)) return make_leaf(box, s, n);
            if (best_axis >= 0) {
                double scale = kBins / (cbox.hi[best_axis] - cbox.lo[best_axis]);
                auto it = std::partition(idx.begin() + s, idx.begin() + e, [&](int64_t t) {
                    int b = (int)((cen[3 * t + best_axis] - cbox.lo[best_axis]) * scale);
                    b = std::min(std::max(b, 0), kBins - 1);
                    return b <= best_bin;
                });
                mid = it - idx.begin();
                split_found = mid > s && mid < e;
            }
        } else if (n <= kMaxLeaf) {
            return make_leaf(box, s, n);
        }
        if (!split_found) {
            // object median along the widest centroid axis (also the deep-tree
            // fallback, which bounds the depth by log2(n) more levels)
            int ax = 0;
            for (int k = 1; k < 3; ++k)
                if (cbox.hi[k] - cbox.lo[k] > cbox.hi[ax] - cbox.lo[ax]) ax = k;
            mid = s + n / 2;
            std::nth_element(idx.begin() + s, idx.begin() + mid, idx.begin() + e,
                             [&](int64_t a, int64_t b) {
                                 double ca = cen[3 * a + ax], cb = cen[3 * b + ax];
                                 return ca < cb || (ca == cb && a < b);
                             });
        }
        BNode nd;
        nd.box = box;
        nodes.push_back(nd);
        int32_t me = (int32_t)nodes.size() - 1;
        int32_t l = build(s, mid, depth + 1);
        int32_t r = build(mid, e, depth + 1);
        nodes[me].left = l;
        nodes[me].right = r;
        return me;
    }
};

float round_down(double x) {
    float f = (float)x;
    if ((double)f > x) f = std::nextafter(f, -INFINITY);
    return f;
}
float round_up(double x) {
    float f = (float)x;
    if ((double)f < x) f = std::nextafter(f, INFINITY);
    return f;
}

}  // namespace

void build_bvh(const double* v0, const double* e1, const double* e2, int64_t n, HostBvh& out) {
    if (n <= 0) throw std::runtime_error("build_bvh: empty scene");
    if (n >= (int64_t(1) << 28)) throw std::runtime_error("build_bvh: too many triangles (>= 2^28)");
    std::vector<Box> tb(n);
    std::vector<double> cen(3 * n);
    double scale = 0.0;
    for (int64_t t = 0; t < n; ++t) {
        Box b;
        double p[3];
        for (int k = 0; k < 3; ++k) p[k] = v0[3 * t + k];
        b.grow_pt(p);
        for (int k = 0; k < 3; ++k) p[k] = v0[3 * t + k] + e1[3 * t + k];
        b.grow_pt(p);
        for (int k = 0; k < 3; ++k) p[k] = v0[3 * t + k] + e2[3 * t + k];
        b.grow_pt(p);
        tb[t] = b;
        for (int k = 0; k < 3; ++k) {
            cen[3 * t + k] = 0.5 * (b.lo[k] + b.hi[k]);
            scale = std::max(scale, std::max(std::fabs(b.lo[k]), std::fabs(b.hi[k])));
        }
    }
    // Absolute padding: covers f32 rounding of ray origins up to 100x the
    // scene scale and the f64 test's barycentric slack (1e-10).
    const double pad = 1e-5 * std::max(scale, 1.0);
    std::vector<int64_t> idx(n);
    for (int64_t i = 0; i < n; ++i) idx[i] = i;
    Builder B(tb, cen, idx);
    B.nodes.reserve(2 * n);
    int32_t root = B.build(0, n, 0);

    // Convert to two-child device nodes in depth-first order.
    out.nodes.clear();
    out.order = idx;
    out.max_depth = B.max_depth;
    out.max_leaf = B.max_leaf;
    auto enc_leaf = [&](const BNode& nd) -> int32_t {
        return ~(int32_t)((nd.start << 3) | (nd.count - 1));
    };
    auto put_box = [&](GpuNode& g, int slot, const Box& b) {
        float lo[3], hi[3];
        for (int k = 0; k < 3; ++k) {
            lo[k] = round_down(b.lo[k] - pad);
            hi[k] = round_up(b.hi[k] + pad);
        }
        float* xy = slot == 0 ? g.a : g.b;
        xy[0] = lo[0]; xy[1] = hi[0]; xy[2] = lo[1]; xy[3] = hi[1];
        g.c[2 * slot + 0] = lo[2];
        g.c[2 * slot + 1] = hi[2];
    };
    if (B.nodes[root].left < 0) {
        // single-leaf scene: root with the leaf and an empty (never hit) child
        GpuNode g;
        std::memset(&g, 0, sizeof g);
        // both slots reference the same leaf: an "empty" f32 box is not
        // reliably rejected by the slab test, a duplicate leaf is harmless
        put_box(g, 0, B.nodes[root].box);
        put_box(g, 1, B.nodes[root].box);
        g.d[0] = enc_leaf(B.nodes[root]);
        g.d[1] = enc_leaf(B.nodes[root]);
        out.nodes.push_back(g);
        return;
    }
    // iterative DFS: each inner build node gets the next device slot
    std::vector<std::pair<int32_t, int32_t>> stack;  // (build node, device slot)
    out.nodes.push_back(GpuNode());
    stack.push_back({root, 0});
    while (!stack.empty()) {
        auto [bn, slot] = stack.back();
        stack.pop_back();
        const BNode& nd = B.nodes[bn];
        GpuNode g;
        std::memset(&g, 0, sizeof g);
        int32_t kids[2] = {nd.left, nd.right};
        for (int c = 0; c < 2; ++c) {
            const BNode& ch = B.nodes[kids[c]];
            put_box(g, c, ch.box);
            if (ch.left < 0) {
                g.d[c] = enc_leaf(ch);
            } else {
                int32_t s2 = (int32_t)out.nodes.size();
                out.nodes.push_back(GpuNode());
                g.d[c] = s2;
                stack.push_back({kids[c], s2});
            }
        }
        out.nodes[slot] = g;
    }
}

}  // namespace ef
