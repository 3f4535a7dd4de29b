// Host-side binned-SAH BVH2 builder for the device traversal (K2).
//
// Replaces the reference's recursive Python builder (bvh.py:51-128: 16 bins
// on the widest centroid axis, leaves <= 4, median fallback).  The device
// tree is deliberately NOT the reference's tree: hit ids do not depend on the
// tree because the leaf test is the reference's exact f64 arithmetic and
// equal-t ties resolve to the lowest id.  What changes is the
// layout: boxes rounded outward and padded so the f32 slab
// test never culls a hit the f64 test would accept, SAH over all three axes
// with 32 bins, then collapsed to 4-wide nodes (128 B, child boxes as f32
// structure-of-arrays) numbered depth-first for locality.
#include <algorithm>
#include <cmath>
#include <cstdlib>
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
// f64 Moeller-Trumbore vs an f32 box test; EF_BVH_CI / EF_BVH_MAXLEAF override
// (tuning experiments only)
double intersect_cost() {
    const char* e = std::getenv("EF_BVH_CI");
    return e ? std::atof(e) : 2.0;
}
int max_leaf() {
    const char* e = std::getenv("EF_BVH_MAXLEAF");
    const int v = e ? std::atoi(e) : kMaxLeaf;
    return v < 1 ? 1 : (v > 8 ? 8 : v);
}
constexpr int kForceMedianDepth = 32;

struct Builder {
    const std::vector<Box>& tb;
    const std::vector<double>& cen;  // (n,3)
    std::vector<int64_t>& idx;
    std::vector<BNode> nodes;
    int max_depth = 0;
    int max_leaf = 0;
    const double kIntersectCost = intersect_cost();
    const int kLeafMax = ef::max_leaf();

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
            if (n <= kLeafMax && (best_axis < 0 || leaf_cost <= best)) return make_leaf(box, s, n);
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
        } else if (n <= kLeafMax) {
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

    // Collapse the binary tree into 4-wide device nodes (repeatedly open the
    // largest inner child until four slots are used), depth-first numbering.
    out.nodes.clear();
    out.order = idx;
    out.max_leaf = B.max_leaf;
    auto enc_leaf = [&](const BNode& nd) -> int32_t {
        return ~(int32_t)((nd.start << 3) | (nd.count - 1));
    };
    auto put_box = [&](GpuNode& g, int slot, const Box& b) {
        g.lox[slot] = round_down(b.lo[0] - pad);
        g.hix[slot] = round_up(b.hi[0] + pad);
        g.loy[slot] = round_down(b.lo[1] - pad);
        g.hiy[slot] = round_up(b.hi[1] + pad);
        g.loz[slot] = round_down(b.lo[2] - pad);
        g.hiz[slot] = round_up(b.hi[2] + pad);
    };
    auto empty_node = []() {
        GpuNode g;
        std::memset(&g, 0, sizeof g);
        for (int c = 0; c < 4; ++c) {
            // lo = +inf, hi = -inf: both sign-selected planes give t_near = +inf
            g.lox[c] = g.loy[c] = g.loz[c] = INFINITY;
            g.hix[c] = g.hiy[c] = g.hiz[c] = -INFINITY;
            g.child[c] = kEmptyChild;
        }
        return g;
    };
    if (B.nodes[root].left < 0) {
        GpuNode g = empty_node();
        put_box(g, 0, B.nodes[root].box);
        g.child[0] = enc_leaf(B.nodes[root]);
        out.nodes.push_back(g);
        out.max_depth = 1;
        out.max_stack = 1;
        out.pad = pad;
        out.level_nodes.assign(1, 0);
        out.level_start = {0, 1};
        return;
    }
    struct Item { int32_t bn; int32_t slot; int depth; };
    std::vector<Item> stack;
    out.nodes.push_back(empty_node());
    stack.push_back({root, 0, 1});
    int max_depth = 1;
    while (!stack.empty()) {
        Item it = stack.back();
        stack.pop_back();
        max_depth = std::max(max_depth, it.depth);
        int32_t kids[4] = {B.nodes[it.bn].left, B.nodes[it.bn].right, -1, -1};
        int nk = 2;
        while (nk < 4) {
            int best = -1;
            double best_area = -1.0;
            for (int c = 0; c < nk; ++c) {
                const BNode& ch = B.nodes[kids[c]];
                if (ch.left >= 0 && ch.box.half_area() > best_area) {
                    best_area = ch.box.half_area();
                    best = c;
                }
            }
            if (best < 0) break;
            const BNode& op = B.nodes[kids[best]];
            kids[best] = op.left;
            kids[nk++] = op.right;
        }
        GpuNode g = empty_node();
        for (int c = 0; c < nk; ++c) {
            const BNode& ch = B.nodes[kids[c]];
            put_box(g, c, ch.box);
            if (ch.left < 0) {
                g.child[c] = enc_leaf(ch);
            } else {
                int32_t s2 = (int32_t)out.nodes.size();
                out.nodes.push_back(empty_node());
                g.child[c] = s2;
                stack.push_back({kids[c], s2, it.depth + 1});
            }
        }
        out.nodes[it.slot] = g;
    }
    out.max_depth = max_depth;
    out.max_stack = 3 * max_depth + 1;   // at most three pushes per level
    out.pad = pad;
    // depth of every node (children are allocated after their parent)
    std::vector<int> depth(out.nodes.size(), 0);
    for (size_t i = 0; i < out.nodes.size(); ++i)
        for (int c = 0; c < 4; ++c) {
            const int32_t ch = out.nodes[i].child[c];
            if (ch >= 0) depth[ch] = depth[i] + 1;
        }
    std::vector<std::vector<int32_t>> lv(max_depth);
    for (size_t i = 0; i < out.nodes.size(); ++i) lv[depth[i]].push_back((int32_t)i);
    out.level_start.assign(1, 0);
    for (auto& l : lv) {
        out.level_nodes.insert(out.level_nodes.end(), l.begin(), l.end());
        out.level_start.push_back((int64_t)out.level_nodes.size());
    }
}

}  // namespace ef
