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
    int64_t start = 0, count = 0;   // leaf: range of the reference list
};

// A triangle reference: with spatial splits one triangle may be referenced
// by several leaves, each with the box of the part of it in that leaf.
struct Ref {
    int64_t id;
    Box box;
    double c(int ax) const { return 0.5 * (box.lo[ax] + box.hi[ax]); }
};

constexpr int kBins = 32;
constexpr double kTraverseCost = 1.0;
// f64 Moeller-Trumbore vs an f32 box test; EF_BVH_CI / EF_BVH_MAXLEAF /
// EF_BVH_SPLITS override (tuning experiments only)
double intersect_cost() {
    const char* e = std::getenv("EF_BVH_CI");
    return e ? std::atof(e) : 2.0;
}
// Leaves of at most this many triangles are never split (tuning:
// EF_BVH_MINLEAF; 1 = pure SAH decision).
int min_leaf() {
    const char* e = std::getenv("EF_BVH_MINLEAF");
    const int v = e ? std::atoi(e) : 1;
    return v < 1 ? 1 : (v > 8 ? 8 : v);
}
int max_leaf() {
    const char* e = std::getenv("EF_BVH_MAXLEAF");
    const int v = e ? std::atoi(e) : kMaxLeaf;
    return v < 1 ? 1 : (v > 8 ? 8 : v);
}
// Reference budget for spatial splits, as a fraction of the triangle count
// (0 disables them: a plain binned-SAH object-split tree).  Measured
// (profiles/r01_split_sweep.txt): -11% per segment on the longest C2 path,
// -7% on the C3 frame, +7-10% on the C5 frame (964k triangles whose facades
// are already finely subdivided), so large scenes build without them.
constexpr int64_t kSplitMaxTris = int64_t(1) << 19;
double split_budget(int64_t n) {
    const char* e = std::getenv("EF_BVH_SPLITS");
    if (e) return std::atof(e);
    return n <= kSplitMaxTris ? 0.5 : 0.0;
}
constexpr int kForceMedianDepth = 32;
// Spatial splits are tried where the best object split's children overlap by
// more than this fraction of the root's surface (Stich et al. 2009);
// EF_BVH_SPLIT_ALPHA overrides (tuning).
double split_alpha() {
    const char* e = std::getenv("EF_BVH_SPLIT_ALPHA");
    return e ? std::atof(e) : 1e-3;
}

struct Builder {
    const double *v0, *e1, *e2;
    std::vector<BNode> nodes;
    std::vector<int64_t> order;      // leaf-ordered triangle ids (with repeats)
    int max_depth = 0;
    int max_leaf = 0;
    double root_area = 0.0;
    int64_t budget = 0;              // spatial-split duplications left
    const double kIntersectCost = intersect_cost();
    const int kLeafMax = ef::max_leaf();
    const int kLeafMin = std::min(ef::min_leaf(), kLeafMax);
    const double kSplitAlpha = split_alpha();

    Builder(const double* a, const double* b, const double* c) : v0(a), e1(b), e2(c) {}

    int32_t make_leaf(const Box& box, const std::vector<Ref>& refs) {
        BNode nd;
        nd.box = box;
        nd.start = (int64_t)order.size();
        nd.count = (int64_t)refs.size();
        for (const Ref& r : refs) order.push_back(r.id);
        nodes.push_back(nd);
        max_leaf = std::max<int>(max_leaf, (int)refs.size());
        return (int32_t)nodes.size() - 1;
    }

    // Bounds of triangle `id` clipped to the slab lo <= x_ax <= hi, within `in`.
    Box clip(int64_t id, int ax, double lo, double hi, const Box& in) const {
        double p[3][3];
        for (int k = 0; k < 3; ++k) {
            p[0][k] = v0[3 * id + k];
            p[1][k] = v0[3 * id + k] + e1[3 * id + k];
            p[2][k] = v0[3 * id + k] + e2[3 * id + k];
        }
        Box out;
        for (int i = 0; i < 3; ++i) {
            const double* a = p[i];
            const double* b = p[(i + 1) % 3];
            if (a[ax] >= lo && a[ax] <= hi) out.grow_pt(a);
            for (double pl : {lo, hi}) {
                if ((a[ax] < pl && b[ax] > pl) || (a[ax] > pl && b[ax] < pl)) {
                    const double t = (pl - a[ax]) / (b[ax] - a[ax]);
                    double q[3];
                    for (int k = 0; k < 3; ++k) q[k] = a[k] + (b[k] - a[k]) * t;
                    q[ax] = pl;
                    out.grow_pt(q);
                }
            }
        }
        for (int k = 0; k < 3; ++k) {
            out.lo[k] = std::max(out.lo[k], in.lo[k]);
            out.hi[k] = std::min(out.hi[k], in.hi[k]);
        }
        return out;
    }

    static bool empty(const Box& b) { return !(b.lo[0] <= b.hi[0] && b.lo[1] <= b.hi[1] && b.lo[2] <= b.hi[2]); }

    int32_t build(std::vector<Ref>& refs, int depth) {
        max_depth = std::max(max_depth, depth);
        Box box, cbox;
        for (const Ref& r : refs) {
            box.grow(r.box);
            double c[3] = {r.c(0), r.c(1), r.c(2)};
            cbox.grow_pt(c);
        }
        if (depth == 0) root_area = box.half_area();
        const int64_t n = (int64_t)refs.size();
        if (n <= kLeafMin) return make_leaf(box, refs);
        const double parent = std::max(box.half_area(), 1e-300);
        std::vector<Ref> L, R;
        bool split_found = false;
        if (depth < kForceMedianDepth) {
            // ---- object split: binned SAH over reference centroids, 3 axes
            double best = INFINITY;
            int best_axis = -1, best_bin = -1;
            Box best_l, best_r;
            for (int ax = 0; ax < 3; ++ax) {
                const double ext = cbox.hi[ax] - cbox.lo[ax];
                if (!(ext > 0.0)) continue;
                Box bb[kBins];
                int64_t bc[kBins] = {0};
                const double scale = kBins / ext;
                for (const Ref& r : refs) {
                    int b = (int)((r.c(ax) - cbox.lo[ax]) * scale);
                    b = std::min(std::max(b, 0), kBins - 1);
                    bb[b].grow(r.box);
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
                    const double cost = kTraverseCost + kIntersectCost *
                        (acc.half_area() * cnt + rb[b + 1].half_area() * rc[b + 1]) / parent;
                    if (cost < best) {
                        best = cost; best_axis = ax; best_bin = b;
                        best_l = acc; best_r = rb[b + 1];
                    }
                }
            }
            const double leaf_cost = kIntersectCost * (double)n;
            if (n <= kLeafMax && (best_axis < 0 || leaf_cost <= best)) return make_leaf(box, refs);

            // ---- spatial split where the object split's children overlap
            double sbest = INFINITY;
            int s_axis = -1;
            double s_pos = 0.0;
            if (budget > 0 && best_axis >= 0) {
                Box ov;
                for (int k = 0; k < 3; ++k) {
                    ov.lo[k] = std::max(best_l.lo[k], best_r.lo[k]);
                    ov.hi[k] = std::min(best_l.hi[k], best_r.hi[k]);
                }
                if (!empty(ov) && ov.half_area() > kSplitAlpha * root_area) {
                    for (int ax = 0; ax < 3; ++ax) {
                        const double ext = box.hi[ax] - box.lo[ax];
                        if (!(ext > 0.0)) continue;
                        const double w = ext / kBins;
                        Box bb[kBins];
                        int64_t enter[kBins] = {0}, leave[kBins] = {0};
                        for (const Ref& r : refs) {
                            int b0 = (int)((r.box.lo[ax] - box.lo[ax]) / w);
                            int b1 = (int)((r.box.hi[ax] - box.lo[ax]) / w);
                            b0 = std::min(std::max(b0, 0), kBins - 1);
                            b1 = std::min(std::max(b1, b0), kBins - 1);
                            if (b0 == b1) {
                                bb[b0].grow(r.box);
                            } else {
                                for (int b = b0; b <= b1; ++b) {
                                    const double lo = box.lo[ax] + w * b;
                                    const double hi = b == kBins - 1 ? box.hi[ax] : box.lo[ax] + w * (b + 1);
                                    Box cb = clip(r.id, ax, lo, hi, r.box);
                                    if (!empty(cb)) bb[b].grow(cb);
                                }
                            }
                            enter[b0]++;
                            leave[b1]++;
                        }
                        Box rb[kBins];
                        int64_t rc[kBins];
                        Box acc;
                        int64_t cnt = 0;
                        for (int b = kBins - 1; b >= 0; --b) {
                            acc.grow(bb[b]);
                            cnt += leave[b];
                            rb[b] = acc;
                            rc[b] = cnt;
                        }
                        acc = Box();
                        cnt = 0;
                        for (int b = 0; b < kBins - 1; ++b) {
                            acc.grow(bb[b]);
                            cnt += enter[b];
                            if (cnt == 0 || rc[b + 1] == 0) continue;
                            const double cost = kTraverseCost + kIntersectCost *
                                (acc.half_area() * cnt + rb[b + 1].half_area() * rc[b + 1]) / parent;
                            if (cost < sbest) {
                                sbest = cost; s_axis = ax; s_pos = box.lo[ax] + w * (b + 1);
                            }
                        }
                    }
                }
            }
            if (s_axis >= 0 && sbest < best) {
                for (const Ref& r : refs) {
                    if (r.box.hi[s_axis] <= s_pos) {
                        L.push_back(r);
                    } else if (r.box.lo[s_axis] >= s_pos) {
                        R.push_back(r);
                    } else {
                        Box lb = clip(r.id, s_axis, -INFINITY, s_pos, r.box);
                        Box rb = clip(r.id, s_axis, s_pos, INFINITY, r.box);
                        if (!empty(lb)) L.push_back({r.id, lb});
                        if (!empty(rb)) R.push_back({r.id, rb});
                        if (!empty(lb) && !empty(rb)) --budget;
                    }
                }
                // must separate something (depth >= kForceMedianDepth ends
                // any chain of splits that keeps every reference on one side)
                split_found = !L.empty() && !R.empty() &&
                              !((int64_t)L.size() == n && (int64_t)R.size() == n);
                if (!split_found) { L.clear(); R.clear(); }
            }
            if (!split_found && best_axis >= 0) {
                const double scale = kBins / (cbox.hi[best_axis] - cbox.lo[best_axis]);
                for (const Ref& r : refs) {
                    int b = (int)((r.c(best_axis) - cbox.lo[best_axis]) * scale);
                    b = std::min(std::max(b, 0), kBins - 1);
                    (b <= best_bin ? L : R).push_back(r);
                }
                split_found = !L.empty() && !R.empty();
                if (!split_found) { L.clear(); R.clear(); }
            }
        } else if (n <= kLeafMax) {
            return make_leaf(box, refs);
        }
        if (!split_found) {
            // object median along the widest centroid axis (also the deep-tree
            // fallback, which bounds the depth by log2(n) more levels)
            int ax = 0;
            for (int k = 1; k < 3; ++k)
                if (cbox.hi[k] - cbox.lo[k] > cbox.hi[ax] - cbox.lo[ax]) ax = k;
            const int64_t mid = n / 2;
            std::nth_element(refs.begin(), refs.begin() + mid, refs.end(), [&](const Ref& a, const Ref& b) {
                const double ca = a.c(ax), cb = b.c(ax);
                return ca < cb || (ca == cb && a.id < b.id);
            });
            L.assign(refs.begin(), refs.begin() + mid);
            R.assign(refs.begin() + mid, refs.end());
        }
        std::vector<Ref>().swap(refs);   // release before recursing
        BNode nd;
        nd.box = box;
        nodes.push_back(nd);
        const int32_t me = (int32_t)nodes.size() - 1;
        const int32_t l = build(L, depth + 1);
        const int32_t r = build(R, depth + 1);
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
    std::vector<Ref> refs(n);
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
        refs[t] = {t, b};
        for (int k = 0; k < 3; ++k)
            scale = std::max(scale, std::max(std::fabs(b.lo[k]), std::fabs(b.hi[k])));
    }
    // Absolute padding: covers f32 rounding of ray origins up to 100x the
    // scene scale, the f64 test's barycentric slack (1e-10) and the rounding
    // of clipped reference boxes.
    const double pad = 1e-5 * std::max(scale, 1.0);
    Builder B(v0, e1, e2);
    B.budget = (int64_t)(split_budget(n) * (double)n);
    B.nodes.reserve(2 * n);
    B.order.reserve(n);
    int32_t root = B.build(refs, 0);
    if (B.order.size() >= (size_t(1) << 28)) throw std::runtime_error("build_bvh: too many references");

    if (out.keep_binary) {
        out.binary.resize(B.nodes.size());
        for (size_t i = 0; i < B.nodes.size(); ++i) {
            HostBinNode& h = out.binary[i];
            for (int k = 0; k < 3; ++k) {
                h.lo[k] = B.nodes[i].box.lo[k];
                h.hi[k] = B.nodes[i].box.hi[k];
            }
            h.left = B.nodes[i].left;
            h.right = B.nodes[i].right;
            h.start = B.nodes[i].start;
            h.count = B.nodes[i].count;
        }
        out.binary_root = root;
    }

    // Collapse the binary tree into 4-wide device nodes (repeatedly open the
    // largest inner child until four slots are used), depth-first numbering.
    out.nodes.clear();
    out.order = std::move(B.order);
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
            // lo = hi = +inf: misses in the slab test (ef_device.cuh slab_key)
            g.lox[c] = g.loy[c] = g.loz[c] = INFINITY;
            g.hix[c] = g.hiy[c] = g.hiz[c] = INFINITY;
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
