// Device BVH builder (kernel K2 on the GPU).
//
// The host builder (bvh_build.cpp) is a binned-SAH tree like the reference's
// (bvh.py:51-128); it costs ~1.5 s for the 964k-triangle C5 city, which is
// too slow for scenes whose geometry changes every frame beyond what a refit
// keeps tight.  This builder makes the same 128-byte four-child nodes on the
// device in a few milliseconds:
//
//   1. prim_box_kernel   f64 box of (v0, v0+e1, v0+e2) per triangle (the same
//                        expressions as the refit), centroid bounds, scale
//   2. morton_kernel     63-bit Morton code of the f32 centroid (21 bits/axis)
//   3. radix sort        (code, triangle) pairs, CUB's device radix sort
//   4. karras_kernel     one binary inner node per thread from the sorted
//                        codes (Karras 2012: longest-common-prefix split, ties
//                        broken by position so equal codes still split)
//   5. bottom_up_kernel  f64 inner boxes, leaf-to-root with an arrival flag
//   6. collapse_kernel   one launch per output level: each four-child node
//                        opens its largest-area binary child until 4 slots;
//                        subtrees of <= kMaxLeaf triangles become leaves
//                        (contiguous in code order); nodes are numbered
//                        level by level, which is also the refit order.
//   7. gather_kernel     f64 triangle payload in leaf (code) order
//
// Hit results do not depend on the tree (lowest id wins on exact-t ties,
// DESIGN.md 3.2), so every parity test of the host-built tree applies; only
// the node-visit counts change (the LBVH is looser than SAH).
#include <cub/device/device_radix_sort.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "ef_internal.h"

using namespace ef;

namespace {

constexpr int kThreads = 256;
constexpr int kLevelChunk = 4;          // levels launched between host checks
constexpr int kMaxLevels = (kStackSize - 1) / 3;   // max_stack = 3 * depth + 1

__device__ __forceinline__ int f2o(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float o2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

__device__ __forceinline__ uint64_t spread21(uint32_t v) {
    uint64_t x = v & 0x1fffffu;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}

struct BuildBounds {
    int cmin[3];                 // ordered-int f32 centroid bounds
    int cmax[3];
    unsigned long long scale;    // bits of max |coordinate| (non-negative f64)
    int max_leaf;
};

__global__ void prim_box_kernel(const double* __restrict__ v0, const double* __restrict__ e1,
                                const double* __restrict__ e2, int64_t stride, int64_t n,
                                double* __restrict__ pbox, BuildBounds* bb) {
    float cmin[3] = {INFINITY, INFINITY, INFINITY}, cmax[3] = {-INFINITY, -INFINITY, -INFINITY};
    double sc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const double a = v0[i * stride + k];
            const double b = a + e1[i * stride + k], d = a + e2[i * stride + k];
            const double lo = fmin(a, fmin(b, d)), hi = fmax(a, fmax(b, d));
            pbox[6 * i + k] = lo;
            pbox[6 * i + 3 + k] = hi;
            const float c = (float)(0.5 * (lo + hi));
            cmin[k] = fminf(cmin[k], c);
            cmax[k] = fmaxf(cmax[k], c);
            sc = fmax(sc, fmax(fabs(lo), fabs(hi)));
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            cmin[k] = fminf(cmin[k], __shfl_xor_sync(0xffffffffu, cmin[k], off));
            cmax[k] = fmaxf(cmax[k], __shfl_xor_sync(0xffffffffu, cmax[k], off));
        }
        sc = fmax(sc, __shfl_xor_sync(0xffffffffu, sc, off));
    }
    if ((threadIdx.x & 31) == 0) {
        for (int k = 0; k < 3; ++k) {
            atomicMin(&bb->cmin[k], f2o(cmin[k]));
            atomicMax(&bb->cmax[k], f2o(cmax[k]));
        }
        atomicMax(&bb->scale, (unsigned long long)__double_as_longlong(sc));
    }
}

__global__ void morton_kernel(const double* __restrict__ pbox, int64_t n, const BuildBounds* bb,
                              uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    // cubic cells (one scale for all axes, the largest centroid extent):
    // flat scenes such as cities then split along their long axes first
    float lo[3], inv[3], ext = 0.0f;
    for (int k = 0; k < 3; ++k) {
        lo[k] = o2f(bb->cmin[k]);
        ext = fmaxf(ext, o2f(bb->cmax[k]) - lo[k]);
    }
    for (int k = 0; k < 3; ++k) inv[k] = ext > 0.0f ? 2097151.0f / ext : 0.0f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key = 0;
        float diag2 = 0.0f;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float c = (float)(0.5 * (pbox[6 * i + k] + pbox[6 * i + 3 + k]));
            const float q = fminf(fmaxf((c - lo[k]) * inv[k], 0.0f), 2097151.0f);
            key |= spread21((uint32_t)q) << (2 - k);
            const float e = (float)(pbox[6 * i + 3 + k] - pbox[6 * i + k]);
            diag2 += e * e;
        }
        // triangles spanning a quarter of the scene (ground planes, long
        // walls) sort after all others: the hierarchy splits them off at the
        // root instead of inflating the boxes of small-triangle subtrees
        key >>= 1;   // 62 Morton bits under the flag: a 63-bit sort
        if (diag2 > 0.0625f * ext * ext) key |= 1ull << 62;
        keys[i] = key;
        vals[i] = (uint32_t)i;
    }
}

// Length of the common prefix of sorted keys i and j (position-augmented so
// duplicates still order), -1 outside [0, n).
__device__ __forceinline__ int delta(const uint64_t* keys, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    const uint64_t a = keys[i], b = keys[j];
    return a != b ? __clzll((long long)(a ^ b)) : 64 + __clz(i ^ j);
}

// Binary inner node i covers sorted positions [first, last]; child refs are
// inner indices (>= 0) or ~position for single-triangle leaves.
__global__ void karras_kernel(const uint64_t* __restrict__ keys, int n, int* __restrict__ left,
                              int* __restrict__ right, int* __restrict__ first,
                              int* __restrict__ last, int* __restrict__ parent_in,
                              int* __restrict__ parent_leaf) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n - 1; i += gridDim.x * blockDim.x) {
        const int d = delta(keys, n, i, i + 1) - delta(keys, n, i, i - 1) > 0 ? 1 : -1;
        const int dmin = delta(keys, n, i, i - d);
        int lmax = 2;
        while (delta(keys, n, i, i + lmax * d) > dmin) lmax <<= 1;
        int l = 0;
        for (int t = lmax >> 1; t >= 1; t >>= 1)
            if (delta(keys, n, i, i + (l + t) * d) > dmin) l += t;
        const int j = i + l * d;
        const int dnode = delta(keys, n, i, j);
        int s = 0, t = l;
        do {
            t = (t + 1) >> 1;
            if (delta(keys, n, i, i + (s + t) * d) > dnode) s += t;
        } while (t > 1);
        const int g = i + s * d + min(d, 0);
        const int lo = min(i, j), hi = max(i, j);
        const int lc = lo == g ? ~g : g;
        const int rc = hi == g + 1 ? ~(g + 1) : g + 1;
        left[i] = lc;
        right[i] = rc;
        first[i] = lo;
        last[i] = hi;
        if (lc < 0) parent_leaf[~lc] = i; else parent_in[lc] = i;
        if (rc < 0) parent_leaf[~rc] = i; else parent_in[rc] = i;
        if (i == 0) parent_in[0] = -1;
    }
}

__device__ __forceinline__ const double* ref_box(int r, const double* pbox, const double* ibox,
                                                 const uint32_t* sorted) {
    return r < 0 ? pbox + 6 * (int64_t)sorted[~r] : ibox + 6 * (int64_t)r;
}

__device__ __forceinline__ double half_area(const double* b) {
    const double dx = b[3] - b[0], dy = b[4] - b[1], dz = b[5] - b[2];
    return dx * dy + dy * dz + dz * dx;
}

// SAH costs of the host builder (bvh_build.cpp): traversal 1, triangle test 2.
constexpr double kCostNode = 1.0, kCostTri = 2.0;

// Inner boxes leaf-to-root; the second thread to reach a node finishes it.
// Each node also gets its SAH cost and whether it is cheaper kept as one
// leaf (<= max_leaf triangles) than split (Karras 2013's leaf collapse).
__global__ void bottom_up_kernel(int n, const int* __restrict__ left, const int* __restrict__ right,
                                 const int* __restrict__ first, const int* __restrict__ last,
                                 const int* __restrict__ parent_in,
                                 const int* __restrict__ parent_leaf, const uint32_t* sorted,
                                 const double* pbox, double* ibox, double* cost, uint8_t* as_leaf,
                                 int* flag, int max_leaf) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        int p = parent_leaf[j];
        while (p >= 0) {
            __threadfence();
            if (atomicAdd(&flag[p], 1) == 0) break;   // sibling subtree not done yet
            const int lc = left[p], rc = right[p];
            const double* a = ref_box(lc, pbox, ibox, sorted);
            const double* b = ref_box(rc, pbox, ibox, sorted);
            double o[6];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                o[k] = fmin(__ldcg(a + k), __ldcg(b + k));
                o[3 + k] = fmax(__ldcg(a + 3 + k), __ldcg(b + 3 + k));
            }
            double ca, cb;
            if (lc < 0) { double t[6]; for (int k = 0; k < 6; ++k) t[k] = a[k]; ca = kCostTri * half_area(t); }
            else ca = __ldcg(cost + lc);
            if (rc < 0) { double t[6]; for (int k = 0; k < 6; ++k) t[k] = b[k]; cb = kCostTri * half_area(t); }
            else cb = __ldcg(cost + rc);
            const double area = half_area(o);
            const double split = kCostNode * area + ca + cb;
            const int cnt = last[p] - first[p] + 1;
            const double leaf = cnt <= max_leaf ? kCostTri * cnt * area : INFINITY;
#pragma unroll
            for (int k = 0; k < 6; ++k) ibox[6 * (int64_t)p + k] = o[k];
            cost[p] = fmin(leaf, split);
            as_leaf[p] = leaf <= split;
            p = parent_in[p];
        }
    }
}

__device__ __forceinline__ int ref_count(int r, const int* first, const int* last) {
    return r < 0 ? 1 : last[r] - first[r] + 1;
}

__device__ __forceinline__ bool ref_is_leaf(int r, const uint8_t* as_leaf) {
    return r < 0 || as_leaf[r];
}

// Level l of the four-child tree: nodes [lvl[l], lvl[l] + cnt[l]) with binary
// sources src[]; inner children are appended to level l + 1.
__global__ void collapse_kernel(int l, int* lvl, int* cnt, int* src, GpuNode* __restrict__ nodes,
                                const int* __restrict__ left, const int* __restrict__ right,
                                const int* __restrict__ first, const int* __restrict__ last,
                                const uint32_t* __restrict__ sorted, const double* __restrict__ pbox,
                                const double* __restrict__ ibox, const uint8_t* __restrict__ as_leaf,
                                BuildBounds* bb) {
    const int begin = lvl[l], end = begin + cnt[l];
    if (blockIdx.x == 0 && threadIdx.x == 0) lvl[l + 1] = end;
    const double pad = 1e-5 * fmax(__longlong_as_double((long long)bb->scale), 1.0);
    for (int item = begin + blockIdx.x * blockDim.x + threadIdx.x; item < end;
         item += gridDim.x * blockDim.x) {
        int cand[4] = {src[item], 0, 0, 0};
        int nc = 1;
        while (nc < 4) {
            int best = -1;
            double best_a = -1.0;
            for (int k = 0; k < nc; ++k) {
                const int r = cand[k];
                if (ref_is_leaf(r, as_leaf)) continue;
                const double a = half_area(ibox + 6 * (int64_t)r);
                if (a > best_a) { best_a = a; best = k; }
            }
            if (best < 0) break;
            const int r = cand[best];
            cand[best] = left[r];
            cand[nc++] = right[r];
        }
        GpuNode g;
        int leaf_max = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            g.pad[k] = 0;
            if (k >= nc) {
                g.lox[k] = g.loy[k] = g.loz[k] = INFINITY;
                g.hix[k] = g.hiy[k] = g.hiz[k] = INFINITY;
                g.child[k] = kEmptyChild;
                continue;
            }
            const int r = cand[k];
            const double* b = ref_box(r, pbox, ibox, sorted);
            g.lox[k] = __double2float_rd(b[0] - pad); g.hix[k] = __double2float_ru(b[3] + pad);
            g.loy[k] = __double2float_rd(b[1] - pad); g.hiy[k] = __double2float_ru(b[4] + pad);
            g.loz[k] = __double2float_rd(b[2] - pad); g.hiz[k] = __double2float_ru(b[5] + pad);
            const int c = ref_count(r, first, last);
            if (ref_is_leaf(r, as_leaf)) {
                const int f = r < 0 ? ~r : first[r];
                g.child[k] = ~(int32_t)(((uint32_t)f << 3) | (uint32_t)(c - 1));
                leaf_max = max(leaf_max, c);
            } else {
                const int idx = end + atomicAdd(&cnt[l + 1], 1);
                src[idx] = r;
                g.child[k] = idx;
            }
        }
        nodes[item] = g;
        if (leaf_max) atomicMax(&bb->max_leaf, leaf_max);
    }
}

__global__ void gather_kernel(const double* __restrict__ v0, const double* __restrict__ e1,
                              const double* __restrict__ e2, int64_t stride, int64_t n,
                              const uint32_t* __restrict__ sorted, GpuTri* __restrict__ tris,
                              int64_t* __restrict__ leaf_order) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t id = sorted[i];
        GpuTri t;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            t.v[k] = v0[id * stride + k];
            t.v[3 + k] = e1[id * stride + k];
            t.v[6 + k] = e2[id * stride + k];
        }
        t.id = id;
        tris[i] = t;
        leaf_order[i] = id;
    }
}

__global__ void iota_kernel(int32_t* out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)i;
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + kThreads - 1) / kThreads, 148 * 8)); }

template <class T>
cudaError_t alloc(T** p, size_t count, cudaStream_t st) {
    return cudaMallocAsync((void**)p, std::max<size_t>(count, 1) * sizeof(T), st);
}

}  // namespace

namespace ef {

// Builds s->nodes / tris / leaf_order / level_nodes / level_start / pad /
// n_nodes / max_depth / max_leaf from DEVICE triangle arrays whose rows are
// `stride` doubles apart.  Ends with one host synchronisation (the level
// counts size the refit schedule).  s->tris and s->leaf_order must hold
// s->n_tri entries.
int device_build_bvh(ef_scene* s, const double* v0, const double* e1, const double* e2,
                     int64_t stride, cudaStream_t st) {
    const int64_t n64 = s->n_tri;
    if (n64 <= 0) return EF_OK;
    if (n64 >= (1ll << 29)) return set_error(EF_EUNSUPPORTED, "device BVH build: more than 2^29 triangles");
    const int n = (int)n64;
    keep_pool_memory();
    const int max_leaf = kMaxLeaf;
    const int64_t cap = n64;   // each four-child node comes from a distinct binary inner node

    double *pbox = nullptr, *ibox = nullptr, *cost = nullptr;
    uint8_t* as_leaf = nullptr;
    uint64_t *keys = nullptr, *keys2 = nullptr;
    uint32_t *vals = nullptr, *vals2 = nullptr;
    int *left = nullptr, *right = nullptr, *first = nullptr, *last = nullptr, *par_in = nullptr,
        *par_leaf = nullptr, *flag = nullptr, *src = nullptr, *lvl = nullptr, *cnt = nullptr;
    BuildBounds* bb = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t e = cudaSuccess;
    auto ok = [&](cudaError_t r) { if (e == cudaSuccess) e = r; return e == cudaSuccess; };

    ok(alloc(&pbox, 6 * (size_t)n, st));
    ok(alloc(&ibox, 6 * (size_t)n, st));
    ok(alloc(&keys, n, st));
    ok(alloc(&keys2, n, st));
    ok(alloc(&vals, n, st));
    ok(alloc(&vals2, n, st));
    ok(alloc(&left, n, st));
    ok(alloc(&right, n, st));
    ok(alloc(&first, n, st));
    ok(alloc(&last, n, st));
    ok(alloc(&par_in, n, st));
    ok(alloc(&par_leaf, n, st));
    ok(alloc(&flag, n, st));
    ok(alloc(&cost, n, st));
    ok(alloc(&as_leaf, n, st));
    ok(alloc(&src, cap, st));
    ok(alloc(&lvl, kMaxLevels + 2, st));
    ok(alloc(&cnt, kMaxLevels + 2, st));
    ok(alloc(&bb, 1, st));
    cub::DoubleBuffer<uint64_t> kb(keys, keys2);
    cub::DoubleBuffer<uint32_t> vb(vals, vals2);
    if (e == cudaSuccess)
        ok(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, kb, vb, n, 0, 63, st));
    if (e == cudaSuccess) ok(cudaMallocAsync(&tmp, std::max<size_t>(tmp_bytes, 1), st));

    GpuNode* nodes = nullptr;   // scratch, level-ordered; copied out at the end
    std::vector<int> h_lvl(kMaxLevels + 2, 0), h_cnt(kMaxLevels + 2, 0);
    BuildBounds h_bb;
    int levels = 0;
    if (e == cudaSuccess) {
        BuildBounds init;
        for (int k = 0; k < 3; ++k) { init.cmin[k] = INT_MAX; init.cmax[k] = INT_MIN; }
        init.scale = 0;
        init.max_leaf = 0;
        const int root = n >= 2 ? 0 : ~0;
        ok(cudaMemcpyAsync(bb, &init, sizeof init, cudaMemcpyHostToDevice, st));
        ok(cudaMemsetAsync(lvl, 0, (kMaxLevels + 2) * sizeof(int), st));
        ok(cudaMemsetAsync(cnt, 0, (kMaxLevels + 2) * sizeof(int), st));
        ok(cudaMemsetAsync(flag, 0, (size_t)n * sizeof(int), st));
        ok(cudaMemsetAsync(as_leaf, 0, (size_t)n, st));
        const int one = 1;
        ok(cudaMemcpyAsync(cnt, &one, sizeof(int), cudaMemcpyHostToDevice, st));
        ok(cudaMemcpyAsync(src, &root, sizeof(int), cudaMemcpyHostToDevice, st));
        ok(cudaMallocAsync((void**)&nodes, (size_t)cap * sizeof(GpuNode), st));
        // the pageable copies above are synchronous with respect to the host
    }
    if (e == cudaSuccess) {
        const int g = grid_for(n);
        prim_box_kernel<<<g, kThreads, 0, st>>>(v0, e1, e2, stride, n, pbox, bb);
        morton_kernel<<<g, kThreads, 0, st>>>(pbox, n, bb, kb.Current(), vb.Current());
        count_launch(2);
        // library sort (CUB); its kernels are not counted by ef_launch_count
        ok(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, kb, vb, n, 0, 63, st));
        if (n >= 2) {
            karras_kernel<<<g, kThreads, 0, st>>>(kb.Current(), n, left, right, first, last, par_in, par_leaf);
            bottom_up_kernel<<<g, kThreads, 0, st>>>(n, left, right, first, last, par_in, par_leaf,
                                                     vb.Current(), pbox, ibox, cost, as_leaf, flag,
                                                     max_leaf);
            count_launch(2);
        }
        ok(cudaGetLastError());
        for (int l0 = 0; e == cudaSuccess && l0 < kMaxLevels; l0 += kLevelChunk) {
            const int lend = std::min(l0 + kLevelChunk, kMaxLevels);
            for (int l = l0; l < lend; ++l) {
                collapse_kernel<<<grid_for(std::min<int64_t>(cap, 148 * kThreads * 4)), kThreads, 0, st>>>(
                    l, lvl, cnt, src, nodes, left, right, first, last, vb.Current(), pbox, ibox,
                    as_leaf, bb);
                count_launch();
            }
            ok(cudaMemcpyAsync(h_cnt.data(), cnt, h_cnt.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
            ok(cudaMemcpyAsync(h_lvl.data(), lvl, h_lvl.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
            ok(cudaStreamSynchronize(st));
            if (e == cudaSuccess && h_cnt[lend] == 0) {
                while (levels < lend && h_cnt[levels] > 0) ++levels;
                break;
            }
        }
    }
    if (e == cudaSuccess) {
        ok(cudaMemcpyAsync(&h_bb, bb, sizeof h_bb, cudaMemcpyDeviceToHost, st));
        gather_kernel<<<grid_for(n), kThreads, 0, st>>>(v0, e1, e2, stride, n, vb.Current(), s->tris,
                                                         s->leaf_order);
        count_launch();
    }
    const int64_t n_nodes = levels ? (int64_t)h_lvl[levels - 1] + h_cnt[levels - 1] : 0;
    // Final arrays: reuse the scene's allocations when they are big enough
    // (per-frame rebuilds), else exact-size new ones.
    GpuNode* out_nodes = s->nodes;
    int32_t* out_levels = s->level_nodes;
    const bool new_nodes = !s->nodes || s->n_nodes_cap < n_nodes;
    const bool new_levels = !s->level_nodes || s->level_nodes_len < n_nodes;
    if (e == cudaSuccess && levels > 0) {
        if (new_nodes) ok(cudaMalloc((void**)&out_nodes, (size_t)n_nodes * sizeof(GpuNode)));
        if (new_levels) ok(cudaMalloc((void**)&out_levels, (size_t)n_nodes * sizeof(int32_t)));
        ok(cudaMemcpyAsync(out_nodes, nodes, (size_t)n_nodes * sizeof(GpuNode), cudaMemcpyDeviceToDevice, st));
        if (e == cudaSuccess) {
            iota_kernel<<<grid_for(n_nodes), kThreads, 0, st>>>(out_levels, n_nodes);
            count_launch();
        }
    }
    for (void* p : {(void*)pbox, (void*)ibox, (void*)cost, (void*)as_leaf, (void*)keys, (void*)keys2,
                    (void*)vals, (void*)vals2, (void*)left, (void*)right, (void*)first, (void*)last,
                    (void*)par_in, (void*)par_leaf, (void*)flag, (void*)src, (void*)lvl, (void*)cnt,
                    (void*)bb, tmp, (void*)nodes})
        if (p) cudaFreeAsync(p, st);
    cudaError_t es = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = es;
    if (e != cudaSuccess || levels == 0) {
        if (new_nodes && out_nodes != s->nodes) cudaFree(out_nodes);
        if (new_levels && out_levels != s->level_nodes) cudaFree(out_levels);
        if (e == cudaSuccess)
            return set_error(EF_EUNSUPPORTED, "device BVH build: tree deeper than the traversal stack");
        return check_cuda(e, "device BVH build");
    }
    if (new_nodes) {
        if (s->nodes) { s->device_bytes -= s->n_nodes_cap * (int64_t)sizeof(GpuNode); cudaFree(s->nodes); }
        s->nodes = out_nodes;
        s->n_nodes_cap = n_nodes;
        s->device_bytes += n_nodes * (int64_t)sizeof(GpuNode);
    }
    if (new_levels) {
        if (s->level_nodes) { s->device_bytes -= s->level_nodes_len * (int64_t)sizeof(int32_t); cudaFree(s->level_nodes); }
        s->level_nodes = out_levels;
        s->level_nodes_len = n_nodes;
        s->device_bytes += n_nodes * (int64_t)sizeof(int32_t);
    }
    s->n_nodes = n_nodes;
    s->n_refs = n64;
    s->max_depth = levels;
    s->max_leaf = h_bb.max_leaf;
    double scale;
    std::memcpy(&scale, &h_bb.scale, sizeof scale);
    s->pad = 1e-5 * std::max(scale, 1.0);
    s->level_start.assign(levels + 1, 0);
    for (int l = 0; l < levels; ++l) s->level_start[l + 1] = (int64_t)h_lvl[l] + h_cnt[l];
    s->level_start[0] = 0;
    return EF_OK;
}

}  // namespace ef
