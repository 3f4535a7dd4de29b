// Scene construction: validates the reference's arrays, builds the device
// BVH (bvh_build.cpp) and uploads everything once (SceneModel.__init__,
// scene.py:149-171; SceneModel is immutable after construction).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <exception>
#include <string>
#include <vector>

#include "ef_device.cuh"
#include "ef_internal.h"

using namespace ef;

namespace {

template <class T>
cudaError_t upload(T** dst, const T* src, size_t count, int64_t& bytes) {
    if (count == 0) return cudaSuccess;
    cudaError_t e = cudaMalloc((void**)dst, count * sizeof(T));
    if (e != cudaSuccess) return e;
    bytes += (int64_t)(count * sizeof(T));
    return cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
}

void free_scene(ef_scene* s) {
    if (!s) return;
    cudaFree(s->nodes);
    cudaFree(s->tnodes_base);
    cudaFree(s->tris);
    cudaFree(s->tris_by_id);
    cudaFree(s->normals);
    cudaFree(s->mat);
    cudaFree(s->fd);
    cudaFree(s->fs);
    cudaFree(s->pdiff);
    cudaFree(s->fr);
    cudaFree(s->shade);
    cudaFree(s->tri_box);
    cudaFree(s->clu_box);
    cudaFree(s->clu_ids);
    cudaFree(s->leaf_order);
    cudaFree(s->level_nodes);
    delete s;
}

// Shading records (GpuShade) from the original-order normals and materials.
__global__ void shade_kernel(GpuShade* out, const double* normals, const int32_t* mat,
                             const double* pdiff, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        GpuShade r;
        for (int k = 0; k < 3; ++k) r.n[k] = normals[3 * i + k];
        r.m = mat[i];
        r.p = pdiff[r.m];
        for (int k = 0; k < (int)(sizeof(r.pad) / sizeof(r.pad[0])); ++k) r.pad[k] = 0;
        out[i] = r;
    }
}

// Per-triangle f32 boxes over v0, v0+e1, v0+e2 rounded outward and padded
// exactly like the BVH's leaf boxes, so the conservative slab test of a box
// never drops a triangle the exact test would accept.
__global__ void tribox_kernel(float* out, const double* tris, int64_t n, double pad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double* v = tris + 9 * i;
        float* o = out + 8 * i;
        for (int k = 0; k < 3; ++k) {
            const double a = v[k], b = v[k] + v[3 + k], d = v[k] + v[6 + k];
            o[k] = __double2float_rd(fmin(a, fmin(b, d)) - pad);
            o[3 + k] = __double2float_ru(fmax(a, fmax(b, d)) + pad);
        }
        o[6] = o[7] = 0.0f;
    }
}

// Clusters of kTailCluster consecutive leaf-order triangles (spatially
// coherent runs): the union of their padded boxes (still conservative) and
// their ids, for the tail sweep's first level.
__global__ void order_kernel(int32_t* clu_ids, const int64_t* leaf_order, int64_t n) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        clu_ids[r] = (int32_t)leaf_order[r];
}

__global__ void cluster_kernel(float* clu_box, const int32_t* clu_ids, const float* tri_box,
                               int64_t n_ids, int64_t n_clu) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_clu;
         c += (int64_t)gridDim.x * blockDim.x) {
        float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
        for (int64_t r = c * kTailCluster; r < n_ids && r < (c + 1) * kTailCluster; ++r) {
            const int64_t id = clu_ids[r];
            for (int k = 0; k < 3; ++k) {
                lo[k] = fminf(lo[k], tri_box[8 * id + k]);
                hi[k] = fmaxf(hi[k], tri_box[8 * id + 3 + k]);
            }
        }
        float* o = clu_box + 8 * c;
        for (int k = 0; k < 3; ++k) {
            o[k] = lo[k];
            o[3 + k] = hi[k];
        }
        o[6] = o[7] = 0.0f;
    }
}

#if !EF_QNODE
// One child box of one axis in the traversal form: centre c (rounded to
// nearest) and half extent e (rounded up) with [c - e, c + e] enclosing
// [lo, hi] exactly: hi - c and c - lo are exact in f64 (f32 operands).  An
// empty slot (lo = hi = +inf) becomes c = +inf, e = 0, which every ray
// misses: an axis of positive direction gives near = +inf, and a ray with
// every direction component negative gets far = -inf on every axis.
__device__ __forceinline__ void encode_slab(float lo, float hi, float& c, float& e) {
#if EF_SLAB_CE
    if (isinf(lo) || isinf(hi)) {
        c = INFINITY;
        e = 0.0f;
        return;
    }
    c = (float)(0.5 * ((double)lo + (double)hi));
    e = __double2float_ru(fmax((double)hi - (double)c, (double)c - (double)lo));
#else
    c = lo;
    e = hi;
#endif
}
#endif

#if EF_QNODE
// The 16-bit grid over the root's child boxes (the scene's padded bounds),
// three cells of margin on each side so the widened planes stay in range.
__global__ void encode_grid_kernel(ef::TravGrid* __restrict__ grid, const ef::GpuNode* __restrict__ in) {
    const ef::GpuNode g = in[0];
    float lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int k = 0; k < 4; ++k) {
        if (g.child[k] == ef::kEmptyChild) continue;
        lo[0] = fminf(lo[0], g.lox[k]); hi[0] = fmaxf(hi[0], g.hix[k]);
        lo[1] = fminf(lo[1], g.loy[k]); hi[1] = fmaxf(hi[1], g.hiy[k]);
        lo[2] = fminf(lo[2], g.loz[k]); hi[2] = fmaxf(hi[2], g.hiz[k]);
    }
    ef::TravGrid t = {};
    float scale = 1e-30f;
    for (int a = 0; a < 3; ++a) scale = fmaxf(scale, fmaxf(fabsf(lo[a]), fabsf(hi[a])));
    for (int a = 0; a < 3; ++a) {
        // a flat axis still gets cells of finite size
        const double ext = fmax((double)hi[a] - (double)lo[a], 1e-6 * (double)scale);
        const float cell = __double2float_ru(ext / 65528.0);
        t.cell[a] = cell;
        t.lo[a] = __double2float_rd((double)lo[a] - 3.0 * (double)cell);
    }
    *grid = t;
}

// lo | hi << 16 of one child box on one axis: floor / ceil to the grid and
// one more cell outward (the traversal's arithmetic error is below one
// cell, ef_device.cuh slab_q2)
__device__ __forceinline__ uint32_t encode_planes(float lo, float hi, float glo, float cell) {
    if (isinf(lo) || isinf(hi)) return ef::kEmptyPlanes;
    const double ql = floor(((double)lo - (double)glo) / (double)cell) - 1.0;
    const double qh = ceil(((double)hi - (double)glo) / (double)cell) + 1.0;
    const uint32_t l = (uint32_t)fmin(fmax(ql, 0.0), 65535.0), h = (uint32_t)fmin(fmax(qh, 0.0), 65535.0);
    return l | (h << 16);
}

__global__ void encode_nodes_kernel(ef::TravNode* __restrict__ out, const ef::GpuNode* __restrict__ in,
                                    int64_t n) {
    const ef::TravGrid G = *reinterpret_cast<const ef::TravGrid*>(out - 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const ef::GpuNode g = in[i];
        ef::TravNode t;
        for (int k = 0; k < 4; ++k) {
            const bool empty = g.child[k] == ef::kEmptyChild;
            t.px[k] = empty ? ef::kEmptyPlanes : encode_planes(g.lox[k], g.hix[k], G.lo[0], G.cell[0]);
            t.py[k] = empty ? ef::kEmptyPlanes : encode_planes(g.loy[k], g.hiy[k], G.lo[1], G.cell[1]);
            t.pz[k] = empty ? ef::kEmptyPlanes : encode_planes(g.loz[k], g.hiz[k], G.lo[2], G.cell[2]);
            t.child[k] = g.child[k];
        }
        out[i] = t;
    }
}
#else
__global__ void encode_nodes_kernel(ef::TravNode* __restrict__ out, const ef::GpuNode* __restrict__ in,
                                    int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const ef::GpuNode g = in[i];
        ef::TravNode t;
        for (int k = 0; k < 4; ++k) {
            encode_slab(g.lox[k], g.hix[k], t.cx[k], t.ex[k]);
            encode_slab(g.loy[k], g.hiy[k], t.cy[k], t.ey[k]);
            encode_slab(g.loz[k], g.hiz[k], t.cz[k], t.ez[k]);
            t.child[k] = g.child[k];
            t.pad[k] = 0;
        }
        out[i] = t;
    }
}
#endif

}  // namespace

// The allocation has one slot before node 0 (EF_QNODE: the TravGrid).
int ef::encode_nodes(ef_scene* s, cudaStream_t st) {
    if (s->n_nodes == 0) return EF_OK;
    if (!s->tnodes || s->n_tnodes_cap < s->n_nodes) {
        if (s->tnodes_base) {
            s->device_bytes -= (s->n_tnodes_cap + 1) * (int64_t)sizeof(TravNode);
            cudaFree(s->tnodes_base);
            s->tnodes_base = s->tnodes = nullptr;
        }
        cudaError_t e = cudaMalloc((void**)&s->tnodes_base, (size_t)(s->n_nodes + 1) * sizeof(TravNode));
        if (e != cudaSuccess) return check_cuda(e, "encode_nodes");
        s->tnodes = s->tnodes_base + 1;
        s->n_tnodes_cap = s->n_nodes;
        s->device_bytes += (s->n_nodes + 1) * (int64_t)sizeof(TravNode);
    }
#if EF_QNODE
    encode_grid_kernel<<<1, 1, 0, st>>>(reinterpret_cast<TravGrid*>(s->tnodes_base), s->nodes);
    count_launch();
#endif
    encode_nodes_kernel<<<(int)std::min<int64_t>((s->n_nodes + 255) / 256, 148 * 8), 256, 0, st>>>(
        s->tnodes, s->nodes, s->n_nodes);
    count_launch();
    return check_cuda(cudaGetLastError(), "encode_nodes");
}

int ef::update_shade(ef_scene* s, cudaStream_t st) {
    if (s->n_tri == 0) return EF_OK;
    if (!s->shade) {
        cudaError_t e = cudaMalloc((void**)&s->shade, (size_t)s->n_tri * sizeof(GpuShade));
        if (e != cudaSuccess) return check_cuda(e, "update_shade");
        s->device_bytes += s->n_tri * (int64_t)sizeof(GpuShade);
    }
    shade_kernel<<<(int)std::min<int64_t>((s->n_tri + 255) / 256, 148 * 8), 256, 0, st>>>(
        s->shade, s->normals, s->mat, s->pdiff, s->n_tri);
    count_launch();
    if (s->n_tri <= kTailMaxTris) {
        if (!s->tri_box) {
            cudaError_t e = cudaMalloc((void**)&s->tri_box, (size_t)s->n_tri * 8 * sizeof(float));
            if (e != cudaSuccess) return check_cuda(e, "update_shade");
            s->device_bytes += s->n_tri * 8 * (int64_t)sizeof(float);
        }
        tribox_kernel<<<(int)((s->n_tri + 255) / 256), 256, 0, st>>>(s->tri_box, s->tris_by_id,
                                                                      s->n_tri, s->pad);
        count_launch();
        // each triangle once, in (first) leaf order
        const bool host_order = (int64_t)s->clu_order.size() == s->n_tri;
        if (host_order || (s->leaf_order && s->n_refs == s->n_tri)) {
            const int64_t n_clu = (s->n_tri + kTailCluster - 1) / kTailCluster;
            if (!s->clu_box) {
                cudaError_t e = cudaMalloc((void**)&s->clu_box, (size_t)n_clu * 8 * sizeof(float));
                if (e == cudaSuccess) e = cudaMalloc((void**)&s->clu_ids, (size_t)s->n_tri * sizeof(int32_t));
                if (e != cudaSuccess) return check_cuda(e, "update_shade clusters");
                s->device_bytes += n_clu * 32 + s->n_tri * 4;
            }
            s->n_clu = n_clu;
            cudaError_t e = cudaSuccess;
            if (host_order) {
                e = cudaMemcpyAsync(s->clu_ids, s->clu_order.data(), (size_t)s->n_tri * sizeof(int32_t),
                                    cudaMemcpyHostToDevice, st);
            } else {
                order_kernel<<<(int)((s->n_tri + 255) / 256), 256, 0, st>>>(s->clu_ids, s->leaf_order, s->n_tri);
                count_launch();
            }
            if (e != cudaSuccess) return check_cuda(e, "update_shade clusters");
            cluster_kernel<<<(int)((n_clu + 127) / 128), 128, 0, st>>>(s->clu_box, s->clu_ids, s->tri_box,
                                                                      s->n_tri, n_clu);
            count_launch();
        }
    }
    return check_cuda(cudaGetLastError(), "shade_kernel");
}

extern "C" int ef_scene_create(const double* v0, const double* e1, const double* e2,
                               const double* normals, const int64_t* material_index, int64_t n_tri,
                               const double* absorption, const double* scattering,
                               int32_t n_materials, int32_t n_bands, ef_scene** out) {
    return ef_scene_create_ex(v0, e1, e2, normals, material_index, n_tri, absorption, scattering,
                              n_materials, n_bands, 0u, out);
}

extern "C" int ef_scene_create_ex(const double* v0, const double* e1, const double* e2,
                                  const double* normals, const int64_t* material_index, int64_t n_tri,
                                  const double* absorption, const double* scattering,
                                  int32_t n_materials, int32_t n_bands, uint32_t flags,
                                  ef_scene** out) {
    if (!out) return set_error(EF_EINVAL, "ef_scene_create: out is null");
    if (flags & ~(uint32_t)EF_SCENE_DEVICE_BUILD)
        return set_error(EF_EINVAL, "ef_scene_create: unknown flags");
    *out = nullptr;
    if (n_tri < 0) return set_error(EF_EINVAL, "ef_scene_create: n_tri < 0");
    if (n_bands < 1 || n_bands > kMaxBands)
        return set_error(EF_EINVAL, "ef_scene_create: n_bands must be in [1, 8]");
    if (n_materials < 1) return set_error(EF_EINVAL, "ef_scene_create: need at least one material");
    if (!absorption || !scattering) return set_error(EF_EINVAL, "ef_scene_create: null material table");
    if (n_tri > 0 && (!v0 || !e1 || !e2 || !normals || !material_index))
        return set_error(EF_EINVAL, "ef_scene_create: null geometry array");
    for (int64_t i = 0; i < (int64_t)n_materials * n_bands; ++i) {
        // Material.__post_init__ (scene.py:38-45)
        if (!(absorption[i] >= 0.0 && absorption[i] <= 1.0) ||
            !(scattering[i] >= 0.0 && scattering[i] <= 1.0))
            return set_error(EF_EINVAL, "ef_scene_create: absorption and scattering coefficients must lie in [0, 1]");
    }
    for (int64_t t = 0; t < n_tri; ++t)
        if (material_index[t] < 0 || material_index[t] >= n_materials)
            return set_error(EF_EINVAL, "ef_scene_create: material index out of range at triangle " + std::to_string(t));
    for (int64_t i = 0; i < 9 * n_tri / 3; ++i)
        if (!std::isfinite(v0[i]) || !std::isfinite(e1[i]) || !std::isfinite(e2[i]))
            return set_error(EF_EINVAL, "ef_scene_create: non-finite vertex data");

    ef_scene* s = new ef_scene();
    s->n_tri = n_tri;
    s->n_bands = n_bands;
    s->n_mat = n_materials;
    try {
        // material reflection factors: p = mean_b(s_b) summed
        // sequentially; E_b *= (1 - a_b) * s_b/p (diffuse) or (1-s_b)/(1-p)
        std::vector<float> fd((size_t)n_materials * n_bands), fs(fd.size()), fr(fd.size());
        std::vector<double> pd(n_materials);
        for (int m = 0; m < n_materials; ++m) {
            double p = 0.0;
            for (int b = 0; b < n_bands; ++b) p += scattering[m * n_bands + b];
            p = p / (double)n_bands;
            pd[m] = p;
            for (int b = 0; b < n_bands; ++b) {
                const double keep = 1.0 - absorption[m * n_bands + b];
                const double sb = scattering[m * n_bands + b];
                fd[m * n_bands + b] = p > 0.0 ? (float)(keep * (sb / p)) : 0.0f;
                fs[m * n_bands + b] = p < 1.0 ? (float)(keep * ((1.0 - sb) / (1.0 - p))) : 0.0f;
                fr[m * n_bands + b] = (float)(keep * sb);
            }
        }
        cudaError_t e = cudaSuccess;
#define EF_UP(dst, src, n)                                                        \
    if (e == cudaSuccess) e = upload(&s->dst, src, n, s->device_bytes);
        EF_UP(fd, fd.data(), fd.size());
        EF_UP(fs, fs.data(), fs.size());
        EF_UP(pdiff, pd.data(), pd.size());
        EF_UP(fr, fr.data(), fr.size());
        if (n_tri > 0 && (flags & EF_SCENE_DEVICE_BUILD)) {
            std::vector<double> by_id(9 * n_tri);
            std::vector<int32_t> mat(n_tri);
            for (int64_t t = 0; t < n_tri; ++t) {
                for (int k = 0; k < 3; ++k) {
                    by_id[9 * t + k] = v0[3 * t + k];
                    by_id[9 * t + 3 + k] = e1[3 * t + k];
                    by_id[9 * t + 6 + k] = e2[3 * t + k];
                }
                mat[t] = (int32_t)material_index[t];
            }
            EF_UP(tris_by_id, by_id.data(), by_id.size());
            EF_UP(normals, normals, (size_t)3 * n_tri);
            EF_UP(mat, mat.data(), mat.size());
            s->n_refs = n_tri;
            if (e == cudaSuccess) e = cudaMalloc((void**)&s->tris, (size_t)n_tri * sizeof(GpuTri));
            if (e == cudaSuccess) e = cudaMalloc((void**)&s->leaf_order, (size_t)n_tri * sizeof(int64_t));
            if (e == cudaSuccess) {
                s->device_bytes += n_tri * (int64_t)(sizeof(GpuTri) + sizeof(int64_t));
                const int rc = device_build_bvh(s, s->tris_by_id, s->tris_by_id + 3,
                                                s->tris_by_id + 6, 9, nullptr);
                if (rc != EF_OK) {
                    free_scene(s);
                    return rc;
                }
            }
        } else if (n_tri > 0) {
            HostBvh bvh;
            build_bvh(v0, e1, e2, n_tri, bvh);
            const int64_t n_refs = (int64_t)bvh.order.size();
            std::vector<GpuTri> tris(n_refs);
            std::vector<double> by_id(9 * n_tri);
            std::vector<int32_t> mat(n_tri);
            for (int64_t i = 0; i < n_refs; ++i) {
                const int64_t id = bvh.order[i];
                for (int k = 0; k < 3; ++k) {
                    tris[i].v[k] = v0[3 * id + k];
                    tris[i].v[3 + k] = e1[3 * id + k];
                    tris[i].v[6 + k] = e2[3 * id + k];
                }
                tris[i].id = id;
            }
            for (int64_t t = 0; t < n_tri; ++t) {
                for (int k = 0; k < 3; ++k) {
                    by_id[9 * t + k] = v0[3 * t + k];
                    by_id[9 * t + 3 + k] = e1[3 * t + k];
                    by_id[9 * t + 6 + k] = e2[3 * t + k];
                }
                mat[t] = (int32_t)material_index[t];
            }
            s->n_refs = n_refs;
            if (n_tri <= kTailMaxTris) {   // leaf order with repeats dropped (tail sweep clusters)
                std::vector<char> seen(n_tri, 0);
                for (int64_t i = 0; i < n_refs; ++i)
                    if (!seen[bvh.order[i]]) {
                        seen[bvh.order[i]] = 1;
                        s->clu_order.push_back((int32_t)bvh.order[i]);
                    }
            }
            s->n_nodes = (int64_t)bvh.nodes.size();
            s->max_depth = bvh.max_depth;
            s->max_leaf = bvh.max_leaf;
            if (bvh.max_stack > kStackSize) {
                free_scene(s);
                return set_error(EF_EUNSUPPORTED, "ef_scene_create: BVH deeper than the traversal stack");
            }
            EF_UP(nodes, bvh.nodes.data(), bvh.nodes.size());
            EF_UP(leaf_order, bvh.order.data(), bvh.order.size());
            EF_UP(level_nodes, bvh.level_nodes.data(), bvh.level_nodes.size());
            s->level_start = bvh.level_start;
            s->n_nodes_cap = s->n_nodes;
            s->level_nodes_len = (int64_t)bvh.level_nodes.size();
            s->pad = bvh.pad;
            EF_UP(tris, tris.data(), tris.size());
            EF_UP(tris_by_id, by_id.data(), by_id.size());
            EF_UP(normals, normals, (size_t)3 * n_tri);
            EF_UP(mat, mat.data(), mat.size());
        }
#undef EF_UP
        if (e != cudaSuccess) {
            free_scene(s);
            return check_cuda(e, "ef_scene_create upload");
        }
        int rc = encode_nodes(s, nullptr);
        if (rc == EF_OK) rc = update_shade(s, nullptr);
        if (rc == EF_OK) e = cudaStreamSynchronize(nullptr);
        if (rc != EF_OK || e != cudaSuccess) {
            free_scene(s);
            return rc != EF_OK ? rc : check_cuda(e, "ef_scene_create shade");
        }
    } catch (const std::exception& ex) {
        free_scene(s);
        return set_error(EF_EINVAL, std::string("ef_scene_create: ") + ex.what());
    }
    *out = s;
    return EF_OK;
}

extern "C" int ef_scene_destroy(ef_scene* s) {
    free_scene(s);
    return EF_OK;
}

extern "C" int ef_scene_info(const ef_scene* s, int64_t* o) {
    if (!s || !o) return set_error(EF_EINVAL, "ef_scene_info: null argument");
    o[0] = s->n_tri;
    o[7] = s->n_refs;
    o[1] = s->n_nodes;
    o[2] = s->max_depth;
    o[3] = s->device_bytes;
    o[4] = s->max_leaf;
    o[5] = s->n_bands;
    o[6] = s->n_mat;
    return EF_OK;
}

// ---------------------------------------------------------------------------
// Dynamic scenes: new vertex data for the same triangle
// list, then a bottom-up refit of the 4-wide tree on the device, one launch
// per tree level (deepest first).  Topology and leaf order are kept.
namespace {

__global__ void update_tris_kernel(ef::GpuTri* tris, double* by_id, double* normals_out,
                                   const int64_t* order, const double* v0, const double* e1,
                                   const double* e2, const double* normals, int64_t n,
                                   int64_t n_refs) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_refs || i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n_refs) {
            const int64_t id = order[i];
            ef::GpuTri t;
            for (int k = 0; k < 3; ++k) {
                t.v[k] = v0[3 * id + k];
                t.v[3 + k] = e1[3 * id + k];
                t.v[6 + k] = e2[3 * id + k];
            }
            t.id = id;
            tris[i] = t;
        }
        if (i >= n) continue;
        for (int k = 0; k < 3; ++k) {
            by_id[9 * i + k] = v0[3 * i + k];
            by_id[9 * i + 3 + k] = e1[3 * i + k];
            by_id[9 * i + 6 + k] = e2[3 * i + k];
            normals_out[3 * i + k] = normals[3 * i + k];
        }
    }
}

__global__ void copy_rows_kernel(double* by_id, double* normals_out, const double* v0,
                                 const double* e1, const double* e2, const double* normals,
                                 int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        for (int k = 0; k < 3; ++k) {
            by_id[9 * i + k] = v0[3 * i + k];
            by_id[9 * i + 3 + k] = e1[3 * i + k];
            by_id[9 * i + 6 + k] = e2[3 * i + k];
            normals_out[3 * i + k] = normals[3 * i + k];
        }
    }
}

__global__ void refit_level_kernel(ef::GpuNode* nodes, const ef::GpuTri* tris,
                                   const int32_t* level, int64_t count, double pad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        ef::GpuNode& g = nodes[level[i]];
        for (int c = 0; c < 4; ++c) {
            const int32_t ch = g.child[c];
            if (ch == ef::kEmptyChild) continue;
            double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
            if (ch >= 0) {   // inner child: union of its (already refit) slots
                const ef::GpuNode& cn = nodes[ch];
                for (int k = 0; k < 4; ++k) {
                    if (cn.child[k] == ef::kEmptyChild) continue;
                    lo[0] = fmin(lo[0], (double)cn.lox[k]); hi[0] = fmax(hi[0], (double)cn.hix[k]);
                    lo[1] = fmin(lo[1], (double)cn.loy[k]); hi[1] = fmax(hi[1], (double)cn.hiy[k]);
                    lo[2] = fmin(lo[2], (double)cn.loz[k]); hi[2] = fmax(hi[2], (double)cn.hiz[k]);
                }
                // already padded and rounded outward one level down
                g.lox[c] = (float)lo[0]; g.hix[c] = (float)hi[0];
                g.loy[c] = (float)lo[1]; g.hiy[c] = (float)hi[1];
                g.loz[c] = (float)lo[2]; g.hiz[c] = (float)hi[2];
            } else {         // leaf: vertices v0, v0+e1, v0+e2 of its triangles
                const uint32_t e = ~(uint32_t)ch;
                const uint32_t start = e >> 3, cnt = (e & 7u) + 1u;
                for (uint32_t j = 0; j < cnt; ++j) {
                    const double* v = tris[start + j].v;
                    for (int k = 0; k < 3; ++k) {
                        const double a = v[k], b = v[k] + v[3 + k], d = v[k] + v[6 + k];
                        lo[k] = fmin(lo[k], fmin(a, fmin(b, d)));
                        hi[k] = fmax(hi[k], fmax(a, fmax(b, d)));
                    }
                }
                g.lox[c] = __double2float_rd(lo[0] - pad); g.hix[c] = __double2float_ru(hi[0] + pad);
                g.loy[c] = __double2float_rd(lo[1] - pad); g.hiy[c] = __double2float_ru(hi[1] + pad);
                g.loz[c] = __double2float_rd(lo[2] - pad); g.hiz[c] = __double2float_ru(hi[2] + pad);
            }
        }
    }
}

}  // namespace

extern "C" int ef_scene_rebuild(ef_scene* s, const double* v0, const double* e1, const double* e2,
                                const double* normals, void* stream) {
    if (!s || !v0 || !e1 || !e2 || !normals) return set_error(EF_EINVAL, "ef_scene_rebuild: null argument");
    if (s->n_tri == 0) return EF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = s->n_tri;
    // original-order copies first (the all-pairs path and the shading normals)
    copy_rows_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, st>>>(
        s->tris_by_id, s->normals, v0, e1, e2, normals, n);
    count_launch();
    int rc = check_cuda(cudaGetLastError(), "ef_scene_rebuild");
    s->clu_order.clear();   // the device tree's leaf order from now on
    if (rc == EF_OK) rc = device_build_bvh(s, v0, e1, e2, 3, st);
    if (rc == EF_OK) rc = encode_nodes(s, st);
    if (rc != EF_OK) return rc;
    return update_shade(s, st);   // after the build: the boxes use its padding
}

extern "C" int ef_scene_refit(ef_scene* s, const double* v0, const double* e1, const double* e2,
                              const double* normals, void* stream) {
    if (!s || !v0 || !e1 || !e2 || !normals) return set_error(EF_EINVAL, "ef_scene_refit: null argument");
    if (s->n_tri == 0) return EF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = s->n_tri;
    const int64_t nm = std::max(n, s->n_refs);
    update_tris_kernel<<<(int)std::min<int64_t>((nm + 255) / 256, 148 * 8), 256, 0, st>>>(
        s->tris, s->tris_by_id, s->normals, s->leaf_order, v0, e1, e2, normals, n, s->n_refs);
    count_launch();
    const int rc = update_shade(s, st);
    if (rc != EF_OK) return rc;
    const int levels = (int)s->level_start.size() - 1;
    for (int l = levels - 1; l >= 0; --l) {
        const int64_t a = s->level_start[l], cnt = s->level_start[l + 1] - a;
        refit_level_kernel<<<(int)std::min<int64_t>((cnt + 127) / 128, 148 * 8), 128, 0, st>>>(
            s->nodes, s->tris, s->level_nodes + a, cnt, s->pad);
        count_launch();
    }
    const int rc2 = check_cuda(cudaGetLastError(), "ef_scene_refit");
    return rc2 != EF_OK ? rc2 : encode_nodes(s, st);
}
