// Batched ray-query and SH kernels behind the reference's query API, and
// the C ABI of the trace (the trace kernels themselves: ef_trace_kernels.cuh,
// compiled per instantiation in ef_trace_{brute,bvh}_nb{4,8}.cu).
//
// Reference functions replaced (see include/echoforge_b200.h):
//   SceneModel.intersect_batch  scene.py:208-230
//   BVH.intersect               bvh.py:130-160
//   SceneModel.occluded_batch   scene.py:232-252
//   eval_sh_batch               sh.py:86-126
//   trace_frame                 SPEC.md:207-215 (bounce model: DESIGN.md 3)
#include "ef_trace_kernels.cuh"

namespace ef {

// ---------------------------------------------------------------------------
__global__ void intersect_kernel(const TravNode* __restrict__ nodes, const GpuTri* __restrict__ tris,
                                 const double* __restrict__ tris_by_id, int32_t n_tri, bool brute,
                                 const double* __restrict__ o, const double* __restrict__ d,
                                 int64_t n, double t_min, const double* __restrict__ t_max,
                                 double* t_out, int64_t* tri_out, uint8_t* hit_out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double ox = o[3 * i], oy = o[3 * i + 1], oz = o[3 * i + 2];
        const double dx = d[3 * i], dy = d[3 * i + 1], dz = d[3 * i + 2];
        const double tm = t_max ? t_max[i] : INFINITY;
        Hit h;
        if (brute)
            h = closest_brute(tris_by_id, n_tri, ox, oy, oz, dx, dy, dz, t_min, tm);
        else
            h = closest_bvh(nodes, tris, ox, oy, oz, dx, dy, dz, t_min, tm);
        const bool hit = h.id != INT32_MAX;
        t_out[i] = hit ? h.t : INFINITY;
        tri_out[i] = hit ? h.id : -1;
        hit_out[i] = hit;
    }
}

// occluded_batch (scene.py:232-252): segment visibility with the
// reference's limit = dist - RAY_EPS; all-pairs uses t < limit (scene.py:247),
// the BVH path t <= limit (scene.py:250).
__global__ void occluded_kernel(const TravNode* __restrict__ nodes, const GpuTri* __restrict__ tris,
                                const double* __restrict__ tris_by_id, int32_t n_tri, bool brute,
                                const double* __restrict__ o, const double* __restrict__ tg,
                                int64_t n, uint8_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double ox = o[3 * i], oy = o[3 * i + 1], oz = o[3 * i + 2];
        const double ex = tg[3 * i] - ox, ey = tg[3 * i + 1] - oy, ez = tg[3 * i + 2] - oz;
        const double dist = sqrt((ex * ex + ey * ey) + ez * ez);   // np.linalg.norm order
        const double safe = fmax(dist, 1e-12);
        const double dx = ex / safe, dy = ey / safe, dz = ez / safe;
        const double limit = dist - kRayEps;
        bool blocked = false;
        if (brute) {
            for (int k = 0; k < n_tri && !blocked; ++k) {
                double t;
                blocked = mt_exact(ox, oy, oz, dx, dy, dz, tris_by_id + 9 * k, t) && t > kRayEps &&
                          t < limit;
            }
        } else {
            blocked = closest_bvh(nodes, tris, ox, oy, oz, dx, dy, dz, kRayEps, limit).id != INT32_MAX;
        }
        out[i] = blocked;
    }
}

template <int ORDER>
__global__ void eval_sh_kernel(const double* __restrict__ dirs, int64_t n, double* __restrict__ out) {
    constexpr int NK = (ORDER + 1) * (ORDER + 1);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double Y[NK];
        eval_sh<ORDER>(dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2], Y);
#pragma unroll
        for (int k = 0; k < NK; ++k) out[i * NK + k] = Y[k];
    }
}

__global__ void ray_triangles_kernel(const double* __restrict__ o, const double* __restrict__ d,
                                     int64_t nr, const double* __restrict__ v0,
                                     const double* __restrict__ e1, const double* __restrict__ e2,
                                     int64_t nt, double t_min, const double* __restrict__ t_max,
                                     double* t_out, uint8_t* valid_out) {
    const int64_t total = nr * nt;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / nt, k = i - r * nt;
        double v[9];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            v[c] = v0[3 * k + c];
            v[3 + c] = e1[3 * k + c];
            v[6 + c] = e2[3 * k + c];
        }
        double t;
        bool ok = mt_full(o[3 * r], o[3 * r + 1], o[3 * r + 2], d[3 * r], d[3 * r + 1], d[3 * r + 2], v, t);
        ok = ok && t > t_min && (!t_max || t <= t_max[r]);
        t_out[i] = t;
        valid_out[i] = ok;
    }
}

template <int ORDER>
__global__ void loudness_kernel(const double* __restrict__ avg, int64_t n,
                                const double* __restrict__ design, int n_design, double* out) {
    // one warp per distribution: gains on the design, then (4 pi/N) B^T diag(g) B
    constexpr int NK = (ORDER + 1) * (ORDER + 1);
    extern __shared__ double sh[];
    double* sB = sh;                                       // n_design * NK
    double* sg = sh + n_design * NK + (threadIdx.x >> 5) * n_design;
    for (int j = threadIdx.x; j < n_design; j += blockDim.x) {
        double Y[NK];
        eval_sh<ORDER>(design[3 * j], design[3 * j + 1], design[3 * j + 2], Y);
        for (int k = 0; k < NK; ++k) sB[j * NK + k] = Y[k];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t w = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    if (w >= n) return;
    const double* a = avg + w * NK;
    for (int j = lane; j < n_design; j += 32) {
        double g = 0.0;
        for (int k = 0; k < NK; ++k) g += sB[j * NK + k] * a[k];
        sg[j] = fmax(0.0, g);
    }
    __syncwarp();
    const double scale = 4.0 * M_PI / (double)n_design;
    for (int e = lane; e < NK * NK; e += 32) {
        const int k1 = e / NK, k2 = e % NK;
        double acc = 0.0;
        for (int j = 0; j < n_design; ++j) acc += sB[j * NK + k1] * sg[j] * sB[j * NK + k2];
        out[w * NK * NK + e] = scale * acc;
    }
}

static int grid_for(int64_t n, int threads) {
    long long g = (n + threads - 1) / threads;
    return (int)std::max(1LL, std::min(g, 148LL * 32));
}

}  // namespace ef

using namespace ef;

extern "C" int ef_intersect_batch(const ef_scene* s, const double* origins, const double* dirs,
                                  int64_t n, double t_min, const double* t_max, int32_t mode,
                                  double* t_out, int64_t* tri_out, uint8_t* hit_out, void* stream) {
    if (!s || (n > 0 && (!origins || !dirs || !t_out || !tri_out || !hit_out)))
        return set_error(EF_EINVAL, "ef_intersect_batch: null argument");
    if (mode < 0 || mode > 2) return set_error(EF_EINVAL, "ef_intersect_batch: mode must be 0, 1 or 2");
    if (n == 0) return EF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (s->n_tri == 0) {
        // scene.py:213-215: all miss
        return set_error(EF_EUNSUPPORTED, "ef_intersect_batch: empty scene is handled by the host");
    }
    const bool brute = mode == 1 || (mode == 0 && s->n_tri <= kBruteMaxTris);
    intersect_kernel<<<grid_for(n, 128), 128, 0, st>>>(s->tnodes, s->tris, s->tris_by_id,
                                                       (int32_t)s->n_tri, brute, origins, dirs, n,
                                                       t_min, t_max, t_out, tri_out, hit_out);
    count_launch();
    return check_cuda(cudaGetLastError(), "intersect_kernel");
}

extern "C" int ef_occluded_batch(const ef_scene* s, const double* origins, const double* targets,
                                 int64_t n, uint8_t* out, void* stream) {
    if (!s || (n > 0 && (!origins || !targets || !out)))
        return set_error(EF_EINVAL, "ef_occluded_batch: null argument");
    if (n == 0) return EF_OK;
    if (s->n_tri == 0) return set_error(EF_EUNSUPPORTED, "ef_occluded_batch: empty scene is handled by the host");
    const bool brute = s->n_tri <= kBruteMaxTris;
    occluded_kernel<<<grid_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
        s->tnodes, s->tris, s->tris_by_id, (int32_t)s->n_tri, brute, origins, targets, n, out);
    count_launch();
    return check_cuda(cudaGetLastError(), "occluded_kernel");
}

extern "C" int ef_eval_sh_batch(const double* dirs, int64_t n, int32_t order, double* out,
                                void* stream) {
    if (order < 0 || order > kMaxOrder)
        return set_error(EF_EINVAL, "order must be in [0, 4], got " + std::to_string(order));
    if (n == 0) return EF_OK;
    if (!dirs || !out) return set_error(EF_EINVAL, "ef_eval_sh_batch: null argument");
    cudaStream_t st = (cudaStream_t)stream;
    const int g = grid_for(n, 128);
    switch (order) {
        case 0: eval_sh_kernel<0><<<g, 128, 0, st>>>(dirs, n, out); break;
        case 1: eval_sh_kernel<1><<<g, 128, 0, st>>>(dirs, n, out); break;
        case 2: eval_sh_kernel<2><<<g, 128, 0, st>>>(dirs, n, out); break;
        case 3: eval_sh_kernel<3><<<g, 128, 0, st>>>(dirs, n, out); break;
        default: eval_sh_kernel<4><<<g, 128, 0, st>>>(dirs, n, out); break;
    }
    count_launch();
    return check_cuda(cudaGetLastError(), "eval_sh_kernel");
}

namespace {

// The BVH trace kernels address their shared-memory stack columns from the
// constant kDynSmemBase (ef_device.cuh) and trap if their dynamic shared
// memory starts elsewhere.  A one-time probe (a kernel without static shared
// memory, like them) turns that into an error message before the first BVH
// trace of the process; it is not counted as a launch of the path.
__global__ void smem_base_probe(uint32_t* out) {
    extern __shared__ unsigned char probe_smem[];
    *out = (uint32_t)__cvta_generic_to_shared(probe_smem);
}

int check_smem_base() {
    static bool probed = false;
    static uint32_t base = 0;
    if (!probed) {
        uint32_t* d = nullptr;
        cudaError_t e = cudaMalloc(&d, sizeof(uint32_t));
        if (e == cudaSuccess) {
            smem_base_probe<<<1, 1, 16>>>(d);
            e = cudaGetLastError();
            if (e == cudaSuccess) e = cudaMemcpy(&base, d, sizeof(uint32_t), cudaMemcpyDeviceToHost);
            cudaFree(d);
        }
        if (e != cudaSuccess) return check_cuda(e, "smem_base_probe");   // probed again by the next call
        probed = true;
    }
    if (base == kDynSmemBase) return EF_OK;
    return set_error(EF_EUNSUPPORTED, "ef_trace: dynamic shared memory starts at window address " +
                                          std::to_string(base) + ", the kernels were built for " +
                                          std::to_string(kDynSmemBase) + " (kDynSmemBase, ef_device.cuh)");
}

// ef_trace and ef_trace_fused: either local H/Dir, or the ranks' blocks
// Hp/Dp (host arrays of n_ranks device pointers) with `spr` sources per rank
// (H = Dir = null).
int trace_impl(const ef_scene* s, const ef_trace_config* cfg, const double* src_pos,
               const uint32_t* src_key, const uint32_t* ray_ids, float* H, float* Dir,
               float* const* Hp, float* const* Dp, int32_t spr, unsigned long long* stats,
               double* sum_t, int32_t* path_nseg, int32_t* path_ids, void* stream) {
    if (!s || !cfg) return set_error(EF_EINVAL, "ef_trace: null scene or config");
    if (cfg->n_sources < 1) return set_error(EF_EINVAL, "ef_trace: need at least one source");
    if (cfg->order < 0 || cfg->order > kMaxOrder) return set_error(EF_EINVAL, "ef_trace: order must be in [0, 4]");
    if (cfg->n_bins < 1 || cfg->max_bounces < 1 || cfg->n_rays < 1)
        return set_error(EF_EINVAL, "ef_trace: n_bins, max_bounces and n_rays must be >= 1");
    if (cfg->n_rays > 0xffffffffLL) return set_error(EF_EINVAL, "ef_trace: n_rays must fit in 32 bits");
    if (!(cfg->bin_len > 0.0) || !(cfg->radius >= 0.0))
        return set_error(EF_EINVAL, "ef_trace: bin_len must be > 0 and radius >= 0");
    if (cfg->mode < 0 || cfg->mode > 2) return set_error(EF_EINVAL, "ef_trace: mode must be 0, 1 or 2");
    if (cfg->er_entries && (!cfg->er_count || cfg->er_capacity < 0))
        return set_error(EF_EINVAL, "ef_trace: an early-reflection list needs er_count and er_capacity >= 0");
    const bool fused = Hp != nullptr;
    if (!src_pos || !stats || !sum_t || (fused ? !Dp : (!H || !Dir)))
        return set_error(EF_EINVAL, "ef_trace: null buffer");
    if (fused && (spr < 1 || cfg->n_sources % spr != 0 || cfg->n_sources / spr > kMaxRanks))
        return set_error(EF_EINVAL, "ef_trace_fused: sources_per_rank must divide n_sources "
                                    "into at most 8 ranks");
    if (s->n_tri == 0) return set_error(EF_EUNSUPPORTED, "ef_trace: empty scene is handled by the host");
    const bool brute = cfg->mode == 1 || (cfg->mode == 0 && s->n_tri <= kBruteMaxTris);
    if (brute && s->n_tri > 2048) return set_error(EF_EINVAL, "ef_trace: all-pairs mode supports <= 2048 triangles");
    if (!brute) {
        const int rc = check_smem_base();
        if (rc != EF_OK) return rc;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int nk = (cfg->order + 1) * (cfg->order + 1);
    cudaError_t e = cudaSuccess;
    if (cfg->clear_outputs) {
        // DMA-engine clears, no kernel launch
        // (fused: the peer blocks belong to their owners, only local outputs)
        const size_t nh = (size_t)cfg->n_sources * cfg->n_bins * s->n_bands * nk;
        const size_t nd = (size_t)cfg->n_sources * s->n_bands * nk;
        const size_t nst = (size_t)cfg->n_sources * EF_ST_COUNT * 8;
        const char* h0 = reinterpret_cast<const char*>(H);
        // H | Dir | stats | sum_t back to back (FrameTracer's single
        // allocation; stats 8-byte aligned right after Dir): one memset
        const bool packed = !fused && (4 * (nh + nd)) % 8 == 0 &&
                            reinterpret_cast<const char*>(Dir) == h0 + 4 * nh &&
                            reinterpret_cast<const char*>(stats) == h0 + 4 * (nh + nd) &&
                            reinterpret_cast<const char*>(sum_t) == h0 + 4 * (nh + nd) + nst;
        if (packed) {
            e = cudaMemsetAsync(H, 0, 4 * (nh + nd) + nst + (size_t)cfg->n_sources * 8, st);
        } else {
            if (!fused) {
                e = cudaMemsetAsync(H, 0, nh * sizeof(float), st);
                if (e == cudaSuccess) e = cudaMemsetAsync(Dir, 0, nd * sizeof(float), st);
            }
            if (e == cudaSuccess) e = cudaMemsetAsync(stats, 0, nst, st);
            if (e == cudaSuccess) e = cudaMemsetAsync(sum_t, 0, (size_t)cfg->n_sources * 8, st);
        }
        if (e != cudaSuccess) return check_cuda(e, "cudaMemsetAsync");
    }
    // tail hand-off for small BVH scenes (tail_kernel): at most two paths
    // per SM (C2 sweep 32..592: 296 best, 1.53 vs 1.40 G seg/s without;
    // larger lists make whole CTAs run short paths one segment at a time);
    // EF_TAIL_LIVE overrides the threshold (0 = off; tuning)
    static const int tail_env = [] {
        const char* v = std::getenv("EF_TAIL_LIVE");
        return v ? std::atoi(v) : -1;
    }();
    const int tail_live = (brute || s->n_tri > kTailMaxTris || !s->tri_box || !s->clu_box ||
                           s->n_clu > kTailThreads) ? 0
                          : (tail_env >= 0 ? tail_env : 2 * sm_count());
    // scratch header: path counter (u64), finished paths (u64), continuation
    // counts (u32 long, u32 short), entries taken (u32); then the list
    constexpr size_t kHdr = 32;
    unsigned char* scratch = nullptr;
    keep_pool_memory();
    e = cudaMallocAsync((void**)&scratch, kHdr + (size_t)tail_live * sizeof(PathState<8>), st);
    if (e != cudaSuccess) return check_cuda(e, "cudaMallocAsync");
    unsigned long long* counter = reinterpret_cast<unsigned long long*>(scratch);
    for (int s0 = 0; s0 < cfg->n_sources; s0 += kMaxSourcesPerLaunch) {
        const int ns = std::min(kMaxSourcesPerLaunch, cfg->n_sources - s0);
        e = cudaMemsetAsync(scratch, 0, kHdr, st);
        if (e != cudaSuccess) break;
        TraceParams P;
        P.nodes = s->tnodes;
        P.tris = s->tris;
        P.tris_by_id = s->tris_by_id;
        P.n_tri = (int32_t)s->n_tri;
        P.shade = s->shade;
        P.tri_box = s->tri_box;
        P.clu_box = s->clu_box;
        P.clu_ids = s->clu_ids;
        P.n_clu = (int32_t)s->n_clu;
        P.n_refs = (int32_t)s->n_tri;   // ids in clu_ids: each triangle once
        P.fd = s->fd;
        P.fs = s->fs;
        P.nb = s->n_bands;
        P.src_pos = src_pos + 3 * s0;
        P.src_key = src_key ? src_key + s0 : nullptr;
        P.ray_ids = ray_ids;
        P.n_src = ns;
        P.n_rays = cfg->n_rays;
        P.ray0 = cfg->ray0;
        P.seed = cfg->seed;
        P.frame = cfg->frame;
        P.n_bins = cfg->n_bins;
        P.max_bounces = cfg->max_bounces;
        P.bin_len = cfg->bin_len;
        P.lx = cfg->listener[0];
        P.ly = cfg->listener[1];
        P.lz = cfg->listener[2];
        P.r2 = cfg->radius * cfg->radius;
        P.e0 = cfg->e0;
        if (fused) {
            for (int k = 0; k < kMaxRanks; ++k) {
                P.Hp[k] = k < cfg->n_sources / spr ? Hp[k] : nullptr;
                P.Dp[k] = k < cfg->n_sources / spr ? Dp[k] : nullptr;
            }
            P.spr = spr;
            P.src0 = s0;
        } else {   // one rank owning every source of this launch
            for (int k = 0; k < kMaxRanks; ++k) P.Hp[k] = P.Dp[k] = nullptr;
            P.Hp[0] = H + (size_t)s0 * cfg->n_bins * s->n_bands * nk;
            P.Dp[0] = Dir + (size_t)s0 * s->n_bands * nk;
            P.spr = ns;
            P.src0 = 0;
        }
        // vector reductions into this GPU's own blocks; scalar f32 reds over
        // the peer mapping (remote NVLink targets)
        static const int vec_env = [] {   // A/B: EF_VEC_RED=0 commits with scalar reds
            const char* e = std::getenv("EF_VEC_RED");
            return e ? std::atoi(e) : 1;
        }();
        // (the caller's H / Dir must start on 16-byte boundaries for the
        // vector form; any other base falls back to scalar reds)
        const bool aligned16 = !fused && (reinterpret_cast<uintptr_t>(H) % 16 == 0) &&
                               (reinterpret_cast<uintptr_t>(Dir) % 16 == 0);
        P.vec_red = (aligned16 && vec_env) ? 1 : 0;
        P.stats = stats + (size_t)s0 * EF_ST_COUNT;
        P.sum_t = sum_t + s0;
        P.path_nseg = path_nseg ? path_nseg + (size_t)s0 * cfg->n_rays : nullptr;
        P.path_ids = (path_ids && cfg->record_ids) ? path_ids + (size_t)s0 * cfg->n_rays * cfg->max_bounces : nullptr;
        P.timing = (P.path_ids && cfg->record_ids == 2 && cfg->max_bounces >= 6) ? 1 : 0;
        P.rain = cfg->diffuse_rain ? 1 : 0;
        P.fr = s->fr;
        P.er_max_order = cfg->er_entries ? std::max(0, std::min(cfg->er_max_order, 2)) : 0;
        P.er = static_cast<ef_er_entry*>(cfg->er_entries);
        P.er_count = cfg->er_count;
        P.er_cap = cfg->er_capacity;
        P.counter = counter;
        P.total = (unsigned long long)ns * (unsigned long long)cfg->n_rays;
        P.tail_live = tail_live;
        P.done = counter + 1;
        P.cont_count = reinterpret_cast<unsigned int*>(scratch + 16);   // [0], [1]
        P.cont_take = reinterpret_cast<unsigned int*>(scratch + 24);
        P.cont = scratch + kHdr;
        static const int force_big = [] {
            const char* e = std::getenv("EF_TRACE_BIG");   // tuning only: 0 / 1
            return e ? std::atoi(e) : -1;
        }();
        const bool big = force_big >= 0 ? force_big == 1
                                         : (int64_t)s->n_nodes * (int64_t)sizeof(GpuNode) +
                                                   s->n_refs * (int64_t)sizeof(GpuTri) > kBigSceneBytes;
        // the whole traversal stack in shared memory when the tree's bound
        // fits next to the counters (EF_SSTACK=0 disables; tuning)
        static const int sstack_env = [] {
            const char* e = std::getenv("EF_SSTACK");
            return e ? std::atoi(e) : 1;
        }();
        const int max_stack = 3 * s->max_depth + 1;
        const size_t sstack_bytes = (size_t)max_stack * kSmallThreads * sizeof(uint2) +
                                    (size_t)ns * (EF_ST_COUNT * 4 + 8) + 64;
        static const size_t sstack_max = [] {   // tuning: shared-stack budget (KB)
            const char* e = std::getenv("EF_SSTACK_MAXKB");
            return e ? (size_t)std::atoi(e) * 1024 : kMaxSstackBytes;
        }();
        const bool sstack_fits = max_stack <= kStackSize && sstack_bytes <= sstack_max;
        P.smem_stack = (!brute && (!big || sstack_max != kMaxSstackBytes) && sstack_env && sstack_fits)
                           ? max_stack : 0;
        // the tail hand-off is compiled into the shared-stack kernel only
        // (scenes of <= kTailMaxTris triangles whose whole stack fits)
        if (P.smem_stack == 0) P.tail_live = 0;
        if (s->n_bands <= 4) {
            e = brute ? trace_dispatch_brute_nb4(cfg->order, P, st)
                      : trace_dispatch_bvh_nb4(big, cfg->order, P, st);
            if (e == cudaSuccess && P.tail_live > 0) e = tail_dispatch_nb4(cfg->order, P, st);
        } else {
            e = brute ? trace_dispatch_brute_nb8(cfg->order, P, st)
                      : trace_dispatch_bvh_nb8(big, cfg->order, P, st);
            if (e == cudaSuccess && P.tail_live > 0) e = tail_dispatch_nb8(cfg->order, P, st);
        }
        if (e != cudaSuccess) break;
    }
    cudaError_t e2 = cudaFreeAsync(scratch, st);
    if (e != cudaSuccess) return check_cuda(e, "trace_kernel");
    return check_cuda(e2, "cudaFreeAsync");
}

}  // namespace

extern "C" int ef_trace(const ef_scene* s, const ef_trace_config* cfg, const double* src_pos,
                        const uint32_t* src_key, const uint32_t* ray_ids, float* H, float* Dir,
                        unsigned long long* stats, double* sum_t, int32_t* path_nseg,
                        int32_t* path_ids, void* stream) {
    return trace_impl(s, cfg, src_pos, src_key, ray_ids, H, Dir, nullptr, nullptr, 1, stats, sum_t,
                      path_nseg, path_ids, stream);
}

extern "C" int ef_trace_fused(const ef_scene* s, const ef_trace_config* cfg, const double* src_pos,
                              const uint32_t* src_key, const uint32_t* ray_ids,
                              float* const* hist_peers, float* const* dir_peers,
                              int32_t sources_per_rank, unsigned long long* stats, double* sum_t,
                              int32_t* path_nseg, int32_t* path_ids, void* stream) {
    if (!hist_peers || !dir_peers) return set_error(EF_EINVAL, "ef_trace_fused: null peer table");
    return trace_impl(s, cfg, src_pos, src_key, ray_ids, nullptr, nullptr, hist_peers, dir_peers,
                      sources_per_rank, stats, sum_t, path_nseg, path_ids, stream);
}

extern "C" int ef_ray_triangles(const double* origins, const double* dirs, int64_t n_rays,
                                const double* v0, const double* e1, const double* e2, int64_t n_tri,
                                double t_min, const double* t_max, double* t_out, uint8_t* valid_out,
                                void* stream) {
    if (n_rays < 0 || n_tri < 0) return set_error(EF_EINVAL, "ef_ray_triangles: negative size");
    if (n_rays == 0 || n_tri == 0) return EF_OK;
    if (!origins || !dirs || !v0 || !e1 || !e2 || !t_out || !valid_out)
        return set_error(EF_EINVAL, "ef_ray_triangles: null argument");
    ray_triangles_kernel<<<grid_for(n_rays * n_tri, 128), 128, 0, (cudaStream_t)stream>>>(
        origins, dirs, n_rays, v0, e1, e2, n_tri, t_min, t_max, t_out, valid_out);
    count_launch();
    return check_cuda(cudaGetLastError(), "ray_triangles_kernel");
}

extern "C" int ef_loudness_batch(const double* avg, int64_t n, int32_t order, const double* design,
                                 int32_t n_design, double* out, void* stream) {
    if (order < 0 || order > kMaxOrder) return set_error(EF_EINVAL, "order must be in [0, 4]");
    if (n == 0) return EF_OK;
    if (!avg || !design || !out || n_design < 1 || n_design > 256)
        return set_error(EF_EINVAL, "ef_loudness_batch: bad arguments");
    const int nk = (order + 1) * (order + 1);
    const int warps = 4;
    const size_t smem = (size_t)(n_design * nk + warps * n_design) * sizeof(double);
    const int grid = (int)((n + warps - 1) / warps);
    cudaStream_t st = (cudaStream_t)stream;
    switch (order) {
        case 0: loudness_kernel<0><<<grid, 32 * warps, smem, st>>>(avg, n, design, n_design, out); break;
        case 1: loudness_kernel<1><<<grid, 32 * warps, smem, st>>>(avg, n, design, n_design, out); break;
        case 2: loudness_kernel<2><<<grid, 32 * warps, smem, st>>>(avg, n, design, n_design, out); break;
        case 3: loudness_kernel<3><<<grid, 32 * warps, smem, st>>>(avg, n, design, n_design, out); break;
        default: loudness_kernel<4><<<grid, 32 * warps, smem, st>>>(avg, n, design, n_design, out); break;
    }
    count_launch();
    return check_cuda(cudaGetLastError(), "loudness_kernel");
}

#ifdef EF_PROFILE_PHASES
extern "C" int ef_debug_phases(unsigned long long* out8, int reset) {
    // the phase counters live in each trace translation unit: sum them
    for (int i = 0; i < ef::kPhaseSlots; ++i) out8[i] = 0;
    ef::debug_phases_brute_nb4(out8, reset);
    ef::debug_phases_brute_nb8(out8, reset);
    ef::debug_phases_bvh_nb4(out8, reset);
    ef::debug_phases_bvh_nb8(out8, reset);
    return EF_OK;
}
#endif
