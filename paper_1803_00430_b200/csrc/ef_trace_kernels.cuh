// K1 + K3 kernels: counter-based ray generation and the persistent trace
// megakernel (closest hit -> listener sphere -> SH histogram commit ->
// reflection), the frame-tail kernel, and their launchers.  Included by the
// per-instantiation translation units ef_trace_{brute,bvh}_nb{4,8}.cu (so the
// ~70 kernel instantiations compile in parallel) and by ef_trace.cu (the
// query kernels and the C ABI), which calls them through trace_dispatch /
// tail_dispatch below.
//
// Reference functions replaced (see include/echoforge_b200.h):
//   SceneModel.intersect_batch  scene.py:208-230
//   BVH.intersect               bvh.py:130-160
//   SceneModel.occluded_batch   scene.py:232-252
//   eval_sh_batch               sh.py:86-126
//   trace_frame                 SPEC.md:207-215 (bounce model: DESIGN.md 3)
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "ef_device.cuh"

namespace ef {

// One fat CTA per SM.  Scenes whose whole traversal stack fits in shared
// memory (C2) and the all-pairs scenes (C1) run 512 threads at 128
// registers.  Every other scene (C3, C5: nodes + triangles far beyond L1)
// runs kBigThreads = 1024 threads at 64 registers with the split stack
// (shared top + local overflow): with the 64-byte quantized nodes a node
// visit holds 16 node registers instead of 28, the spills that remain sit
// in the per-segment code, and twice the warps hide the dependent L1/L2
// latency of the descent (C5 4.02 -> 4.23, C3 2.69 -> 3.08 G seg/s against
// 512 threads; 768: 4.03 / 2.85, 896: 4.21 / 3.06; C2 loses at more than
// 512: 1.73 -> 1.46).  Tuning builds: EF_TRACE_THREADS, EF_BIG_THREADS.
#ifndef EF_TRACE_THREADS
#define EF_TRACE_THREADS 512
#endif
#ifndef EF_BIG_THREADS
#define EF_BIG_THREADS 1024
#endif
constexpr int kSmallThreads = EF_TRACE_THREADS;
constexpr int kBigThreads = EF_BIG_THREADS;
constexpr int64_t kBigSceneBytes = 4ll << 20;
// Shared traversal-stack entries per thread (the rest in local memory) when
// the tree's whole stack does not fit: 6 x 1024 threads (48 KB; 4 / 8 / 12
// entries: C5 4.21 / 4.23 / 4.19 against 4.25, C3 within 1%), columns for
// THREADS threads (compile-time stride).  A C5 segment pushes 2.8 entries
// and its stack never passes 12 (tools/probe_simt.py).
#ifndef EF_SPLIT_DEPTH
#define EF_SPLIT_DEPTH 6
#endif
template <int THREADS>
constexpr int kSplitDepth = EF_SPLIT_DEPTH;
// (A shared-memory copy of the top of the tree measured slower than leaving
// the space to L1 -- C5 2.93 vs 3.34 G seg/s with 128 KB, C2 flat -- and was
// removed; profiles/r01_node_cache_sweep.txt.)
constexpr size_t kMaxTraceSmem = 220 * 1024;
constexpr size_t kMaxSstackBytes = 128 * 1024;   // leave >= 128 KB of the SM's 256 KB to L1
constexpr int kMaxSourcesPerLaunch = 256;
constexpr int kMaxRanks = 8;   // GPUs of one node reachable by ef_trace_fused
constexpr int kTailLongSegs = 16;   // tail hand-off: paths with this many segments are taken first
constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// all-pairs closest hit over triangles staged in shared memory (T <= 512),
// ids ascending with a strict '<': ties go to the lowest id (scene.py:220)
// All-pairs closest hit (scene.py:208-230 for <= 512 triangles): the exact
// test of every triangle, lowest index on equal t.  Two triangles per step,
// each tested against t_max alone, so their f64 chains are independent and
// overlap; the running minimum is folded in afterwards in index order.
__device__ __forceinline__ Hit closest_brute(const double* __restrict__ s_tri, int n, double ox,
                                             double oy, double oz, double dx, double dy, double dz,
                                             double t_min, double t_max) {
    Hit h{INFINITY, INT32_MAX};
    int i = 0;
    for (; i + 1 < n; i += 2) {
        double ta, tb;
        const bool ha = mt_hit(ox, oy, oz, dx, dy, dz, s_tri + 9 * i, t_min, t_max, ta);
        const bool hb = mt_hit(ox, oy, oz, dx, dy, dz, s_tri + 9 * (i + 1), t_min, t_max, tb);
        if (ha && ta < h.t) {
            h.t = ta;
            h.id = i;
        }
        if (hb && tb < h.t) {
            h.t = tb;
            h.id = i + 1;
        }
    }
    if (i < n) {
        double t;
        if (mt_hit(ox, oy, oz, dx, dy, dz, s_tri + 9 * i, t_min, t_max, t) && t < h.t) {
            h.t = t;
            h.id = i;
        }
    }
    return h;
}

// All-pairs closest hit shared by the G lanes of a lane group (G a power of
// two dividing 32, `gmask` the group's lanes, `gl` this lane's rank in it):
// lane gl tests triangles gl, gl+G, ... against t_max alone, then a
// butterfly over the group keeps the lexicographic minimum of (t, id) -- the
// same answer as closest_brute (lowest id on equal t), on every lane.
template <int G>
__device__ __forceinline__ Hit closest_brute_group(const double* __restrict__ s_tri, int n, double ox,
                                                   double oy, double oz, double dx, double dy,
                                                   double dz, double t_min, double t_max,
                                                   unsigned gmask, int gl) {
    Hit h{INFINITY, INT32_MAX};
    for (int i = gl; i < n; i += G) {
        double t;
        if (mt_hit(ox, oy, oz, dx, dy, dz, s_tri + 9 * i, t_min, t_max, t) && t < h.t) {
            h.t = t;
            h.id = i;
        }
    }
#pragma unroll
    for (int k = G / 2; k >= 1; k >>= 1) {
        const double t2 = __shfl_xor_sync(gmask, h.t, k, G);
        const int id2 = __shfl_xor_sync(gmask, h.id, k, G);
        if (t2 < h.t || (t2 == h.t && id2 < h.id)) {
            h.t = t2;
            h.id = id2;
        }
    }
    return h;
}

struct TraceParams {
    const TravNode* nodes;   // traversal form (encode_nodes)
    const GpuTri* tris;
    const double* tris_by_id;
    int32_t n_tri;
    const GpuShade* shade;
    const float* tri_box;
    const float* clu_box;       // tail sweep level 1 (n_clu clusters of kTailCluster leaf-order triangles)
    const int32_t* clu_ids;
    int32_t n_clu, n_refs;
    const float* fd;
    const float* fs;
    int32_t nb;
    const double* src_pos;
    const uint32_t* src_key;
    const uint32_t* ray_ids;
    int32_t n_src;
    int64_t n_rays;
    uint32_t ray0, seed, frame;
    int32_t n_bins, max_bounces;
    double bin_len, lx, ly, lz, r2;
    float e0;
    // histogram / direct-sound blocks: global source g lives on rank g / spr
    // at block g % spr (ef_trace: one "rank", this process's H and Dir)
    float* Hp[kMaxRanks];
    float* Dp[kMaxRanks];
    int32_t spr;
    int32_t src0;           // global index of this launch's source 0
    int32_t vec_red;        // blocks are local: commit with 16-byte vector reductions
    unsigned long long* stats;
    double* sum_t;
    int32_t* path_nseg;
    int32_t* path_ids;
    unsigned long long* counter;
    unsigned long long total;
    int32_t rain;           // diffuse rain (next-event estimation)
    const float* fr;        // (n_mat, nb) diffusely reflected fraction (1-a)*s, f32
    int32_t er_max_order;   // arrivals of order 1..er_max_order -> ER list
    ef_er_entry* er;        // ER list (capacity er_cap), er_count = used entries
    unsigned int* er_count;
    int64_t er_cap;
    int32_t timing;         // debug: path_ids rows get (t0, t1, smid, nseg)
    int32_t smem_stack;     // traversal stack entries per thread kept in shared memory
    // tail hand-off (tail_kernel): once the path counter is exhausted and at
    // most tail_live paths are unfinished, they move to `cont` (0 = off)
    int32_t tail_live;
    unsigned long long* done;   // finished paths (warp-aggregated)
    void* cont;                 // PathState<NBMAX>[tail_live]
    unsigned int* cont_count;   // [0] long paths (cont[0..)), [1] short ones (cont[tail_live-1..] down)
    unsigned int* cont_take;    // entries taken by tail_kernel (long ones first)
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

struct LaneStats {
    int src = -1;
    uint32_t c[EF_ST_COUNT] = {};
    double sum_t = 0.0;
};

__device__ __forceinline__ void flush_stats(LaneStats& ls, unsigned int* s_stats,
                                            double* s_sumt) {
    if (ls.src >= 0) {
#pragma unroll
        for (int i = 0; i < EF_ST_COUNT; ++i)
            if (ls.c[i]) atomicAdd(&s_stats[ls.src * EF_ST_COUNT + i], ls.c[i]);   // native 32-bit ATOMS
        if (ls.sum_t != 0.0) atomicAdd(&s_sumt[ls.src], ls.sum_t);
    }
#pragma unroll
    for (int i = 0; i < EF_ST_COUNT; ++i) ls.c[i] = 0;
    ls.sum_t = 0.0;
}

// Block of launch source `src` in the peer table: rank g / spr, block g % spr
// (its histogram or direct-sound block is `per` floats).  Remote atomics go
// over NVLink to the owning GPU, so the frame's reduce-scatter happens inside
// the trace kernel, splat by splat.
__device__ __forceinline__ float* peer_block(float* const (&tab)[kMaxRanks], const TraceParams& P,
                                             int src, size_t per) {
    const int g = P.src0 + src;
    const int o = g / P.spr;
    return tab[o] + (size_t)(g - o * P.spr) * per;
}

// Adds one arrival's splat c[b] * Y[k] (b < nb, k < NK) into the nb * NK
// contiguous floats at dst.  Warp-aggregated: the lanes committing together
// are grouped by destination (__match_any_sync on the block address -- the
// same source's Dir block, or the same histogram bin); a group's leader
// alone commits the group's sum (shuffled from its peers, in lane order).
// With local blocks the commit is 16-byte vector reductions
// (red.global.add.v4.f32; nb * NK is a multiple of 4 for nb in {4, 8}, and
// every bin / block starts on a 16-byte boundary): nb * NK / 4 requests per
// arrival instead of nb * NK.
template <int NBMAX, int NK>
__device__ __forceinline__ void commit_splat(const TraceParams& P, float* dst, const float* c,
                                             const float* Yf) {
    const int nb = P.nb;
    const unsigned am = __activemask();
    const unsigned peers = __match_any_sync(am, reinterpret_cast<unsigned long long>(dst));
    const int lane = threadIdx.x & 31;
    const bool lead = lane == __ffs(peers) - 1;
    if (P.vec_red && (nb * NK) % 4 == 0) {
#pragma unroll
        for (int j = 0; j < NBMAX * NK; j += 4) {
            if (j < nb * NK) {
                float v[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) v[q] = c[(j + q) / NK] * Yf[(j + q) % NK];
                if (peers != (1u << lane)) {   // rare: several lanes, one destination
                    float a[4] = {0.f, 0.f, 0.f, 0.f};
                    for (unsigned rest = peers; rest; rest &= rest - 1) {
                        const int p = __ffs(rest) - 1;
#pragma unroll
                        for (int q = 0; q < 4; ++q) a[q] += __shfl_sync(peers, v[q], p);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) v[q] = a[q];
                }
                if (lead)
                    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + j),
                                 "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3])
                                 : "memory");
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < NBMAX * NK; ++j) {
            if (j < nb * NK) {
                float v = c[j / NK] * Yf[j % NK];
                if (peers != (1u << lane)) {
                    float a = 0.f;
                    for (unsigned rest = peers; rest; rest &= rest - 1) a += __shfl_sync(peers, v, __ffs(rest) - 1);
                    v = a;
                }
                if (lead) atomicAdd(dst + j, v);
            }
        }
    }
}

// One listener arrival of order `order` (reflections before it) at path
// length `dist` from arrival direction (ux,uy,uz) with per-band energies c[]:
// order 0 -> Dir, 1..er_max_order -> early-reflection list (when enabled),
// otherwise the SH histogram bin of dist.
template <int NBMAX, int ORDER>
__device__ __forceinline__ void commit_arrival(const TraceParams& P, int src, int order, int tri0,
                                               int tri1, double dist, double ux, double uy, double uz,
                                               const float* c, LaneStats& ls) {
    constexpr int NK = (ORDER + 1) * (ORDER + 1);
    const int nb = P.nb;
    ls.c[EF_ST_ARRIVALS]++;
    float* dst = nullptr;
    if (order == 0) {
        ls.c[EF_ST_DIRECT]++;
        dst = peer_block(P.Dp, P, src, (size_t)nb * NK);
    } else if (order <= P.er_max_order) {
        const unsigned int slot = atomicAdd(P.er_count, 1u);
        if (slot < (unsigned int)P.er_cap) {
            ef_er_entry& e = P.er[slot];
            e.src = src;
            e.order = order;
            e.tri0 = tri0;
            e.tri1 = tri1;
            e.dist = dist;
            e.dir[0] = (float)ux;
            e.dir[1] = (float)uy;
            e.dir[2] = (float)uz;
#pragma unroll
            for (int b = 0; b < 8; ++b) e.energy[b] = b < nb ? c[b] : 0.f;
        }
        return;
    } else {
        const double q = dist / P.bin_len;
        if (q < (double)P.n_bins)
            dst = peer_block(P.Hp, P, src, (size_t)P.n_bins * nb * NK) + (size_t)q * nb * NK;
        else
            ls.c[EF_ST_DROPPED]++;
    }
    if (dst) {
        double Y[NK];
        eval_sh<ORDER>(ux, uy, uz, Y);
        float Yf[NK];
#pragma unroll
        for (int k = 0; k < NK; ++k) Yf[k] = (float)Y[k];
        commit_splat<NBMAX, NK>(P, dst, c, Yf);
    }
}

// Per-path state of the bounce loop (one path per lane, or one per lane
// group with identical copies on the group's lanes).
template <int NBMAX>
struct PathState {
    double ox, oy, oz, dx, dy, dz, plen;
    float E[NBMAX];
    uint32_t ray, skey;
    int src, nrefl, nseg, tri0, tri1;
    bool last_diffuse, active;
    unsigned long long path, t_start;
};

// Lane-group geometry: G lanes (a power of two dividing 32) share one path.
struct LaneGroup {
    int gl;          // rank in the group
    int gbase;       // warp lane of the group's rank 0
    unsigned gmask;  // the group's lanes
    bool lead;       // rank 0: commits arrivals, counters and records
};

template <int G>
__device__ __forceinline__ LaneGroup lane_group() {
    LaneGroup g;
    const int lane = threadIdx.x & 31;
    g.gl = lane & (G - 1);
    g.gbase = lane - g.gl;
    g.gmask = G == 32 ? kFull : ((1u << G) - 1u) << g.gbase;
    g.lead = g.gl == 0;
    return g;
}

// The parts of a segment that do not depend on its hit, computed ahead by
// the tail kernel's warp 0 while the other warps sweep: the listener test's
// dot products and this lane's Philox draw for the reflection (same
// expressions as finish_segment's, so the same bits).
struct SegPre {
    double tc, dist2;
    uint4 xg;
};

// The rest of a segment once its closest hit h is known: listener sphere and
// SH histogram commit -> reflection.  With G > 1 the
// group's lanes split the Philox draws (and diffuse-rain shadow rays on the
// all-pairs path); everything else runs identically on each lane of the group.
template <int NBMAX, int ORDER, bool BRUTE, int THREADS, int G, bool SSTACK, bool FEAT = true>
__device__ __forceinline__ void finish_segment(const TraceParams& P, PathState<NBMAX>& S, LaneStats& ls,
                                               const Hit h, const double* s_tri, uint2* s_stack,
                                               const LaneGroup& lg, const SegPre* pre = nullptr);

// One segment of an active path: closest hit, then finish_segment.  With
// G > 1 the group's lanes split the closest hit's triangle tests.
template <int NBMAX, int ORDER, bool BRUTE, int THREADS, int G, bool SSTACK, bool FEAT>
__device__ __forceinline__ void trace_segment(const TraceParams& P, PathState<NBMAX>& S, LaneStats& ls,
                                              const double* s_tri, uint2* s_stack,
                                              const LaneGroup& lg) {
    const int gl = lg.gl;
    // ---- closest hit (exact f64 leaf test)
    Hit h;
    if (BRUTE) {
        if (G > 1)
            h = closest_brute_group<G>(s_tri, P.n_tri, S.ox, S.oy, S.oz, S.dx, S.dy, S.dz, kRayEps,
                                       INFINITY, lg.gmask, gl);
        else
            h = closest_brute(s_tri, P.n_tri, S.ox, S.oy, S.oz, S.dx, S.dy, S.dz, kRayEps, INFINITY);
        ls.c[EF_ST_TRIS] += P.n_tri;
    } else {
        h = closest_bvh_column<THREADS, kSplitDepth<THREADS>, SSTACK>(
            P.nodes, P.tris, S.ox, S.oy, S.oz, S.dx, S.dy, S.dz, kRayEps, INFINITY, ls.c[EF_ST_NODES],
            ls.c[EF_ST_TRIS], s_stack);
    }
    finish_segment<NBMAX, ORDER, BRUTE, THREADS, G, SSTACK, FEAT>(P, S, ls, h, s_tri, s_stack, lg);
}

template <int NBMAX, int ORDER, bool BRUTE, int THREADS, int G, bool SSTACK, bool FEAT>
__device__ __forceinline__ void finish_segment(const TraceParams& P, PathState<NBMAX>& S, LaneStats& ls,
                                               const Hit h, const double* s_tri, uint2* s_stack,
                                               const LaneGroup& lg, const SegPre* pre) {
    const int nb = P.nb;
    const int gl = lg.gl;
    const bool lead = lg.lead;
    const bool hit = h.id != INT32_MAX;
    EF_PHASE_T0(tsh);
    if (FEAT && P.path_ids && !P.timing && lead) P.path_ids[S.path * P.max_bounces + S.nseg] = hit ? h.id : -1;

    // ---- listener sphere receiver + SH histogram commit (with diffuse
    // rain, segments leaving a diffuse bounce reach the listener only
    // through the next-event connection: SPEC.md:257, no double count)
    if (!(FEAT && P.rain && S.last_diffuse)) {
        const double Lx = P.lx - S.ox, Ly = P.ly - S.oy, Lz = P.lz - S.oz;
        const double tc = pre ? pre->tc : dot3(Lx, Ly, Lz, S.dx, S.dy, S.dz);
        const double tlim = hit ? h.t : INFINITY;
        if (tc > 0.0 && tc < tlim) {
            const double dist2 = pre ? pre->dist2 : dot3(Lx, Ly, Lz, Lx, Ly, Lz);
            const double perp2 = dist2 - tc * tc;
            if (perp2 <= P.r2 && lead)
                commit_arrival<NBMAX, ORDER>(P, S.src, S.nrefl, FEAT ? S.tri0 : -1, FEAT ? S.tri1 : -1, S.plen + tc, -S.dx,
                                             -S.dy, -S.dz, S.E, ls);
        }
    }
    ++S.nseg;
    ls.c[EF_ST_SEGMENTS]++;
    if (!hit) {
        ls.c[EF_ST_ESCAPED]++;
        S.active = false;
    } else {
        // ---- reflection
#ifdef EF_PROFILE_PHASES
        const long long fa = clock64();   // tail profile (G == 32): listener part
        if (G == 32 && lead) atomicAdd(&g_phase[0], (unsigned long long)(fa - tsh));
#endif
        const double t = h.t;
        S.plen += t;
        ls.sum_t += t;
        S.ox = S.ox + t * S.dx;
        S.oy = S.oy + t * S.dy;
        S.oz = S.oz + t * S.dz;
        ++S.nrefl;
        if (FEAT) {   // (the ER list's first two reflectors)
            if (S.nrefl == 1) S.tri0 = h.id;
            if (S.nrefl == 2) S.tri1 = h.id;
        }
        ls.c[EF_ST_REFLECTIONS]++;
        // one 48-byte shading record, one level of loads: normal, p_m, material
#if EF_SHADE64
        const GpuShade* rec = P.shade + h.id;
        D4 r01;
        asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r01.x), "=d"(r01.y), "=d"(r01.z), "=d"(r01.w) : "l"(rec));
        const int m = __ldg(&rec->m);
        const double nx = r01.x, ny = r01.y, nz = r01.z, pdiff = r01.w;
#else
        const double2* rec = reinterpret_cast<const double2*>(P.shade + h.id);
        const double2 r0 = __ldg(rec + 0), r1 = __ldg(rec + 1);
        const int m = __ldg(reinterpret_cast<const int*>(rec + 2));
        const double nx = r0.x, ny = r0.y, nz = r1.x, pdiff = r1.y;
#endif
        double u1, u2;
        uint4 xg;   // lane groups: this lane's draw (ray, bounce, gl) -- all of a
                    // group's draws come from one Philox latency instead of a chain
        if (G > 1) {
            xg = pre ? pre->xg
                     : philox(make_uint4(S.ray, (uint32_t)S.nrefl, (uint32_t)gl, P.frame),
                              make_uint2(P.seed, S.skey));
            u1 = u53(__shfl_sync(lg.gmask, xg.x, 0, G), __shfl_sync(lg.gmask, xg.y, 0, G));
        } else {
            draw2(S.ray, (uint32_t)S.nrefl, 0u, P.frame, P.seed, S.skey, u1, u2);
        }
        const bool diffuse = u1 < pdiff;
        const double nd = dot3(nx, ny, nz, S.dx, S.dy, S.dz);
#ifdef EF_PROFILE_PHASES
        const long long fb = clock64();   // shading record + draws
        if (G == 32 && lead) atomicAdd(&g_phase[1], (unsigned long long)(fb - fa));
#endif
        if (FEAT && P.rain && diffuse) {
            // ---- diffuse rain: connect this bounce to the listener
            // centre; Lambertian lobe through the receiver cross-section:
            // c_b = E_b (1-a_b) s_b cos(theta) r^2 / d^2
            const double sg = nd > 0.0 ? -1.0 : 1.0;   // normal facing the incoming side
            const double Lx = P.lx - S.ox, Ly = P.ly - S.oy, Lz = P.lz - S.oz;
            const double d2 = dot3(Lx, Ly, Lz, Lx, Ly, Lz);
            const double dd = sqrt(d2);
            const double cosv = dot3(sg * nx, sg * ny, sg * nz, Lx, Ly, Lz) / dd;
            if (cosv > 0.0 && dd > kRayEps) {
                const double ex = Lx / dd, ey = Ly / dd, ez = Lz / dd;
                const double limit = dd - kRayEps;
                Hit sh;
                if (BRUTE) {
                    if (G > 1)
                        sh = closest_brute_group<G>(s_tri, P.n_tri, S.ox, S.oy, S.oz, ex, ey, ez,
                                                    kRayEps, limit, lg.gmask, gl);
                    else
                        sh = closest_brute(s_tri, P.n_tri, S.ox, S.oy, S.oz, ex, ey, ez, kRayEps, limit);
                } else {
                    if constexpr (G == 1)   // trace kernels: this thread's stack column
                        sh = closest_bvh_column<THREADS, kSplitDepth<THREADS>, SSTACK>(
                            P.nodes, P.tris, S.ox, S.oy, S.oz, ex, ey, ez, kRayEps, limit,
                            ls.c[EF_ST_NODES], ls.c[EF_ST_TRIS], s_stack, true);
                    else {                  // tail kernel (a whole CTA per path): local stack
                        StackLocal ls_st;
                        ls_st.sp = 0;
                        sh = closest_bvh(P.nodes, P.tris, S.ox, S.oy, S.oz, ex, ey, ez, kRayEps, limit,
                                         ls.c[EF_ST_NODES], ls.c[EF_ST_TRIS], ls_st, true);
                    }
                }
                if (sh.id == INT32_MAX && lead) {
                    const float gf = (float)(cosv * P.r2 / d2);
                    float c[NBMAX];
#pragma unroll
                    for (int b = 0; b < NBMAX; ++b)
                        c[b] = b < nb ? S.E[b] * __ldg(P.fr + m * nb + b) * gf : 0.f;
                    commit_arrival<NBMAX, ORDER>(P, S.src, S.nrefl, FEAT ? S.tri0 : -1, FEAT ? S.tri1 : -1, S.plen + dd, -ex,
                                                 -ey, -ez, c, ls);
                }
            }
        }
        S.last_diffuse = diffuse;
        const float* f = (diffuse ? P.fd : P.fs) + m * nb;
        // one vector load per row when it is a whole aligned row (nb = 4 or
        // 8: the tables are cudaMalloc'ed, rows nb floats apart)
        if (NBMAX == 8 && nb == 8) {
            const F8 r = ldg_f8(f);
            S.E[0] *= r.a; S.E[1] *= r.b; S.E[2] *= r.c; S.E[3] *= r.d;
            if constexpr (NBMAX == 8) { S.E[4] *= r.e; S.E[5] *= r.f; S.E[6] *= r.g; S.E[7] *= r.h; }
        } else if (nb == 4) {
            const float4 r = __ldg(reinterpret_cast<const float4*>(f));
            S.E[0] *= r.x; S.E[1] *= r.y; S.E[2] *= r.z; S.E[3] *= r.w;
        } else {
#pragma unroll
            for (int b = 0; b < NBMAX; ++b)
                if (b < nb) S.E[b] = S.E[b] * __ldg(f + b);
        }
        if (diffuse) {
            const double s = nd > 0.0 ? -1.0 : 1.0;
            // basis of the normal facing the incoming side (a precomputed
            // per-triangle basis in a 128-byte record measured slower: C2
            // 1.31 vs 1.33, C5 3.29 vs 3.39 G seg/s -- cache footprint)
            double t1[3], t2[3];
            duff_onb(s * nx, s * ny, s * nz, t1, t2);
            if (G > 1) {
                // disk candidate j = gl - 1 on lanes 1..G-1; the first accepted
                // one (lowest j) is the sequential loop's answer
                const double a = 2.0 * u53(xg.x, xg.y) - 1.0;
                const double b = 2.0 * u53(xg.z, xg.w) - 1.0;
                const double ss = a * a + b * b;
                const unsigned ok = __ballot_sync(lg.gmask, gl >= 1 && ss < 1.0);
                if (ok) {
                    const int f = __ffs(ok) - 1 - lg.gbase;
                    cosine_dir(__shfl_sync(lg.gmask, a, f, G), __shfl_sync(lg.gmask, b, f, G),
                               __shfl_sync(lg.gmask, ss, f, G), s * nx, s * ny, s * nz, t1, t2, S.dx,
                               S.dy, S.dz);
                } else {
                    sample_cosine(P.seed, S.skey, S.ray, (uint32_t)S.nrefl, P.frame, s * nx, s * ny,
                                  s * nz, t1, t2, S.dx, S.dy, S.dz, (uint32_t)(G - 1));
                }
            } else {
                sample_cosine(P.seed, S.skey, S.ray, (uint32_t)S.nrefl, P.frame, s * nx, s * ny,
                              s * nz, t1, t2, S.dx, S.dy, S.dz);
            }
        } else {
            const double k2 = 2.0 * nd;
            S.dx = S.dx - k2 * nx;
            S.dy = S.dy - k2 * ny;
            S.dz = S.dz - k2 * nz;
        }
        if (S.nrefl >= P.max_bounces) S.active = false;
#ifdef EF_PROFILE_PHASES
        if (G == 32 && lead) atomicAdd(&g_phase[2], (unsigned long long)(clock64() - fb));   // direction
#endif
    }
    EF_PHASE_ADD(3, tsh);
#ifdef EF_PROFILE_PHASES
    if (lead) atomicAdd(&g_phase[4], 1ull);
#endif
    if (FEAT && !S.active && P.path_nseg && lead) P.path_nseg[S.path] = S.nseg;
    if (FEAT && P.timing && lead && 5 + S.nseg < P.max_bounces)   // debug: ns since path start, per segment
        P.path_ids[S.path * P.max_bounces + 5 + S.nseg] = (int32_t)(globaltimer() - S.t_start);
    if (FEAT && !S.active && P.timing && lead) {
        const unsigned long long t_end = globaltimer();
        int32_t* row = P.path_ids + S.path * P.max_bounces;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        row[0] = (int32_t)(S.t_start & 0xffffffffu);
        row[1] = (int32_t)(S.t_start >> 32);
        row[2] = (int32_t)(t_end & 0xffffffffu);
        row[3] = (int32_t)(t_end >> 32);
        row[4] = (int32_t)smid;
        row[5] = S.nseg;
    }
}

// Persistent trace kernel: lanes (or lane groups) take paths from a global
// counter and run them segment by segment.
// G > 1 (all-pairs scenes with few paths, C1): G lanes share one path, split
// its triangle tests (closest_brute_group) and otherwise run identical,
// deterministic path code; the group's first lane alone commits arrivals,
// counters and records.
// (A tail mode that compacted a warp's last <= 8 paths into 4-lane groups
// splitting leaf tests and draws measured slower on C2/C3/C5 -- spills in
// the shared loop -- and was removed.)
// SSTACK: the whole traversal stack in shared memory (P.smem_stack >= the
// tree's max_stack), predicated pushes.
// CTAs per SM of the split-stack kernel (tuning builds: EF_BIG_CTAS with
// EF_BIG_THREADS = 1024 / EF_BIG_CTAS)
#ifndef EF_BIG_CTAS
#define EF_BIG_CTAS 1
#endif
template <bool BRUTE, bool SSTACK>
constexpr int kCtasPerSm = (!BRUTE && !SSTACK) ? EF_BIG_CTAS : 1;

template <int NBMAX, int ORDER, bool BRUTE, int THREADS, int G = 1, bool SSTACK = false, bool FEAT = true>
__global__ void __launch_bounds__(THREADS, (kCtasPerSm<BRUTE, SSTACK>)) trace_kernel(const TraceParams P_in) {
    const TraceParams& P = P_in;
    static_assert(G >= 1 && G <= 32 && (G & (G - 1)) == 0, "G must be a power of two <= 32");
    static_assert(G == 1 || BRUTE, "lane groups are for the all-pairs path");
    pdl_trigger();   // the tail / analysis kernel may be scheduled onto SMs this grid frees
    extern __shared__ __align__(16) unsigned char smem[];
    // traversal stacks first (P.smem_stack entries per thread, i-major), so a
    // thread's column address is the shared symbol + 8 * threadIdx.x -- cheap
    // to keep or rematerialise (derived through a 64-bit generic pointer it
    // was rebuilt from the shared window base on every pop: ~13% of the C5
    // kernel's instructions, r02c source counters); then the per-block
    // counters (f64 path-length sums, u32 counters: a block's per-source
    // counts stay far below 2^32) and the all-pairs triangles
    uint2* s_stack = reinterpret_cast<uint2*>(smem);
    if constexpr (!BRUTE) {   // the stacks address their columns from this constant
        if ((uint32_t)__cvta_generic_to_shared(smem) != kDynSmemBase) __trap();
    }
    const uint32_t stack_bytes = BRUTE ? 0u : (uint32_t)P.smem_stack * THREADS * 8u;
    double* s_sumt = reinterpret_cast<double*>(smem + stack_bytes);
    unsigned int* s_stats = reinterpret_cast<unsigned int*>(s_sumt + P.n_src);
    double* s_tri = reinterpret_cast<double*>(
        smem + ((stack_bytes + 8u * P.n_src + 4u * P.n_src * EF_ST_COUNT + 15u) & ~15u));
    for (int i = threadIdx.x; i < P.n_src * EF_ST_COUNT; i += blockDim.x) s_stats[i] = 0u;
    for (int i = threadIdx.x; i < P.n_src; i += blockDim.x) s_sumt[i] = 0.0;
    if (BRUTE)
        for (int i = threadIdx.x; i < 9 * P.n_tri; i += blockDim.x) s_tri[i] = P.tris_by_id[i];
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const LaneGroup lg = lane_group<G>();
    LaneStats ls;
    bool exhausted = false;
    PathState<NBMAX> S;
    S.ox = S.oy = S.oz = S.dx = S.dy = S.plen = 0.0;
    S.dz = 1.0;
#pragma unroll
    for (int b = 0; b < NBMAX; ++b) S.E[b] = 0.f;
    S.ray = S.skey = 0;
    S.src = S.nrefl = S.nseg = 0;
    S.tri0 = S.tri1 = -1;
    S.last_diffuse = S.active = false;
    S.path = S.t_start = 0;

    bool fin = false;                    // this lane's path ended in the last segment
    unsigned long long done_seen = 0;    // P.done as read one iteration earlier
    for (;;) {
        // ---- tail hand-off (P.tail_live > 0): count finished paths; once
        // the path counter is exhausted and at most tail_live paths are
        // unfinished, the warp's live paths move to the continuation list
        // for tail_kernel, which runs each on a whole CTA
        if (SSTACK && P.tail_live > 0) {   // (ef_trace.cu: tail_live = 0 for the other kernels)
            const unsigned fm = __ballot_sync(kFull, fin);
            if (fm && lane == __ffs(fm) - 1) atomicAdd(P.done, (unsigned long long)__popc(fm));
            fin = false;
            if (__any_sync(kFull, exhausted)) {
                if (S.active && P.total - done_seen <= (unsigned long long)P.tail_live) {
                    // paths already long go first (the frame's critical chain
                    // starts at once), the rest fill the list from its end
                    const bool lng = S.nseg >= kTailLongSegs;
                    const unsigned k = atomicAdd(P.cont_count + (lng ? 0 : 1), 1u);
                    const unsigned slot = lng ? k : (unsigned)P.tail_live - 1u - k;
                    if (k < (unsigned)P.tail_live) {   // always: at most tail_live paths are unfinished
                        reinterpret_cast<PathState<NBMAX>*>(P.cont)[slot] = S;
                        S.active = false;
                    }
                }
                done_seen = *reinterpret_cast<volatile unsigned long long*>(P.done);   // used next iteration
            }
        }
        // ---- warp-aggregated refill: idle lanes take the next path indices
        // (lane groups: only group leads count; a group's lanes share its
        // lead's path index)
        const bool need = !S.active && !exhausted;
        const unsigned mask = __ballot_sync(kFull, need && lg.lead);
        if (mask) {
            const int leader = __ffs(mask) - 1;
            const unsigned rank = __popc(mask & ((1u << lg.gbase) - 1u));
            unsigned long long my;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(P.counter, (unsigned long long)__popc(mask));
            my = __shfl_sync(kFull, base, leader) + rank;
            if (need) {
                S.path = my;
                if (S.path >= P.total) {
                    exhausted = true;
                } else {
                    S.src = (int)(S.path / (unsigned long long)P.n_rays);
                    const int64_t local = (int64_t)(S.path - (unsigned long long)S.src * P.n_rays);
                    S.ray = P.ray_ids ? __ldg(P.ray_ids + local) : P.ray0 + (uint32_t)local;
                    S.skey = P.src_key ? __ldg(P.src_key + S.src) : (uint32_t)S.src;
                    S.ox = __ldg(P.src_pos + 3 * S.src + 0);
                    S.oy = __ldg(P.src_pos + 3 * S.src + 1);
                    S.oz = __ldg(P.src_pos + 3 * S.src + 2);
                    sample_sphere(P.seed, S.skey, S.ray, P.frame, S.dx, S.dy, S.dz);
#pragma unroll
                    for (int b = 0; b < NBMAX; ++b) S.E[b] = P.e0;
                    S.plen = 0.0;
                    S.nrefl = 0;
                    S.nseg = 0;
                    S.tri0 = S.tri1 = -1;
                    S.last_diffuse = false;
                    if (S.src != ls.src) {
                        if (lg.lead) flush_stats(ls, s_stats, s_sumt);   // other group lanes' counts are dropped
                        ls.src = S.src;
                    }
                    ls.c[EF_ST_PATHS]++;
                    if (FEAT && P.timing) S.t_start = globaltimer();
                    S.active = true;
                }
            }
        }
        // (ballot + test: measured 5% faster on C2 than the equivalent
        // __all_sync(!active) exit -- the compiler lays the loop out better)
        const unsigned live = __ballot_sync(kFull, S.active);
        if (!live) break;
#ifndef EF_PROFILE_PHASES
        if (!S.active) continue;
        trace_segment<NBMAX, ORDER, BRUTE, THREADS, G, SSTACK, FEAT>(P, S, ls, s_tri, s_stack, lg);
#else
        const uint32_t n0 = ls.c[EF_ST_NODES], t0 = ls.c[EF_ST_TRIS];
        const bool was = S.active;
        if (S.active) trace_segment<NBMAX, ORDER, BRUTE, THREADS, G, SSTACK, FEAT>(P, S, ls, s_tri, s_stack, lg);
        {   // SIMT cost of per-lane traversal lengths: 5 sum of node visits,
            // 6 sum over warp-segments of max visits x 32, 7 the same for
            // triangle tests (8 their sum), 9 segments (active lanes)
            const uint32_t dn = was ? ls.c[EF_ST_NODES] - n0 : 0u, dt = was ? ls.c[EF_ST_TRIS] - t0 : 0u;
            const uint32_t sn = __reduce_add_sync(kFull, dn), mn = __reduce_max_sync(kFull, dn);
            const uint32_t st = __reduce_add_sync(kFull, dt), mt = __reduce_max_sync(kFull, dt);
            const uint32_t na = __popc(__ballot_sync(kFull, was));
            if (lane == 0) {
                atomicAdd(&g_phase[5], (unsigned long long)sn);
                atomicAdd(&g_phase[6], 32ull * mn);
                atomicAdd(&g_phase[7], 32ull * mt);
                atomicAdd(&g_phase[8], (unsigned long long)st);
                atomicAdd(&g_phase[9], (unsigned long long)na);
            }
        }
        if (!was) continue;
#endif
        fin = !S.active;
    }
    if (lg.lead) flush_stats(ls, s_stats, s_sumt);

    __syncthreads();
    for (int i = threadIdx.x; i < P.n_src * EF_ST_COUNT; i += blockDim.x)
        if (s_stats[i]) atomicAdd(P.stats + i, (unsigned long long)s_stats[i]);
    for (int i = threadIdx.x; i < P.n_src; i += blockDim.x)
        if (s_sumt[i] != 0.0) atomicAdd(P.sum_t + i, s_sumt[i]);
}

// Tail of a frame (scenes of <= kTailMaxTris triangles): the paths handed off
// by trace_kernel run one per CTA, long ones first.  Every segment's closest
// hit is the all-pairs answer (lowest id on equal t -- the same hit as the
// BVH's) split over warps 1-15: f32 slab tests of cluster
// boxes (16 leaf-order triangles each), then of the crossed clusters'
// triangle boxes (all padded and rounded outward like the BVH's leaf boxes,
// so conservative) pick the candidates, the exact f64 test decides, and two
// shared-memory atomics reduce (t, id).  Warp 0 meanwhile computes the
// segment's hit-independent work and then finishes it as a 32-lane group
// (parallel draws).  A lone path's segment drops from a serial BVH walk
// (~3.2 us on C2) to ~2.0 us.
#ifndef EF_TAIL_THREADS
#define EF_TAIL_THREADS 512
#endif
constexpr int kTailThreads = EF_TAIL_THREADS;   // (tuning builds may override)

// Triangle boxes staged in shared memory (32 B each, all of a <= 4,096-
// triangle scene); the f64 triangles stay in L1 (staging them instead --
// 72 B each -- shrinks L1 below the boxes' working set: 3.05 vs 2.44 us per
// segment on C2).
constexpr size_t kTailStageBytes = (size_t)kTailMaxTris * 32 + (size_t)kTailThreads * 32 +
                                   (size_t)kTailThreads * kTailCluster * 4;

template <int NBMAX, int ORDER>
__global__ void __launch_bounds__(kTailThreads, 1) tail_kernel(const TraceParams P) {
    extern __shared__ __align__(16) float4 s_box[];   // (n_tri, 2) padded triangle boxes
    __shared__ unsigned long long s_tb;   // closest t (bits of a positive double: ordered as u64)
    __shared__ int s_id;                  // lowest id at that t
    __shared__ int s_nc;                  // exact tests of the segment (counter EF_ST_TRIS)
    __shared__ double s_ray[6];
    __shared__ int s_active;
    __shared__ unsigned s_j;
    __shared__ int s_hitc[kTailThreads];   // clusters whose box the ray crosses
    __shared__ int s_nhit;
    constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    pdl_trigger();
    const PathState<NBMAX>* cont = reinterpret_cast<const PathState<NBMAX>*>(P.cont);
    const LaneGroup lg = lane_group<32>();
    // shared: triangle boxes by id, cluster boxes, leaf-order ids
    float4* s_cbox = s_box + 2 * P.n_tri;
    int* s_cid = reinterpret_cast<int*>(s_cbox + 2 * P.n_clu);
    {
        const float4* src = reinterpret_cast<const float4*>(P.tri_box);
#pragma unroll 4
        for (int k = tid; k < 2 * P.n_tri; k += kTailThreads) s_box[k] = __ldg(src + k);
        const float4* csrc = reinterpret_cast<const float4*>(P.clu_box);
        for (int k = tid; k < 2 * P.n_clu; k += kTailThreads) s_cbox[k] = __ldg(csrc + k);
        for (int k = tid; k < P.n_refs; k += kTailThreads) s_cid[k] = __ldg(P.clu_ids + k);
    }
    pdl_wait();   // (staged while the trace kernel drained) its hand-offs are final from here
    const unsigned n_long = min(P.cont_count[0], (unsigned)P.tail_live);
    const unsigned n = min(n_long + P.cont_count[1], (unsigned)P.tail_live);
    if (blockIdx.x >= n) return;   // no path for this CTA
    const double* tris = P.tris_by_id;
    if (tid == 0) {
        s_tb = kInfBits;
        s_id = INT32_MAX;
        s_nc = 0;
        s_nhit = 0;
    }
    for (;;) {
        if (tid == 0) s_j = atomicAdd(P.cont_take, 1u);
        __syncthreads();
        const unsigned j = s_j;
        __syncthreads();
        if (j >= n) break;
        // long paths first (front of the list), then the short ones (back)
        PathState<NBMAX> S = cont[j < n_long ? j : (unsigned)P.tail_live - 1u - (j - n_long)];
        LaneStats ls;
        ls.src = S.src;
        bool active = S.active;
        double ox = S.ox, oy = S.oy, oz = S.oz, dx = S.dx, dy = S.dy, dz = S.dz;
        while (active) {
#ifdef EF_PROFILE_PHASES
            const long long c0 = clock64();
#endif
            // ---- candidates by box, exact test, (t, id) minimum over the CTA
            const RayF r = make_rayf(ox, oy, oz, dx, dy, dz);
            const float tminf = fmaxf(__double2float_rd(kRayEps), 0.0f);
            Hit h{INFINITY, INT32_MAX};
            int nc = 0;
            // warp 0: the hit-independent part of finish_segment; warps 1..15:
            // the sweep
            SegPre pre;
            if (w == 0) {
                const double Lx = P.lx - S.ox, Ly = P.ly - S.oy, Lz = P.lz - S.oz;
                pre.tc = dot3(Lx, Ly, Lz, S.dx, S.dy, S.dz);
                pre.dist2 = dot3(Lx, Ly, Lz, Lx, Ly, Lz);
                pre.xg = philox(make_uint4(S.ray, (uint32_t)(S.nrefl + 1), (uint32_t)lane, P.frame),
                                make_uint2(P.seed, S.skey));
            }
            constexpr int kSweep = kTailThreads - 32;
            const int st = tid - 32;   // sweep thread index (warp 0: none)
            // level 1: the clusters (unions of 16 leaf-order triangle boxes)
            for (int c = st; c >= 0 && c < P.n_clu; c += kSweep) {
                const float4 a = s_cbox[2 * c], b = s_cbox[2 * c + 1];
                if (slab_key_minmax(r, a.x, a.w, a.y, b.x, a.z, b.y, tminf, 1e38f, 0u) != 0xffffffffu)
                    s_hitc[atomicAdd(&s_nhit, 1)] = c;
            }
            __syncthreads();
            // level 2: the triangles of the crossed clusters, one per thread
            const int nh = s_nhit;
            for (int q = st; q >= 0 && q < nh * kTailCluster; q += kSweep) {
                const int ref = s_hitc[q / kTailCluster] * kTailCluster + q % kTailCluster;
                if (ref >= P.n_refs) continue;
                const int i = s_cid[ref];
                const float4 a = s_box[2 * i], b = s_box[2 * i + 1];
                if (slab_key_minmax(r, a.x, a.w, a.y, b.x, a.z, b.y, tminf, 1e38f, 0u) == 0xffffffffu)
                    continue;
                ++nc;
                double t;   // any order: (t, id) compared lexicographically
                if (mt_hit(ox, oy, oz, dx, dy, dz, tris + 9 * i, kRayEps, INFINITY, t) &&
                    (t < h.t || (t == h.t && i < h.id))) {
                    h.t = t;
                    h.id = i;
                }
            }
#ifdef EF_PROFILE_PHASES
            const long long c1 = clock64();
#endif
            nc = __reduce_add_sync(kFull, nc);
            if (h.id != INT32_MAX) atomicMin(&s_tb, (unsigned long long)__double_as_longlong(h.t));
            if (lane == 0 && nc) atomicAdd(&s_nc, nc);
            __syncthreads();
            const unsigned long long tb = s_tb;
            if (h.id != INT32_MAX && (unsigned long long)__double_as_longlong(h.t) == tb)
                atomicMin(&s_id, h.id);
            __syncthreads();
#ifdef EF_PROFILE_PHASES
            const long long c2 = clock64();
#endif
            if (w == 0) {
                if (tb != kInfBits) {
                    h.t = __longlong_as_double((long long)tb);
                    h.id = s_id;
                } else {
                    h.t = INFINITY;
                    h.id = INT32_MAX;
                }
                ls.c[EF_ST_TRIS] += (uint32_t)s_nc;
                ls.c[EF_ST_TAIL]++;
                finish_segment<NBMAX, ORDER, false, kTailThreads, 32, false>(P, S, ls, h, nullptr, nullptr, lg,
                                                                             &pre);
                if (lane == 0) {
                    s_ray[0] = S.ox; s_ray[1] = S.oy; s_ray[2] = S.oz;
                    s_ray[3] = S.dx; s_ray[4] = S.dy; s_ray[5] = S.dz;
                    s_active = S.active;
                    s_tb = kInfBits;
                    s_id = INT32_MAX;
                    s_nc = 0;
                    s_nhit = 0;
                }
            }
#ifdef EF_PROFILE_PHASES
            const long long c3 = clock64();
#endif
            __syncthreads();
#ifdef EF_PROFILE_PHASES
            if (tid == 0) {   // 8 sweep, 9 reduction, 10 finish_segment, 11 broadcast barrier
                atomicAdd(&g_phase[8], (unsigned long long)(c1 - c0));
                atomicAdd(&g_phase[9], (unsigned long long)(c2 - c1));
                atomicAdd(&g_phase[10], (unsigned long long)(c3 - c2));
                atomicAdd(&g_phase[11], (unsigned long long)(clock64() - c3));
            }
#endif
            ox = s_ray[0]; oy = s_ray[1]; oz = s_ray[2];
            dx = s_ray[3]; dy = s_ray[4]; dz = s_ray[5];
            active = s_active != 0;
        }
        if (tid == 0 && ls.src >= 0) {
#pragma unroll
            for (int i = 0; i < EF_ST_COUNT; ++i)
                if (ls.c[i]) atomicAdd(P.stats + ls.src * EF_ST_COUNT + i, (unsigned long long)ls.c[i]);
            if (ls.sum_t != 0.0) atomicAdd(P.sum_t + ls.src, ls.sum_t);
        }
    }
}

// ---------------------------------------------------------------------------
static int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    }
    return n;
}

template <int NBMAX, int ORDER, bool BRUTE, int THREADS, int G = 1, bool SSTACK = false, bool FEAT = true>
static cudaError_t launch_trace(const TraceParams& P0, cudaStream_t st) {
    TraceParams P = P0;
    if (!SSTACK) P.smem_stack = kSplitDepth<THREADS>;   // else: the tree's max_stack
    // Too few paths to give every SM a full CTA (C1: 4,096 paths): spread them
    // over all SMs in smaller CTAs (>= one warp), so each path's latency-bound
    // chain shares its SM with as few others as possible.
    const long long sms = (long long)sm_count() * kCtasPerSm<BRUTE, SSTACK>;
    const long long lanes = (long long)P.total * G;
    static const int block_env = [] {   // tuning only: threads per CTA (<= THREADS)
        const char* e = std::getenv("EF_BLOCK");
        return e ? std::atoi(e) : 0;
    }();
    int block = (block_env >= 32 && block_env <= THREADS) ? block_env / 32 * 32 : THREADS;
    if (lanes < sms * THREADS) {
        const long long per = (lanes + sms - 1) / sms;
        block = (int)std::min<long long>(THREADS, std::max<long long>(32, (per + 31) / 32 * 32));
    }
    size_t smem = (size_t)P.n_src * (EF_ST_COUNT * 4 + 8) + (BRUTE ? (size_t)P.n_tri * 72 : 0) + 32 +
                  (BRUTE ? 0 : (size_t)P.smem_stack * THREADS * sizeof(uint2));   // THREADS columns
    auto kern = trace_kernel<NBMAX, ORDER, BRUTE, THREADS, G, SSTACK, FEAT>;
    static bool attr_done = false;   // once per instantiation: no per-launch host queries
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kMaxTraceSmem);
        if (e != cudaSuccess) return e;
        if (const char* c = std::getenv("EF_CARVEOUT"))   // tuning: shared-memory carve-out (percent of the SM's 228 KB)
            cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, std::atoi(c));
        attr_done = true;
    }
    if (smem > kMaxTraceSmem) return cudaErrorInvalidValue;
    // persistent grid: one CTA per SM (__launch_bounds__(THREADS, 1) and the
    // register budget leave room for exactly one), no more warps than paths
    const long long need = (lanes + block - 1) / block;
    const int grid = (int)std::max(1LL, std::min(sms, need));
    kern<<<grid, block, smem, st>>>(P);
    count_launch();
    return cudaGetLastError();
}

template <int NBMAX, bool BRUTE, int THREADS, int G = 1, bool SSTACK = false, bool FEAT = true>
static cudaError_t dispatch_order(int order, const TraceParams& P, cudaStream_t st) {
    switch (order) {
        case 0: return launch_trace<NBMAX, 0, BRUTE, THREADS, G, SSTACK, FEAT>(P, st);
        case 1: return launch_trace<NBMAX, 1, BRUTE, THREADS, G, SSTACK, FEAT>(P, st);
        case 2: return launch_trace<NBMAX, 2, BRUTE, THREADS, G, SSTACK, FEAT>(P, st);
        case 3: return launch_trace<NBMAX, 3, BRUTE, THREADS, G, SSTACK, FEAT>(P, st);
        default: return launch_trace<NBMAX, 4, BRUTE, THREADS, G, SSTACK, FEAT>(P, st);
    }
}

// Lanes per path on the all-pairs path: the widest group (<= the triangle
// count rounded up to a power of two, <= 16) whose lanes still fit one full
// CTA per SM, so a frame with few paths (C1: 4,096) spreads each path's
// triangle tests over idle lanes instead of leaving SMs empty.  EF_GROUP
// (1, 4, 8, 16) overrides (tuning).
static int brute_group(unsigned long long paths, int n_tri) {
    static const int force = [] {
        const char* e = std::getenv("EF_GROUP");
        return e ? std::atoi(e) : 0;
    }();
    if (force == 1 || force == 4 || force == 8 || force == 16) return force;
    const unsigned long long cap = (unsigned long long)sm_count() * kSmallThreads;
    int g = 16;
    while (g > 1 && ((unsigned long long)g * paths > cap || g / 2 >= n_tri)) g /= 2;
    return g == 2 ? 1 : g;   // no 2-lane instantiation
}

template <int NBMAX, int ORDER>
static cudaError_t launch_tail_o(const TraceParams& P, cudaStream_t st) {
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(tail_kernel<NBMAX, ORDER>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTailStageBytes);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    const int grid = (int)std::max(1, std::min(P.tail_live, sm_count()));
    // n_tri <= kTailMaxTris, n_clu <= kTailThreads (tail_live == 0 otherwise)
    const size_t smem = (size_t)P.n_tri * 32 + (size_t)P.n_clu * 32 + (size_t)P.n_refs * 4;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(kTailThreads);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL after trace_kernel
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&lc, tail_kernel<NBMAX, ORDER>, P);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <int NBMAX>
static cudaError_t launch_tail(int order, const TraceParams& P, cudaStream_t st) {
    switch (order) {
        case 0: return launch_tail_o<NBMAX, 0>(P, st);
        case 1: return launch_tail_o<NBMAX, 1>(P, st);
        case 2: return launch_tail_o<NBMAX, 2>(P, st);
        case 3: return launch_tail_o<NBMAX, 3>(P, st);
        default: return launch_tail_o<NBMAX, 4>(P, st);
    }
}

template <int NBMAX>
static cudaError_t dispatch_brute(int order, const TraceParams& P, cudaStream_t st) {
    switch (brute_group(P.total, P.n_tri)) {
        case 16: return dispatch_order<NBMAX, true, kSmallThreads, 16>(order, P, st);
        case 8: return dispatch_order<NBMAX, true, kSmallThreads, 8>(order, P, st);
        case 4: return dispatch_order<NBMAX, true, kSmallThreads, 4>(order, P, st);
        default: return dispatch_order<NBMAX, true, kSmallThreads>(order, P, st);
    }
}

template <int NBMAX>
static cudaError_t dispatch_bvh(bool big, int order, const TraceParams& P, cudaStream_t st) {
    (void)big;
    // FEAT = false: the production frame -- no per-path records, timing,
    // diffuse rain or ER list compiled in (their state and checks cost the
    // 64-register kernel 4.5%: C5 4.29 -> 4.49, C3 3.15 -> 3.29 G seg/s)
    const bool feat = P.path_ids || P.path_nseg || P.timing || P.rain || P.er_max_order > 0;
    if (P.smem_stack > 0)
        return feat ? dispatch_order<NBMAX, false, kSmallThreads, 1, true, true>(order, P, st)
                    : dispatch_order<NBMAX, false, kSmallThreads, 1, true, false>(order, P, st);
    return feat ? dispatch_order<NBMAX, false, kBigThreads, 1, false, true>(order, P, st)
                : dispatch_order<NBMAX, false, kBigThreads, 1, false, false>(order, P, st);
}

// Defined one per translation unit (ef_trace_{brute,bvh}_nb{4,8}.cu).
cudaError_t trace_dispatch_brute_nb4(int order, const TraceParams& P, cudaStream_t st);
cudaError_t trace_dispatch_brute_nb8(int order, const TraceParams& P, cudaStream_t st);
cudaError_t trace_dispatch_bvh_nb4(bool big, int order, const TraceParams& P, cudaStream_t st);
cudaError_t trace_dispatch_bvh_nb8(bool big, int order, const TraceParams& P, cudaStream_t st);
cudaError_t tail_dispatch_nb4(int order, const TraceParams& P, cudaStream_t st);
cudaError_t tail_dispatch_nb8(int order, const TraceParams& P, cudaStream_t st);
#ifdef EF_PROFILE_PHASES
void debug_phases_brute_nb4(unsigned long long* acc, int reset);
void debug_phases_brute_nb8(unsigned long long* acc, int reset);
void debug_phases_bvh_nb4(unsigned long long* acc, int reset);
void debug_phases_bvh_nb8(unsigned long long* acc, int reset);
#endif

}  // namespace ef

