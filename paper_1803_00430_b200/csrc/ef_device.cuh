// Device-side building blocks of the hot path (compiled with -fmad=false:
// every f64 expression below is evaluated exactly as written, matching the
// reference's numpy evaluation order bit-for-bit).
#pragma once
#include <type_traits>
#include <cstdint>
#include <cuda_runtime.h>

#include "ef_internal.h"

namespace ef {

// A/B build knob (tools/build_variant.py): nested push branches (default on)
#ifndef EF_NESTED_PUSH
#define EF_NESTED_PUSH 1
#endif
#ifndef EF_KEY_LOP3
#define EF_KEY_LOP3 1
#endif

#ifdef EF_PROFILE_PHASES
// debug builds only: clock64 cycles per phase (0 inner visits, 1 leaves,
// 2 pops after leaves, 3 shading, 4 segments)
constexpr int kPhaseSlots = 24;
#ifndef EF_SPLIT_DEPTH_PROBE
#define EF_SPLIT_DEPTH_PROBE 12   // stack depth whose crossing the probe counts ("past the shared top")
#endif
static __device__ unsigned long long g_phase[kPhaseSlots];   // per translation unit
#define EF_PHASE_T0(v) const long long v = clock64()
#define EF_PHASE_ADD(i, v) atomicAdd(&g_phase[i], (unsigned long long)(clock64() - (v)))
// traversal-stack counters (tools/probe_simt.py): 12 pushes, 13 pushes past
// the shared top, 14 pops taken, 15 pops culled by the closest hit, 16-19
// node visits that hit 0 / 1 / 2 / >= 3 children, 20 leaf visits
#define EF_STK(i) (++stk[i])
#define EF_STK_DECL uint32_t stk[9] = {}
#define EF_STK_FLUSH                                                                  \
    for (int i_ = 0; i_ < 9; ++i_)                                                    \
        if (stk[i_]) atomicAdd(&g_phase[12 + i_], (unsigned long long)stk[i_])
#else
#define EF_PHASE_T0(v)
#define EF_PHASE_ADD(i, v)
#define EF_STK(i)
#define EF_STK_DECL
#define EF_STK_FLUSH
#endif

// ------------------------------------------------ dependent launches ----
// Programmatic dependent launch (PDL): a kernel lets the next kernel on its
// stream be scheduled before it ends (pdl_trigger); the next kernel runs its
// input-independent prologue, then pdl_wait() blocks until this grid has
// completed and its memory is visible.  Both are no-ops without the launch
// attribute (launch_pdl in ef_trace.cu / ef_analyze.cu).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---------------------------------------------------------------- RNG ----
// Philox4x32-10 (Salmon et al. 2011); key = (seed, source key),
// counter = (ray, bounce, draw, frame).  DESIGN.md 3.1.
__device__ __forceinline__ uint4 philox(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
    return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ void draw2(uint32_t ray, uint32_t bounce, uint32_t draw, uint32_t frame,
                                      uint32_t seed, uint32_t src, double& u1, double& u2) {
    const uint4 x = philox(make_uint4(ray, bounce, draw, frame), make_uint2(seed, src));
    u1 = u53(x.x, x.y);
    u2 = u53(x.z, x.w);
}

// Uniform sphere direction, Marsaglia rejection.
__device__ __forceinline__ void sample_sphere(uint32_t seed, uint32_t src, uint32_t ray,
                                              uint32_t frame, double& dx, double& dy, double& dz) {
    dx = 0.0; dy = 0.0; dz = 1.0;
    for (uint32_t j = 0; j < 64u; ++j) {
        double u1, u2;
        draw2(ray, 0u, j, frame, seed, src, u1, u2);
        const double a = 2.0 * u1 - 1.0;
        const double b = 2.0 * u2 - 1.0;
        const double s = a * a + b * b;
        if (s >= 1.0) continue;
        const double f = 2.0 * sqrt(1.0 - s);
        dx = a * f;
        dy = b * f;
        dz = 1.0 - 2.0 * s;
        break;
    }
}

// Duff et al. (2017) orthonormal basis (t1, t2) of unit n.  Computed once
// per triangle (GpuShade); for the flipped normal -n the same expressions
// give (t1, -t2) exactly (every product and quotient only changes sign).
__device__ __forceinline__ void duff_onb(double nx, double ny, double nz, double* t1, double* t2) {
    const double sg = copysign(1.0, nz);
    const double aa = -1.0 / (sg + nz);
    const double bb = nx * ny * aa;
    t1[0] = 1.0 + sg * nx * nx * aa;
    t1[1] = sg * bb;
    t1[2] = -sg * nx;
    t2[0] = bb;
    t2[1] = sg + ny * ny * aa;
    t2[2] = -ny;
}

// Direction of an accepted disk point (a, b), s = a^2 + b^2 < 1, lifted to
// the cosine lobe about unit n with basis (t1, t2).
__device__ __forceinline__ void cosine_dir(double a, double b, double s, double nx, double ny,
                                           double nz, const double* t1, const double* t2,
                                           double& dx, double& dy, double& dz) {
    const double z = sqrt(1.0 - s);
    dx = (a * t1[0] + b * t2[0]) + z * nx;
    dy = (a * t1[1] + b * t2[1]) + z * ny;
    dz = (a * t1[2] + b * t2[2]) + z * nz;
}

// Cosine lobe about unit n with basis (t1, t2): disk rejection (candidate j
// from draw 1 + j, starting at candidate j0) + cosine_dir.
__device__ __forceinline__ void sample_cosine(uint32_t seed, uint32_t src, uint32_t ray,
                                              uint32_t bounce, uint32_t frame, double nx, double ny,
                                              double nz, const double* t1, const double* t2,
                                              double& dx, double& dy, double& dz, uint32_t j0 = 0) {
    dx = nx; dy = ny; dz = nz;
    for (uint32_t j = j0; j < 64u; ++j) {
        double u1, u2;
        draw2(ray, bounce, 1u + j, frame, seed, src, u1, u2);
        const double a = 2.0 * u1 - 1.0;
        const double b = 2.0 * u2 - 1.0;
        const double s = a * a + b * b;
        if (s >= 1.0) continue;
        cosine_dir(a, b, s, nx, ny, nz, t1, t2, dx, dy, dz);
        break;
    }
}

// ------------------------------------------------------ exact geometry ----
// np.einsum 3-term order (p0 + p2) + p1, no FMA.
__device__ __forceinline__ double dot3(double a0, double a1, double a2, double b0, double b1,
                                       double b2) {
    return (a0 * b0 + a2 * b2) + a1 * b1;
}

// Moeller-Trumbore exactly as bvh.py:17-27 / bvh.py:33-44.  Returns the
// barycentric-valid flag (without the t window); writes t.
__device__ __forceinline__ bool mt_exact(double ox, double oy, double oz, double dx, double dy,
                                         double dz, const double* __restrict__ v, double& t) {
    const double v0x = v[0], v0y = v[1], v0z = v[2];
    const double e1x = v[3], e1y = v[4], e1z = v[5];
    const double e2x = v[6], e2y = v[7], e2z = v[8];
    // pvec = cross(d, e2)
    const double px = dy * e2z - dz * e2y;
    const double py = dz * e2x - dx * e2z;
    const double pz = dx * e2y - dy * e2x;
    const double det = dot3(e1x, e1y, e1z, px, py, pz);
    if (!(fabs(det) > 1e-14)) return false;
    const double inv = 1.0 / det;
    const double tx = ox - v0x, ty = oy - v0y, tz = oz - v0z;
    const double u = dot3(tx, ty, tz, px, py, pz) * inv;
    if (!(u >= -1e-10)) return false;
    // qvec = cross(tvec, e1)
    const double qx = ty * e1z - tz * e1y;
    const double qy = tz * e1x - tx * e1z;
    const double qz = tx * e1y - ty * e1x;
    const double vv = dot3(qx, qy, qz, dx, dy, dz) * inv;
    if (!(vv >= -1e-10) || !(u + vv <= 1.0 + 1e-10)) return false;
    t = dot3(e2x, e2y, e2z, qx, qy, qz) * inv;
    return true;
}

// The full reference formula for one pair, including the values it yields
// for invalid pairs (inv_det = 0 -> u = v = t = 0), bvh.py:17-27.
__device__ __forceinline__ bool mt_full(double ox, double oy, double oz, double dx, double dy,
                                        double dz, const double* __restrict__ v, double& t) {
    const double v0x = v[0], v0y = v[1], v0z = v[2];
    const double e1x = v[3], e1y = v[4], e1z = v[5];
    const double e2x = v[6], e2y = v[7], e2z = v[8];
    const double px = dy * e2z - dz * e2y;
    const double py = dz * e2x - dx * e2z;
    const double pz = dx * e2y - dy * e2x;
    const double det = dot3(e1x, e1y, e1z, px, py, pz);
    const bool ok = fabs(det) > 1e-14;
    const double inv = ok ? 1.0 / det : 0.0;
    const double tx = ox - v0x, ty = oy - v0y, tz = oz - v0z;
    const double u = dot3(tx, ty, tz, px, py, pz) * inv;
    const double qx = ty * e1z - tz * e1y;
    const double qy = tz * e1x - tx * e1z;
    const double qz = tx * e1y - ty * e1x;
    const double vv = dot3(qx, qy, qz, dx, dy, dz) * inv;
    t = dot3(e2x, e2y, e2z, qx, qy, qz) * inv;
    return ok && (u >= -1e-10) && (vv >= -1e-10) && (u + vv <= 1.0 + 1e-10);
}

// ------------------------------------------------------ 256-bit loads ----
// sm_100 LDG.E.256: one 32-byte sector per thread per instruction.  The BVH
// nodes (four 32-byte planes/children groups) and the 96-byte triangle
// records are laid out so every load is one full sector; 16-byte loads of
// the same data fetch each sector twice (half-used), which was the largest
// share of the big-scene kernel's L1 wavefronts (ncu, r02a).
struct __align__(32) F8 {
    float a, b, c, d, e, f, g, h;
};
struct __align__(32) D4 {
    double x, y, z, w;
};
// L1 policy hints of the node / triangle loads.  With the 128-byte f32
// nodes at 512 threads the triangle records (tested ~3 per segment) did
// best skipping L1 allocation (C5 3.92 vs 3.88, r02t); with the 64-byte
// nodes at 1024 threads L1 has room for them and the streets' facades are
// hit again and again: L1::evict_first 4.76, plain 4.75, no_allocate 4.51
// G seg/s on C5 (C3 3.29 / 3.29 / 3.30, C2 1.74 / 1.75 / 1.72; A/B abI);
// evict_last on the nodes changes nothing.  Tuning builds:
// EF_NODE_HINT 1 = L1::evict_last; EF_TRI_HINT 0 = none, 1 = L1::no_allocate,
// 2 = L1::evict_first
#ifndef EF_NODE_HINT
#define EF_NODE_HINT 0
#endif
#ifndef EF_TRI_HINT
#define EF_TRI_HINT 2
#endif
#if EF_NODE_HINT == 1
#define EF_NODE_Q ".L1::evict_last"
#else
#define EF_NODE_Q ""
#endif
#if EF_TRI_HINT == 1
#define EF_TRI_Q ".L1::no_allocate"
#elif EF_TRI_HINT == 2
#define EF_TRI_Q ".L1::evict_first"
#else
#define EF_TRI_Q ""
#endif
__device__ __forceinline__ F8 ldg_f8(const void* p) {
    F8 r;
    asm("ld.global.nc" EF_NODE_Q ".v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(r.a), "=f"(r.b), "=f"(r.c), "=f"(r.d), "=f"(r.e), "=f"(r.f), "=f"(r.g), "=f"(r.h)
        : "l"(p));
    return r;
}
__device__ __forceinline__ D4 ldg_d4(const void* p) {
    D4 r;
    asm("ld.global.nc" EF_TRI_Q ".v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ldg_d2(const void* p) {
    double2 r;
    asm("ld.global.nc" EF_TRI_Q ".v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}

// ----------------------------------------------------------- traversal ----
struct RayF {
    float ox, oy, oz;    // origin * inv (for the FMA slab form)
    float ix, iy, iz;    // 1 / direction
    int nx, ny, nz;      // float4 index of the near plane per axis (far = near ^ 1)
};

// 1/d for the slab test.  rcp.approx (<= 1 ulp, no slow path): an error in
// 1/d scales every plane distance of that axis alike, far inside the slab
// test's 3.8e-6 slack and the boxes' 1e-5 * scale padding.
__device__ __forceinline__ float safe_inv(double d) {
    float f = (float)d;
    if (fabsf(f) < 1e-20f) f = copysignf(1e-20f, f);
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f));
    return r;
}

__device__ __forceinline__ RayF make_rayf(double ox, double oy, double oz, double dx, double dy,
                                          double dz) {
    RayF r;
    r.ix = safe_inv(dx);
    r.iy = safe_inv(dy);
    r.iz = safe_inv(dz);
    r.ox = __fmul_rn((float)ox, r.ix);
    r.oy = __fmul_rn((float)oy, r.iy);
    r.oz = __fmul_rn((float)oz, r.iz);
    // node layout lox,hix,loy,hiy,loz,hiz: the near plane of an axis is its
    // lo plane for a positive direction, its hi plane otherwise
    r.nx = r.ix >= 0.0f ? 0 : 1;
    r.ny = r.iy >= 0.0f ? 2 : 3;
    r.nz = r.iz >= 0.0f ? 4 : 5;
    return r;
}

__device__ __forceinline__ float fmax3f(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));   // FMNMX3 (sm_100)
    return d;
}
__device__ __forceinline__ float fmin3f(float a, float b, float c) {
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

struct Hit {
    double t;
    int32_t id;  // original triangle id, INT32_MAX = none
};

// The reference's Moeller-Trumbore decision (bvh.py:17-27) restricted to
// t in (t_min, t_hi], with a division-free conservative pre-rejection: the
// unnormalised U, V, T are compared against |det|-scaled bounds with a 2x
// margin, so a candidate is only dropped early when the exact test would
// drop it too; survivors take the bit-exact path (1/det, u, v, t).
__device__ __forceinline__ bool mt_hit(double ox, double oy, double oz, double dx, double dy,
                                       double dz, const double* __restrict__ v, double t_min,
                                       double t_hi, double& t) {
    const double v0x = v[0], v0y = v[1], v0z = v[2];
    const double e1x = v[3], e1y = v[4], e1z = v[5];
    const double e2x = v[6], e2y = v[7], e2z = v[8];
    const double px = dy * e2z - dz * e2y;
    const double py = dz * e2x - dx * e2z;
    const double pz = dx * e2y - dy * e2x;
    const double det = dot3(e1x, e1y, e1z, px, py, pz);
    const double tx = ox - v0x, ty = oy - v0y, tz = oz - v0z;
    const double U = dot3(tx, ty, tz, px, py, pz);
    const double qx = ty * e1z - tz * e1y;
    const double qy = tz * e1x - tx * e1z;
    const double qz = tx * e1y - ty * e1x;
    const double V = dot3(qx, qy, qz, dx, dy, dz);
    const double T = dot3(e2x, e2y, e2z, qx, qy, qz);
    const double ad = fabs(det);
    if (!(ad > 1e-14)) return false;
    const double sg = det > 0.0 ? 1.0 : -1.0;
    const double Ua = U * sg, Va = V * sg, Ta = T * sg;
    if (Ua < -2e-10 * ad || Va < -2e-10 * ad || Ua + Va > (1.0 + 2e-10) * ad ||
        Ta <= 0.5 * t_min * ad || Ta > t_hi * ad * (1.0 + 1e-9))
        return false;
    const double inv = 1.0 / det;
    const double u = U * inv;
    const double vv = V * inv;
    if (!(u >= -1e-10) || !(vv >= -1e-10) || !(u + vv <= 1.0 + 1e-10)) return false;
    t = T * inv;
    return t > t_min && t <= t_hi;
}

// Conservative slab test of one child box; returns a sortable key (t_near
// bits with the low two bits replaced by the child slot; t_near >= 0 so
// unsigned order == float order) or 0xffffffff on a miss.  Two equivalent
// forms: slab_key_minmax evaluates both planes of an axis and orders them
// (all seven loads of a node then use immediate offsets: fewer instructions),
// slab_key takes the ray's sign-selected near/far planes (fewer registers).
// No multiplicative slack on t_far: every box is padded outward by 1e-5 of
// the largest coordinate magnitude (bvh_build.cpp, bvh_device.cu), which
// moves t_near down and t_far up by >= that distance along the unit ray,
// ~100x the f32 rounding of these products (<= 2^-23 of |o| + |plane|, and
// the <= 1 ulp rcp.approx of 1/d); so a ray meeting a triangle's exact box
// never misses its padded box.  (A 1 + 3.8e-6 factor on t_far cost one
// FMUL per child.)
// Empty slots hold lo = hi = +inf: on an axis of positive direction t_near
// = +inf, and with every direction component negative t_far = -inf, so they
// miss as long as tmax is finite (closest_bvh clamps it to 1e38).
__device__ __forceinline__ uint32_t slab_key_minmax(const RayF& r, float lx, float hx, float ly,
                                                    float hy, float lz, float hz, float tmin,
                                                    float tmax, uint32_t slot) {
    const float ax = __fmaf_rn(lx, r.ix, -r.ox), bx = __fmaf_rn(hx, r.ix, -r.ox);
    const float ay = __fmaf_rn(ly, r.iy, -r.oy), by = __fmaf_rn(hy, r.iy, -r.oy);
    const float az = __fmaf_rn(lz, r.iz, -r.oz), bz = __fmaf_rn(hz, r.iz, -r.oz);
    const float tn = fmax3f(fminf(ax, bx), fminf(ay, by), fmaxf(fminf(az, bz), tmin));
    const float tf = fmin3f(fmaxf(ax, bx), fmaxf(ay, by), fminf(fmaxf(az, bz), tmax));
    return tn <= tf ? ((__float_as_uint(tn) & ~3u) | slot) : 0xffffffffu;
}

__device__ __forceinline__ uint32_t slab_key(const RayF& r, float nx, float fx, float ny, float fy,
                                             float nz, float fz, float tmin, float tmax,
                                             uint32_t slot) {
    const float tn = fmax3f(__fmaf_rn(nx, r.ix, -r.ox), __fmaf_rn(ny, r.iy, -r.oy),
                            fmaxf(__fmaf_rn(nz, r.iz, -r.oz), tmin));
    const float tf = fmin3f(__fmaf_rn(fx, r.ix, -r.ox), __fmaf_rn(fy, r.iy, -r.oy),
                            fminf(__fmaf_rn(fz, r.iz, -r.oz), tmax));
    return tn <= tf ? ((__float_as_uint(tn) & ~3u) | slot) : 0xffffffffu;
}

// Packed f32x2 FMA (sm_100 FFMA2): two children's planes per instruction.
// ptxas folds a pair {x, x} built from one scalar (with - and |.|) into the
// instruction's scalar-broadcast operand, so the ray terms cost no registers.
typedef unsigned long long f32x2_t;
__device__ __forceinline__ f32x2_t pack2(float a, float b) {
    f32x2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ void unpack2(f32x2_t v, float& a, float& b) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f32x2_t ffma2(f32x2_t a, f32x2_t b, f32x2_t c) {
    f32x2_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// Slab distances of one axis for two children in the centre / half-extent
// form (TravNode): m = c (1/d) - o/d, near = m - e |1/d|, far = m + e |1/d|.
// Conservative like the lo/hi form: [c - e, c + e] encloses the padded box,
// and the three roundings stay ~2^-23 of max(|c|, |o|, |e|) |1/d|, far below
// the boxes' 1e-5 * scale padding.
__device__ __forceinline__ void slab_ce2(float c0, float c1, float e0, float e1, float inv, float oinv,
                                         float& n0, float& n1, float& f0, float& f1) {
    const f32x2_t m = ffma2(pack2(c0, c1), pack2(inv, inv), pack2(-oinv, -oinv));
    const f32x2_t e = pack2(e0, e1);
    unpack2(ffma2(e, pack2(-fabsf(inv), -fabsf(inv)), m), n0, n1);
    unpack2(ffma2(e, pack2(fabsf(inv), fabsf(inv)), m), f0, f1);
}

__device__ __forceinline__ uint32_t slab_key_ce(float nx, float fx, float ny, float fy, float nz, float fz,
                                                float tmin, float tmax, uint32_t slot) {
    const float tn = fmax3f(nx, ny, fmaxf(nz, tmin));
    const float tf = fmin3f(fx, fy, fminf(fz, tmax));
    return tn <= tf ? ((__float_as_uint(tn) & ~3u) | slot) : 0xffffffffu;
}

#if EF_KEY_LOP3
// The same key with (bits & ~3) | slot as ONE three-input LOP3: the mask
// comes in a register the compiler cannot fold (an immediate mask plus an
// immediate slot would need two instructions).
template <uint32_t SLOT>
__device__ __forceinline__ uint32_t slab_key_m(float nx, float fx, float ny, float fy, float nz, float fz,
                                               float tmin, float tmax, uint32_t mask) {
    const float tn = fmax3f(nx, ny, fmaxf(nz, tmin));
    const float tf = fmin3f(fx, fy, fminf(fz, tmax));
    uint32_t k;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(k) : "r"(__float_as_uint(tn)), "r"(mask), "n"(SLOT));
    return tn <= tf ? k : 0xffffffffu;
}
#endif

// The four children's sortable keys of one node visit (X, Y, Z: the node's
// three 32-byte plane groups).
__device__ __forceinline__ void node_keys(const RayF& r, const F8& X, const F8& Y, const F8& Z, float tmin,
                                          float tmax, uint32_t& k0, uint32_t& k1, uint32_t& k2,
                                          uint32_t& k3) {
#if EF_SLAB_CE
    float nx[4], fx[4], ny[4], fy[4], nz[4], fz[4];
    slab_ce2(X.a, X.b, X.e, X.f, r.ix, r.ox, nx[0], nx[1], fx[0], fx[1]);
    slab_ce2(X.c, X.d, X.g, X.h, r.ix, r.ox, nx[2], nx[3], fx[2], fx[3]);
    slab_ce2(Y.a, Y.b, Y.e, Y.f, r.iy, r.oy, ny[0], ny[1], fy[0], fy[1]);
    slab_ce2(Y.c, Y.d, Y.g, Y.h, r.iy, r.oy, ny[2], ny[3], fy[2], fy[3]);
    slab_ce2(Z.a, Z.b, Z.e, Z.f, r.iz, r.oz, nz[0], nz[1], fz[0], fz[1]);
    slab_ce2(Z.c, Z.d, Z.g, Z.h, r.iz, r.oz, nz[2], nz[3], fz[2], fz[3]);
    k0 = slab_key_ce(nx[0], fx[0], ny[0], fy[0], nz[0], fz[0], tmin, tmax, 0u);
    k1 = slab_key_ce(nx[1], fx[1], ny[1], fy[1], nz[1], fz[1], tmin, tmax, 1u);
    k2 = slab_key_ce(nx[2], fx[2], ny[2], fy[2], nz[2], fz[2], tmin, tmax, 2u);
    k3 = slab_key_ce(nx[3], fx[3], ny[3], fy[3], nz[3], fz[3], tmin, tmax, 3u);
#else
    k0 = slab_key_minmax(r, X.a, X.e, Y.a, Y.e, Z.a, Z.e, tmin, tmax, 0u);
    k1 = slab_key_minmax(r, X.b, X.f, Y.b, Y.f, Z.b, Z.f, tmin, tmax, 1u);
    k2 = slab_key_minmax(r, X.c, X.g, Y.c, Y.g, Z.c, Z.g, tmin, tmax, 2u);
    k3 = slab_key_minmax(r, X.d, X.h, Y.d, Y.h, Z.d, Z.h, tmin, tmax, 3u);
#endif
}

#if EF_QNODE
// The ray in the units of the 16-bit plane grid (TravGrid): plane q of an
// axis is met at t = q * s + b, s = cell / d, b = (lo - o) / d.  A plane's
// float is built by one PRMT as 2^23 + q (exact), so the FMA below uses
// B = b - 2^23 s; the cancellation leaves an error below one cell in t
// (<= 0.5 ulp of 2^23 |s| twice), which the encoder's extra cell on each
// side of every box covers (ef_scene.cu encode_planes).  sel: PRMT selector
// of the near plane's half word (lo for a positive direction).
struct RayQ {
    float sx, sy, sz;
    float Bx, By, Bz;
    uint32_t selx, sely, selz;
#if EF_KEY_LOP3
    uint32_t mask;
#endif
};

__device__ __forceinline__ RayQ make_rayq(const RayF& r, const F8& G) {
    RayQ q;
    q.sx = __fmul_rn(G.e, r.ix);
    q.sy = __fmul_rn(G.f, r.iy);
    q.sz = __fmul_rn(G.g, r.iz);
    q.Bx = __fmaf_rn(-8388608.0f, q.sx, __fmaf_rn(G.a, r.ix, -r.ox));
    q.By = __fmaf_rn(-8388608.0f, q.sy, __fmaf_rn(G.b, r.iy, -r.oy));
    q.Bz = __fmaf_rn(-8388608.0f, q.sz, __fmaf_rn(G.c, r.iz, -r.oz));
    q.selx = r.ix >= 0.0f ? 0x7410u : 0x7432u;
    q.sely = r.iy >= 0.0f ? 0x7410u : 0x7432u;
    q.selz = r.iz >= 0.0f ? 0x7410u : 0x7432u;
#if EF_KEY_LOP3
    asm volatile("mov.u32 %0, 0xfffffffc;" : "=r"(q.mask));
#endif
    return q;
}

// near / far parameters of one axis for the four children (words w0..w3)
__device__ __forceinline__ void slab_q4(float w0, float w1, float w2, float w3, uint32_t sel, float s, float B,
                                        float* tn, float* tf) {
    const uint32_t self = sel ^ 0x0022u;   // the other half word
    const uint32_t u0 = __float_as_uint(w0), u1 = __float_as_uint(w1), u2 = __float_as_uint(w2),
                   u3 = __float_as_uint(w3);
    const f32x2_t ss = pack2(s, s), bb = pack2(B, B);
    unpack2(ffma2(pack2(__uint_as_float(__byte_perm(u0, 0x4B000000u, sel)),
                        __uint_as_float(__byte_perm(u1, 0x4B000000u, sel))), ss, bb), tn[0], tn[1]);
    unpack2(ffma2(pack2(__uint_as_float(__byte_perm(u2, 0x4B000000u, sel)),
                        __uint_as_float(__byte_perm(u3, 0x4B000000u, sel))), ss, bb), tn[2], tn[3]);
    unpack2(ffma2(pack2(__uint_as_float(__byte_perm(u0, 0x4B000000u, self)),
                        __uint_as_float(__byte_perm(u1, 0x4B000000u, self))), ss, bb), tf[0], tf[1]);
    unpack2(ffma2(pack2(__uint_as_float(__byte_perm(u2, 0x4B000000u, self)),
                        __uint_as_float(__byte_perm(u3, 0x4B000000u, self))), ss, bb), tf[2], tf[3]);
}

// A = px[0..3] py[0..3], Bz = pz[0..3] (the node's second sector also holds the children)
__device__ __forceinline__ void node_keys_q(const RayQ& r, const F8& A, const F8& Bz, float tmin, float tmax,
                                            uint32_t& k0, uint32_t& k1, uint32_t& k2, uint32_t& k3) {
    float nx[4], fx[4], ny[4], fy[4], nz[4], fz[4];
    slab_q4(A.a, A.b, A.c, A.d, r.selx, r.sx, r.Bx, nx, fx);
    slab_q4(A.e, A.f, A.g, A.h, r.sely, r.sy, r.By, ny, fy);
    slab_q4(Bz.a, Bz.b, Bz.c, Bz.d, r.selz, r.sz, r.Bz, nz, fz);
#if EF_KEY_LOP3
    k0 = slab_key_m<0u>(nx[0], fx[0], ny[0], fy[0], nz[0], fz[0], tmin, tmax, r.mask);
    k1 = slab_key_m<1u>(nx[1], fx[1], ny[1], fy[1], nz[1], fz[1], tmin, tmax, r.mask);
    k2 = slab_key_m<2u>(nx[2], fx[2], ny[2], fy[2], nz[2], fz[2], tmin, tmax, r.mask);
    k3 = slab_key_m<3u>(nx[3], fx[3], ny[3], fy[3], nz[3], fz[3], tmin, tmax, r.mask);
#else
    k0 = slab_key_ce(nx[0], fx[0], ny[0], fy[0], nz[0], fz[0], tmin, tmax, 0u);
    k1 = slab_key_ce(nx[1], fx[1], ny[1], fy[1], nz[1], fz[1], tmin, tmax, 1u);
    k2 = slab_key_ce(nx[2], fx[2], ny[2], fy[2], nz[2], fz[2], tmin, tmax, 2u);
    k3 = slab_key_ce(nx[3], fx[3], ny[3], fy[3], nz[3], fz[3], tmin, tmax, 3u);
#endif
}
#endif

__device__ __forceinline__ void kswap(uint32_t& a, uint32_t& b) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

// Child `slot` (the low two bits of a sort key) of a node: a two-level
// select, no branches.  In PTX so that each bit test is an and + setp.ne 0
// (one LOP3 with a predicate result each); the C++ form's i1 truncation of
// bit 0 became and + setp.eq 1, two instructions.
#ifndef EF_PICK_PTX
#define EF_PICK_PTX 1
#endif
__device__ __forceinline__ int32_t pick(const int4& c, uint32_t slot) {
#if EF_PICK_PTX
    int32_t r;
    asm("{\n\t.reg .pred p0, p1;\n\t.reg .b32 t0, t1, a, b;\n\t"
        "and.b32 t0, %5, 1;\n\tsetp.ne.u32 p0, t0, 0;\n\t"
        "and.b32 t1, %5, 2;\n\tsetp.ne.u32 p1, t1, 0;\n\t"
        "selp.b32 a, %2, %1, p0;\n\tselp.b32 b, %4, %3, p0;\n\t"
        "selp.b32 %0, b, a, p1;\n\t}"
        : "=r"(r)
        : "r"(c.x), "r"(c.y), "r"(c.z), "r"(c.w), "r"(slot));
    return r;
#else
    const int32_t a = (slot & 1u) ? c.y : c.x;
    const int32_t b = (slot & 1u) ? c.w : c.z;
    return (slot & 2u) ? b : a;
#endif
}

// Leaf: exact tests of up to 8 consecutive triangles of the leaf-ordered
// payload; equal t resolves to the lowest original id.
__device__ __forceinline__ void leaf_test(const GpuTri* __restrict__ tris, int32_t enc, double ox,
                                          double oy, double oz, double dx, double dy, double dz,
                                          double t_min, Hit& h, float& tb, uint32_t& n_tris) {
    const uint32_t e = ~(uint32_t)enc;
    const uint32_t start = e >> 3, cnt = (e & 7u) + 1u;
#ifndef EF_NO_WORK_COUNTERS
    n_tris += cnt;
#endif
    for (uint32_t i = 0; i < cnt; ++i) {
        const GpuTri* q = tris + start + i;   // 96 bytes: three 256-bit loads
        const D4 a = ldg_d4(q->v), b = ldg_d4(q->v + 4);
        const double2 c = ldg_d2(q->v + 8);
        const double v[9] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x};
        const int32_t id = (int32_t)__double_as_longlong(c.y);
        double t;
        if (mt_hit(ox, oy, oz, dx, dy, dz, v, t_min, h.t, t) && (t < h.t || id < h.id)) {
            h.t = t;
            h.id = id;
            tb = __double2float_ru(t);
        }
    }
}

// Traversal stacks.  Entry = (node, key).  The trace kernels keep a thread's
// stack top in a shared-memory column (i-major: entry i of thread t at
// base + i * STEP + 8 t, conflict-free and immune to L1 thrashing by node and
// triangle traffic), addressed by a 32-bit shared-window address in a
// register; DEPTH and STEP are compile-time constants, so a push is one STS
// at sbase + sp * STEP.  (A runtime depth / stride with a null-column check
// made the compiler rebuild the column address from the shared window base
// on every push and pop: ~13% of the C5 kernel's instructions, r02c.)
constexpr int kSmemStack = 16;   // max shared entries per thread

// Shared-window address of the dynamic shared memory of a kernel without
// static shared memory (sm_100a reserves the first 1 KB of the window).  The
// host probes it before the first BVH trace (check_smem_base, ef_trace.cu)
// and the BVH trace kernels check it at their start and trap otherwise.
constexpr uint32_t kDynSmemBase = 0x400u;

// Shared top (DEPTH entries) + local-memory overflow (rarely touched).  The
// whole stack pointer is ONE register: sa = kDynSmemBase + 8 t + sp * STEP,
// the shared address of entry sp of thread t (the stack area opens the
// kernel's dynamic shared memory, 8 t < STEP).  Emptiness, the shared /
// local split and the entry index are all compares of sa with immediates.
// (With a (column base, sp) pair the compiler, at 64 registers, rebuilt the
// column base on every push and pop -- S2R tid, S2UR cta id, UMOV, ULEA, LEA,
// IMAD: 3.7% of the C5 kernel's instructions at 4 active lanes, r02 source
// view.)
template <int DEPTH, uint32_t STEP>
struct StackSplit {
    static constexpr bool kPredicated = false;
    static constexpr uint32_t kLo = kDynSmemBase + STEP;           // sa < kLo: empty
    static constexpr uint32_t kHi = kDynSmemBase + DEPTH * STEP;   // sa < kHi: entry in shared memory
    uint32_t sa;
    uint2* l;        // local-memory overflow array (outside the struct, so the
                     // scalar can live in a register)

    __device__ __forceinline__ bool empty() const { return sa < kLo; }
    __device__ __forceinline__ int depth() const { return (int)((sa - kDynSmemBase) / STEP); }
    __device__ __forceinline__ void pop() { sa -= STEP; }
    // slot of entry sa in the overflow array: sa / STEP is depth() or
    // depth() + 1 (threads whose 8 t carries into the next STEP), the same
    // for a thread's push and pop of an entry, so no offset is subtracted;
    // the array has one spare slot
    __device__ __forceinline__ uint32_t overflow_slot() const { return sa / STEP; }
    __device__ __forceinline__ void push(int32_t node, uint32_t key) {
        if (sa < kHi) {
            // volatile asm keeps push/pop order; no memory clobber, so global
            // loads (nodes, triangles) still schedule freely around it
            asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(sa), "r"((uint32_t)node), "r"(key));
        } else {
            l[overflow_slot()] = make_uint2((uint32_t)node, key);
        }
        sa += STEP;
    }
    __device__ __forceinline__ uint2 top() const {
        if (sa < kHi) {
            uint2 e;
            asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(e.x), "=r"(e.y) : "r"(sa));
            return e;
        }
        return l[overflow_slot()];
    }
};

// The whole stack in shared memory (the host guarantees the column holds the
// tree's max_stack): pushes are predicated stores, no overflow branch.  Like
// StackSplit the pointer is one register, the shared address of the next
// entry (8 t < STEP).
template <uint32_t STEP>
struct StackShared {
    static constexpr bool kPredicated = true;
    static constexpr uint32_t kLo = kDynSmemBase + STEP;   // sa < kLo: empty
    uint32_t sa;

    __device__ __forceinline__ bool empty() const { return sa < kLo; }
    __device__ __forceinline__ int depth() const { return (int)((sa - kDynSmemBase) / STEP); }
    __device__ __forceinline__ void pop() { sa -= STEP; }
    // push `node, key` if `valid` (no branch: predicated st.shared)
    __device__ __forceinline__ void push_if(int32_t node, uint32_t key, bool valid) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\t"
            "@p st.shared.v2.u32 [%0], {%1, %2};\n\t}" ::"r"(sa),
            "r"((uint32_t)node), "r"(key), "r"((uint32_t)valid));
        sa += valid ? STEP : 0u;
    }
    __device__ __forceinline__ uint2 top() const {
        uint2 e;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(e.x), "=r"(e.y) : "r"(sa));
        return e;
    }
};

// Local memory only (the query kernels: no shared memory).
struct StackLocal {
    static constexpr bool kPredicated = false;
    uint2 l[kStackSize];
    int sp;
    __device__ __forceinline__ bool empty() const { return sp == 0; }
    __device__ __forceinline__ int depth() const { return sp; }
    __device__ __forceinline__ void pop() { --sp; }
    __device__ __forceinline__ void push(int32_t node, uint32_t key) {
        l[sp++] = make_uint2((uint32_t)node, key);
    }
    __device__ __forceinline__ uint2 top() const { return l[sp]; }
};

// Closest hit over the 4-wide device BVH.  Accepts t in (t_min, t_max];
// equal t resolves to the lowest triangle id, so the answer is independent of
// the tree and of the traversal order.  While-while form
// (Aila & Laine 2009): each lane descends through inner nodes (nearest child
// first, packed-key sorting network, farther hits pushed) until it holds a
// leaf, so the expensive f64 leaf tests of a warp run together.  The stack
// (st, empty on entry) is one of the forms above.
template <typename StackT>
__device__ __forceinline__ Hit closest_bvh(const TravNode* __restrict__ nodes,
                                           const GpuTri* __restrict__ tris, double ox, double oy,
                                           double oz, double dx, double dy, double dz, double t_min,
                                           double t_max, uint32_t& n_nodes, uint32_t& n_tris,
                                           StackT& st, bool any_hit = false) {
    Hit h{t_max, INT32_MAX};
    const RayF r = make_rayf(ox, oy, oz, dx, dy, dz);
#if EF_QNODE
    const RayQ rq = make_rayq(r, ldg_f8(nodes - 1));   // the slot before node 0 holds the grid
#endif
    const float tminf = fmaxf(__double2float_rd(t_min), 0.0f);
    float tb = fminf(__double2float_ru(t_max), 1e38f);   // finite: empty slots must miss
    int32_t node = 0;
    bool done = false;
    EF_STK_DECL;
    for (;;) {
        while (node >= 0) {
            EF_PHASE_T0(tv);
#ifndef EF_NO_WORK_COUNTERS
            ++n_nodes;
#endif
#if EF_QNODE
            // two 256-bit loads: x and y plane words, z plane words + children
            const TravNode* q = nodes + node;
            const F8 X = ldg_f8(q->px), Z = ldg_f8(q->pz);
            const int4 ch = make_int4(__float_as_int(Z.e), __float_as_int(Z.f), __float_as_int(Z.g),
                                      __float_as_int(Z.h));
#else
            // three 256-bit loads (centres / half extents of x, y, z), one 128-bit (children)
            const TravNode* q = nodes + node;
            const F8 X = ldg_f8(q->cx), Y = ldg_f8(q->cy), Z = ldg_f8(q->cz);
            const int4 ch = __ldg(reinterpret_cast<const int4*>(q->child));
#endif
            uint32_t k0, k1, k2, k3;
#if EF_QNODE
            node_keys_q(rq, X, Z, tminf, tb, k0, k1, k2, k3);
#else
            node_keys(r, X, Y, Z, tminf, tb, k0, k1, k2, k3);
#endif
            kswap(k0, k1);
            kswap(k2, k3);
            kswap(k0, k2);
            kswap(k1, k3);
            kswap(k1, k2);
#ifdef EF_PROFILE_PHASES
            {
                const int nh = (k0 != 0xffffffffu) + (k1 != 0xffffffffu) + (k2 != 0xffffffffu) + (k3 != 0xffffffffu);
                EF_STK(4 + (nh > 3 ? 3 : nh));
                if (nh > 1) {
                    stk[0] += nh - 1;
                    for (int i_ = 0; i_ < nh - 1; ++i_)
                        if (st.depth() + i_ >= EF_SPLIT_DEPTH_PROBE) EF_STK(1);
                }
            }
#endif
            if constexpr (StackT::kPredicated) {
                st.push_if(pick(ch, k3 & 3u), k3, k3 != 0xffffffffu);
                st.push_if(pick(ch, k2 & 3u), k2, k2 != 0xffffffffu);
                st.push_if(pick(ch, k1 & 3u), k1, k1 != 0xffffffffu);
            } else {
#if EF_NESTED_PUSH
                // keys are sorted and a miss is the largest key: k1 missing
                // means k2 and k3 are missing too (76% of C5's node visits
                // hit one child: one not-taken branch instead of three)
                if (k1 != 0xffffffffu) {
                    if (k2 != 0xffffffffu) {
                        if (k3 != 0xffffffffu) st.push(pick(ch, k3 & 3u), k3);
                        st.push(pick(ch, k2 & 3u), k2);
                    }
                    st.push(pick(ch, k1 & 3u), k1);
                }
#else
                if (k3 != 0xffffffffu) st.push(pick(ch, k3 & 3u), k3);
                if (k2 != 0xffffffffu) st.push(pick(ch, k2 & 3u), k2);
                if (k1 != 0xffffffffu) st.push(pick(ch, k1 & 3u), k1);
#endif
            }
            if (k0 != 0xffffffffu) {
                node = pick(ch, k0 & 3u);
                EF_PHASE_ADD(0, tv);
                continue;
            }
            // no child hit: pop the next node still in front of the closest
            // hit (the key's t is rounded down, so the cull is conservative)
            for (;;) {
                if (st.empty()) {
                    done = true;
                    break;
                }
                st.pop();
                const uint2 e = st.top();
                if (__uint_as_float(e.y & ~3u) <= tb) {
                    node = (int32_t)e.x;
                    EF_STK(2);
                    break;
                }
                EF_STK(3);
            }
            EF_PHASE_ADD(0, tv);
            if (done) break;
        }
        if (done) {
            EF_STK_FLUSH;
            return h;
        }
        EF_PHASE_T0(tl);
        EF_STK(8);
        leaf_test(tris, node, ox, oy, oz, dx, dy, dz, t_min, h, tb, n_tris);
        EF_PHASE_ADD(1, tl);
        if (any_hit && h.id != INT32_MAX) {   // shadow rays: any blocker will do
            EF_STK_FLUSH;
            return h;
        }
        EF_PHASE_T0(tp);
        for (;;) {
            if (st.empty()) {
                EF_STK_FLUSH;
                return h;
            }
            st.pop();
            const uint2 e = st.top();
            if (__uint_as_float(e.y & ~3u) <= tb) {
                node = (int32_t)e.x;
                EF_STK(2);
                break;
            }
            EF_STK(3);
        }
        EF_PHASE_ADD(2, tp);
    }
}

// The trace kernels' forms: the whole stack in shared memory (SSTACK), or
// its top DEPTH entries there and the rest in local memory; THREADS columns.
template <int THREADS, int DEPTH, bool SSTACK>
__device__ __forceinline__ Hit closest_bvh_column(const TravNode* __restrict__ nodes,
                                                  const GpuTri* __restrict__ tris, double ox,
                                                  double oy, double oz, double dx, double dy,
                                                  double dz, double t_min, double t_max,
                                                  uint32_t& n_nodes, uint32_t& n_tris,
                                                  const uint2* s_stack, bool any_hit = false) {
    if constexpr (SSTACK) {
        (void)s_stack;
        StackShared<8u * THREADS> st{kDynSmemBase + 8u * threadIdx.x};
        return closest_bvh(nodes, tris, ox, oy, oz, dx, dy, dz, t_min, t_max, n_nodes, n_tris, st, any_hit);
    } else {
        uint2 overflow[kStackSize + 1];
        (void)s_stack;   // the stack area opens the dynamic shared memory (checked by the kernel)
        StackSplit<DEPTH, 8u * THREADS> st{kDynSmemBase + 8u * threadIdx.x, overflow};
        return closest_bvh(nodes, tris, ox, oy, oz, dx, dy, dz, t_min, t_max, n_nodes, n_tris, st, any_hit);
    }
}

__device__ __forceinline__ Hit closest_bvh(const TravNode* __restrict__ nodes,
                                           const GpuTri* __restrict__ tris, double ox, double oy,
                                           double oz, double dx, double dy, double dz, double t_min,
                                           double t_max) {
    uint32_t a = 0, b = 0;
    StackLocal st;
    st.sp = 0;
    return closest_bvh(nodes, tris, ox, oy, oz, dx, dy, dz, t_min, t_max, a, b, st);
}

// ------------------------------------------------------------------ SH ----
// Real SH, ACN order, exactly sh.py:94-125 (same expression trees).
template <int ORDER>
__device__ __forceinline__ void eval_sh(double x, double y, double z, double* out) {
    constexpr double C0 = 0.28209479177387814;
    constexpr double C1 = 0.4886025119029199;
    out[0] = C0;
    if (ORDER >= 1) {
        out[1] = -C1 * y;
        out[2] = C1 * z;
        out[3] = -C1 * x;
    }
    if (ORDER >= 2) {
        const double xx = x * x, yy = y * y, zz = z * z;
        out[4] = 1.0925484305920792 * x * y;
        out[5] = -1.0925484305920792 * y * z;
        out[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
        out[7] = -1.0925484305920792 * x * z;
        out[8] = 0.5462742152960396 * (xx - yy);
        if (ORDER >= 3) {
            out[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
            out[10] = 2.890611442640554 * x * y * z;
            out[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
            out[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
            out[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
            out[14] = 1.445305721320277 * z * (xx - yy);
            out[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
        }
        if (ORDER >= 4) {
            out[16] = 2.5033429417967046 * x * y * (xx - yy);
            out[17] = -1.7701307697799304 * y * z * (3.0 * xx - yy);
            out[18] = 0.9461746957575601 * x * y * (7.0 * zz - 1.0);
            out[19] = -0.6690465435572892 * y * z * (7.0 * zz - 3.0);
            out[20] = 0.10578554691520431 * (zz * (35.0 * zz - 30.0) + 3.0);
            out[21] = -0.6690465435572892 * x * z * (7.0 * zz - 3.0);
            out[22] = 0.47308734787878004 * (xx - yy) * (7.0 * zz - 1.0);
            out[23] = -1.7701307697799304 * x * z * (xx - 3.0 * yy);
            out[24] = 0.6258357354491761 * (xx * (xx - 3.0 * yy) - yy * (3.0 * xx - yy));
        }
    }
}

}  // namespace ef
