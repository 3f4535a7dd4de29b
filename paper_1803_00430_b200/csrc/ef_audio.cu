// K5 + K6: SH-domain auralization (BASELINE config C4).
//
// Replaces the SPEC-only renderer (crossover, delay taps,
// SH-domain reverberator -- here the 16-line-per-band FDN that C4 asks for --
// and directional loudness) and spatialize_hrtf (Eq. 2).
// Semantics pinned in DESIGN.md 3.7 and restated in oracle/audio.py.
//
// Per 512-sample block:
//   xover_kernel   one thread per (source, band): 5-biquad LR4/allpass
//                  cascade over the block (state carried), band samples
//                  written to the source's band history ring (coalesced via
//                  a shared-memory transpose every 32 samples)
//   render_kernel  persistent CTAs of 512 threads (thread = sample): per
//                  source, direct tap + SH encode and the 16-line FDN of each
//                  band (reads of the delayed line samples, barrier, writes);
//                  line outputs go to SH through g_reverb,b * D_b * E; every
//                  CTA accumulates its sources into a private partial bus
//   bus_kernel     sums the partial buses, keeps the previous bus block and
//                  runs the overlap-save binaural decode: 16 forward FFTs
//                  (1024 points, radix-2 in shared memory), spectral MACs with
//                  the 16 x 2 HRTF spectra, 2 inverse FFTs
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "ef_internal.h"

namespace ef {
namespace {

constexpr int kBlock = 512;
constexpr int kBands = 4;
constexpr int kLines = 16;
constexpr int kSh = 16;
constexpr int kBiquads = 5;
constexpr int kFft = 1024;
constexpr int kXoverThreads = 128;   // 32 sources x 4 bands
constexpr int kChunk = 32;

struct AudioState {
    int S = 0;
    int hist_len = 0;     // power of two
    int line_len = 0;     // power of two
    long long t = 0;      // absolute sample index of the next block
    int grid = 0;
    // parameters
    float* sos = nullptr;        // (4, 5, 5) b0 b1 b2 a1 a2
    float* Y = nullptr;          // (S, 16) direct-path SH encoding
    int* d_int = nullptr;        // (S) floor(direct delay)
    float* d_w = nullptr;        // (S) interpolation weight of the newer sample
    float* gain = nullptr;       // (S, 4) direct gain per band
    int* p_int = nullptr;        // (S) floor(predelay)
    float* p_w = nullptr;
    int* m = nullptr;            // (S, 16) FDN line delays (samples)
    float* g = nullptr;          // (S, 4, 16) FDN line gains
    float* M = nullptr;          // (S, 4, 16 sh, 16 lines) line -> SH matrices
    float2* H = nullptr;         // (16, 2, 513) HRTF spectra
    // state
    float* zi = nullptr;         // (S, 4, 5, 2) biquad states
    float* hist = nullptr;       // (S, 4, hist_len) band history rings
    float* lines = nullptr;      // (S, 4, 16, line_len) FDN line rings
    float* partial = nullptr;    // (grid, 16, 512) partial buses
    float* bus = nullptr;        // (16, 512) current bus block
    float* prev_bus = nullptr;   // (16, 512) previous bus block
    long long bytes = 0;
};

__global__ void __launch_bounds__(kXoverThreads) xover_kernel(AudioState A, const float* __restrict__ x) {
    __shared__ float s_out[kXoverThreads][kChunk + 1];
    __shared__ float s_sos[kBands * kBiquads * 5];
    const int tid = threadIdx.x;
    const int s0 = blockIdx.x * (kXoverThreads / kBands);
    for (int i = tid; i < kBands * kBiquads * 5; i += blockDim.x) s_sos[i] = A.sos[i];
    __syncthreads();
    const int ls = tid >> 2, b = tid & 3;
    const int s = s0 + ls;
    const bool live = s < A.S;
    float z[kBiquads][2];
    float* zs = A.zi + ((size_t)s * kBands + b) * kBiquads * 2;
#pragma unroll
    for (int q = 0; q < kBiquads; ++q) {
        z[q][0] = live ? zs[2 * q] : 0.f;
        z[q][1] = live ? zs[2 * q + 1] : 0.f;
    }
    const float* c = s_sos + b * kBiquads * 5;
    const int hmask = A.hist_len - 1;
    for (int n0 = 0; n0 < kBlock; n0 += kChunk) {
        for (int j = 0; j < kChunk; ++j) {
            float v = live ? __ldg(x + (size_t)s * kBlock + n0 + j) : 0.f;
#pragma unroll
            for (int q = 0; q < kBiquads; ++q) {   // transposed direct form II
                const float y = __fmaf_rn(c[5 * q + 0], v, z[q][0]);
                z[q][0] = __fmaf_rn(-c[5 * q + 3], y, __fmaf_rn(c[5 * q + 1], v, z[q][1]));
                z[q][1] = __fmaf_rn(-c[5 * q + 4], y, c[5 * q + 2] * v);
                v = y;
            }
            s_out[tid][j] = v;
        }
        __syncthreads();
        // coalesced write-out: one warp per (source, band) row of kChunk floats
        for (int r = tid >> 5; r < kXoverThreads; r += kXoverThreads / 32) {
            const int rs = s0 + (r >> 2), rb = r & 3;
            const int j = tid & 31;
            if (rs < A.S && j < kChunk) {
                const long long tt = A.t + n0 + j;
                A.hist[((size_t)rs * kBands + rb) * A.hist_len + (tt & hmask)] = s_out[r][j];
            }
        }
        __syncthreads();
    }
    if (live) {
#pragma unroll
        for (int q = 0; q < kBiquads; ++q) {
            zs[2 * q] = z[q][0];
            zs[2 * q + 1] = z[q][1];
        }
    }
}

__device__ __forceinline__ float tap(const float* __restrict__ row, long long t, int dint, float w,
                                     int mask) {
    // value at time t - D, D = dint + (1 - w) fractional: (1-w) x[i0] + w x[i0+1]
    const long long i0 = t - dint - 1;
    const float a = row[i0 & mask], b = row[(i0 + 1) & mask];
    return __fmaf_rn(w, b - a, a);
}

// ---- bulk-copy (TMA engine) + mbarrier helpers, raw PTX for sm_100a
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// Stage buffer of one (source, band) job: 16 line windows of 512 samples,
// each fetched 16-byte aligned (up to 3 extra samples at either end, and a
// wrap of the ring splits it in two copies landing back to back).
constexpr int kWin = kBlock + 8;
constexpr int kStages = 4;                         // jobs in flight
constexpr int kStageM = kLines * kWin;             // band's line -> SH matrix (256 floats)
constexpr int kStageG = kStageM + kSh * kLines;    // band's line gains (16 floats)
constexpr int kStageFloats = kStageG + kLines;
constexpr size_t kRenderDynSmem = (size_t)kStages * kStageFloats * sizeof(float);
constexpr int kConsumerWarps = kBlock / 32;        // one sample per consumer thread
constexpr int kRenderThreads = kBlock + 32;        // + one producer warp

// Job (s, b)'s line windows: the window of line i starts at sample `start`
// of its ring; it is fetched from the 16-byte aligned a0 <= start, in one
// copy or, when it wraps the ring, two copies landing back to back.
struct Window {
    int a0, n1, n2;   // first copy [a0, a0 + n1) floats, second [0, n2) (0: none)
};
__device__ __forceinline__ Window window(int start, int L) {
    Window w;
    w.a0 = start & ~3;
    const int end = start + kBlock;
    if (end <= L) {
        w.n1 = ((end + 3) & ~3) - w.a0;
        w.n2 = 0;
    } else {
        w.n1 = L - w.a0;
        w.n2 = (end - L + 3) & ~3;
    }
    return w;
}

// Producer lane: arm stage barrier `bar` with the job's byte count, then
// issue the bulk copies of job (s, b) into stage `buf`: the 16 line windows
// (off[i] = window start in line i), the band's line -> SH matrix and gains.
// The offsets are stored BEFORE the arrive.expect_tx: that arrive releases
// the lane's earlier shared-memory writes to the consumers that pass the
// stage's full barrier (complete_tx only publishes the copied bytes).
__device__ __forceinline__ void issue_job(const AudioState& A, int s, int b, float* buf, int* off,
                                          uint32_t bar) {
    const int L = A.line_len;
    int start[kLines];
    uint32_t bytes = (uint32_t)(kSh * kLines + kLines) * 4u;   // M_b and g_b
#pragma unroll
    for (int i = 0; i < kLines; ++i) {
        start[i] = (int)((A.t - __ldg(A.m + s * kLines + i)) & (L - 1));
        const Window w = window(start[i], L);
        bytes += (uint32_t)(w.n1 + w.n2) * 4u;
        off[i] = start[i] - w.a0;
    }
    mbar_expect_tx(bar, bytes);
    const size_t sb = (size_t)s * kBands + b;
    bulk_g2s(smem_addr(buf + kStageM), A.M + sb * kSh * kLines, kSh * kLines * 4u, bar);
    bulk_g2s(smem_addr(buf + kStageG), A.g + sb * kLines, kLines * 4u, bar);
#pragma unroll
    for (int i = 0; i < kLines; ++i) {
        const Window w = window(start[i], L);
        const float* row = A.lines + (((size_t)s * kBands + b) * kLines + i) * L;
        const uint32_t dst = smem_addr(buf + i * kWin);
        bulk_g2s(dst, row + w.a0, (uint32_t)w.n1 * 4u, bar);
        if (w.n2) bulk_g2s(dst + (uint32_t)w.n1 * 4u, row, (uint32_t)w.n2 * 4u, bar);
    }
}

// Persistent CTAs, one per SM: 16 consumer warps (thread = sample) and one
// producer warp.  Work is a sequence of (source, band) jobs.  The producer
// lane fetches each job with bulk copies (the TMA engine: the 16 delayed
// line windows, the band's line -> SH matrix and gains) into a 4-stage
// shared-memory ring, waiting on the stage's "empty" mbarrier and arming its
// "full" one; consumers wait on "full", run the band's FDN (line writes go
// straight to global memory) and SH accumulation, and each warp arrives on
// "empty".  No CTA-wide barrier: warps drift freely, the producer stays up
// to four jobs ahead.  A job's reads are complete in shared memory before
// it writes, so the ring's read/write aliasing is harmless.
__global__ void __launch_bounds__(kRenderThreads, 1) render_kernel(AudioState A) {
    extern __shared__ __align__(128) float s_buf[];   // kStages x kStageFloats
    __shared__ __align__(8) unsigned long long s_full[kStages];
    __shared__ __align__(8) unsigned long long s_empty[kStages];
    __shared__ int s_off[kStages][kLines];
    const int n = threadIdx.x;
    const int my_sources = blockIdx.x < A.S ? (A.S - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int jobs = kBands * my_sources;
    if (n == 0) {
        for (int st = 0; st < kStages; ++st) {
            mbar_init(smem_addr(&s_full[st]), 1);
            mbar_init(smem_addr(&s_empty[st]), kConsumerWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (n >= kBlock) {   // ---- producer warp
        if (n == kBlock) {
            for (int j = 0; j < jobs; ++j) {
                const int st = j % kStages;
                const int use = j / kStages;
                if (use > 0) mbar_wait(smem_addr(&s_empty[st]), (uint32_t)(use - 1) & 1u);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue_job(A, blockIdx.x + (j / kBands) * gridDim.x, j % kBands,
                          s_buf + (size_t)st * kStageFloats, s_off[st], smem_addr(&s_full[st]));
            }
        }
        return;
    }
    // ---- consumers
    const int lane = n & 31;
    const long long t = A.t + n;
    const int hmask = A.hist_len - 1;
    float bus[kSh];
#pragma unroll
    for (int k = 0; k < kSh; ++k) bus[k] = 0.f;
    float send[kBands];
    for (int j = 0; j < jobs; ++j) {
        const int s = blockIdx.x + (j / kBands) * gridDim.x;
        const int b = j % kBands;
        const int st = j % kStages;
        if (b == 0) {
            // direct path: one tap per band, SH encode
            // (per-source scalars read by every thread: L1 broadcasts)
            const float* hs = A.hist + (size_t)s * kBands * A.hist_len;
            const int d0 = __ldg(A.d_int + s), d1 = __ldg(A.p_int + s);
            const float w0 = __ldg(A.d_w + s), w1 = __ldg(A.p_w + s);
            float mono = 0.f;
#pragma unroll
            for (int bb = 0; bb < kBands; ++bb) {
                const float* row = hs + (size_t)bb * A.hist_len;
                mono = __fmaf_rn(__ldg(A.gain + s * kBands + bb), tap(row, t, d0, w0, hmask), mono);
                send[bb] = tap(row, t, d1, w1, hmask);
            }
#pragma unroll
            for (int k = 0; k < kSh; ++k) bus[k] = __fmaf_rn(__ldg(A.Y + s * kSh + k), mono, bus[k]);
        }
        // stage `st` serves job j on its (j / kStages)-th use: phase parity
        mbar_wait(smem_addr(&s_full[st]), (uint32_t)(j / kStages) & 1u);
        const float* sb = s_buf + (size_t)st * kStageFloats;
        const float* sM = sb + kStageM;
        const float* sg = sb + kStageG;
        float y[kLines];
#pragma unroll
        for (int i = 0; i < kLines; ++i) y[i] = sb[i * kWin + s_off[st][i] + n];
        float sum = 0.f;
#pragma unroll
        for (int i = 0; i < kLines; ++i) sum = __fmaf_rn(sg[i], y[i], sum);
        const float in = 0.25f * send[b] - (2.0f / kLines) * sum;   // Householder feedback
        float* ls = A.lines + ((size_t)s * kBands + b) * kLines * A.line_len;
        const int w = (int)(t & (A.line_len - 1));
#pragma unroll
        for (int i = 0; i < kLines; ++i) ls[(size_t)i * A.line_len + w] = __fmaf_rn(sg[i], y[i], in);
        // line outputs -> SH bus through g_reverb,b * D_b * E
#pragma unroll
        for (int k = 0; k < kSh; ++k) {
            float acc = bus[k];
#pragma unroll
            for (int i = 0; i < kLines; ++i) acc = __fmaf_rn(sM[k * kLines + i], y[i], acc);
            bus[k] = acc;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_addr(&s_empty[st]));   // this warp is done with the stage
    }
    for (int k = 0; k < kSh; ++k) A.partial[((size_t)blockIdx.x * kSh + k) * kBlock + n] = bus[k];
}

// In-place radix-2 FFT of kFft complex values in shared memory (bit-reversed
// input order handled by the caller's load); sign -1 forward, +1 inverse.
__device__ void fft_smem(float2* a, float sign) {
    for (int len = 2; len <= kFft; len <<= 1) {
        const int half = len >> 1;
        for (int j = threadIdx.x; j < kFft / 2; j += blockDim.x) {
            const int grp = j / half, pos = j % half;
            const int i0 = grp * len + pos, i1 = i0 + half;
            float sn, cs;
            sincospif(sign * 2.0f * (float)pos / (float)len, &sn, &cs);
            const float2 u = a[i0], v = a[i1];
            const float2 w = make_float2(v.x * cs - v.y * sn, v.x * sn + v.y * cs);
            a[i0] = make_float2(u.x + w.x, u.y + w.y);
            a[i1] = make_float2(u.x - w.x, u.y - w.y);
        }
        __syncthreads();
    }
}

__device__ __forceinline__ int bitrev10(int i) { return __brev(i) >> 22; }

// bus[k][n] = sum of the partial buses (one CTA per SH channel)
__global__ void __launch_bounds__(kBlock) reduce_kernel(AudioState A, float* bus_out) {
    const int k = blockIdx.x, n = threadIdx.x;
    float v = 0.f;
    for (int c = 0; c < A.grid; ++c) v += A.partial[((size_t)c * kSh + k) * kBlock + n];
    A.bus[k * kBlock + n] = v;
    if (bus_out) bus_out[k * kBlock + n] = v;
}

__global__ void __launch_bounds__(512) bus_kernel(AudioState A, float* out) {
    __shared__ float2 s_a[kFft];
    __shared__ float2 s_acc[2][kFft / 2 + 1];
    const int tid = threadIdx.x;
    for (int i = tid; i < 2 * (kFft / 2 + 1); i += blockDim.x) s_acc[i / (kFft / 2 + 1)][i % (kFft / 2 + 1)] = make_float2(0.f, 0.f);
    for (int k = 0; k < kSh; ++k) {
        const float v = A.bus[k * kBlock + tid];
        __syncthreads();
        const float prev = A.prev_bus[k * kBlock + tid];
        // overlap-save input [prev | cur], loaded in bit-reversed order
        s_a[bitrev10(tid)] = make_float2(prev, 0.f);
        s_a[bitrev10(tid + kBlock)] = make_float2(v, 0.f);
        A.prev_bus[k * kBlock + tid] = v;
        __syncthreads();
        fft_smem(s_a, -1.0f);
        for (int f = tid; f <= kFft / 2; f += blockDim.x) {
            const float2 X = s_a[f];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const float2 h = A.H[((size_t)k * 2 + e) * (kFft / 2 + 1) + f];
                s_acc[e][f].x += X.x * h.x - X.y * h.y;
                s_acc[e][f].y += X.x * h.y + X.y * h.x;
            }
        }
        __syncthreads();
    }
    for (int e = 0; e < 2; ++e) {
        // inverse real FFT via a full complex IFFT of the Hermitian spectrum
        for (int f = tid; f < kFft; f += blockDim.x) {
            const float2 v = f <= kFft / 2 ? s_acc[e][f]
                                           : make_float2(s_acc[e][kFft - f].x, -s_acc[e][kFft - f].y);
            s_a[bitrev10(f)] = v;
        }
        __syncthreads();
        fft_smem(s_a, 1.0f);
        out[e * kBlock + tid] = s_a[kBlock + tid].x * (1.0f / kFft);
        __syncthreads();
    }
}

template <class T>
cudaError_t up(T** dst, const T* src, size_t n, long long& bytes) {
    cudaError_t e = cudaMalloc((void**)dst, n * sizeof(T));
    if (e != cudaSuccess) return e;
    bytes += (long long)(n * sizeof(T));
    if (src) return cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice);
    return cudaMemset(*dst, 0, n * sizeof(T));
}

}  // namespace
}  // namespace ef

struct ef_audio {
    ef::AudioState A;
};

using namespace ef;

static void free_audio(ef_audio* h) {
    if (!h) return;
    AudioState& A = h->A;
    for (void* p : {(void*)A.sos, (void*)A.Y, (void*)A.d_int, (void*)A.d_w, (void*)A.gain,
                    (void*)A.p_int, (void*)A.p_w, (void*)A.m, (void*)A.g, (void*)A.M, (void*)A.H,
                    (void*)A.zi, (void*)A.hist, (void*)A.lines, (void*)A.partial, (void*)A.bus,
                    (void*)A.prev_bus})
        cudaFree(p);
    delete h;
}

extern "C" int ef_audio_create(const ef_audio_config* cfg, const float* sos, const float* Y,
                               const int32_t* d_int, const float* d_w, const float* gain,
                               const int32_t* p_int, const float* p_w, const int32_t* fdn_delay,
                               const float* g_line, const float* M, const float* hrtf_spec,
                               ef_audio** out) {
    if (!cfg || !out) return set_error(EF_EINVAL, "ef_audio_create: null argument");
    *out = nullptr;
    const int S = cfg->n_sources;
    if (S < 1) return set_error(EF_EINVAL, "ef_audio_create: need at least one source");
    auto pow2 = [](int v) { return v > 0 && (v & (v - 1)) == 0; };
    if (!pow2(cfg->hist_len) || !pow2(cfg->line_len))
        return set_error(EF_EINVAL, "ef_audio_create: ring lengths must be powers of two");
    if (!sos || !Y || !d_int || !d_w || !gain || !p_int || !p_w || !fdn_delay || !g_line || !M || !hrtf_spec)
        return set_error(EF_EINVAL, "ef_audio_create: null parameter array");
    for (int s = 0; s < S; ++s) {
        if (d_int[s] < 0 || p_int[s] < 0 || d_int[s] + 2 + kBlock > cfg->hist_len ||
            p_int[s] + 2 + kBlock > cfg->hist_len)
            return set_error(EF_EINVAL, "ef_audio_create: direct delay / predelay outside the history ring");
        for (int i = 0; i < kLines; ++i) {
            const int m = fdn_delay[s * kLines + i];
            if (m <= kBlock || m > cfg->line_len)
                return set_error(EF_EINVAL, "ef_audio_create: FDN delays must lie in (block, line_len]");
        }
    }
    ef_audio* h = new ef_audio();
    AudioState& A = h->A;
    A.S = S;
    A.hist_len = cfg->hist_len;
    A.line_len = cfg->line_len;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    A.grid = std::min(S, sms);   // one persistent 544-thread CTA per SM
    cudaError_t e = cudaSuccess;
#define UP(f, src, n) if (e == cudaSuccess) e = up(&A.f, src, (size_t)(n), A.bytes);
    UP(sos, sos, kBands * kBiquads * 5);
    UP(Y, Y, (size_t)S * kSh);
    UP(d_int, d_int, S);
    UP(d_w, d_w, S);
    UP(gain, gain, (size_t)S * kBands);
    UP(p_int, p_int, S);
    UP(p_w, p_w, S);
    UP(m, fdn_delay, (size_t)S * kLines);
    UP(g, g_line, (size_t)S * kBands * kLines);
    UP(M, M, (size_t)S * kBands * kSh * kLines);
    UP(H, reinterpret_cast<const float2*>(hrtf_spec), (size_t)kSh * 2 * (kFft / 2 + 1));
    UP(zi, (const float*)nullptr, (size_t)S * kBands * kBiquads * 2);
    UP(hist, (const float*)nullptr, (size_t)S * kBands * A.hist_len);
    UP(lines, (const float*)nullptr, (size_t)S * kBands * kLines * A.line_len);
    UP(partial, (const float*)nullptr, (size_t)A.grid * kSh * kBlock);
    UP(bus, (const float*)nullptr, (size_t)kSh * kBlock);
    UP(prev_bus, (const float*)nullptr, (size_t)kSh * kBlock);
#undef UP
    if (e != cudaSuccess) {
        free_audio(h);
        return check_cuda(e, "ef_audio_create");
    }
    *out = h;
    return EF_OK;
}

// Parameter swap at a block boundary (SPEC.md:415-420 update_params): the
// given HOST arrays (NULL = keep) are copied on `stream`, so blocks enqueued
// before this call render with the old parameters and later ones with the
// new.  The FDN line delays and the HRTF are properties of the renderer and
// stay; the band histories, line rings and filter states carry over.
extern "C" int ef_audio_update(ef_audio* h, const float* Y, const int32_t* d_int, const float* d_w,
                               const float* gain, const int32_t* p_int, const float* p_w,
                               const float* g_line, const float* M, void* stream) {
    if (!h) return set_error(EF_EINVAL, "ef_audio_update: null renderer");
    AudioState& A = h->A;
    const int S = A.S;
    for (int s = 0; s < S; ++s) {
        if ((d_int && (d_int[s] < 0 || d_int[s] + 2 + kBlock > A.hist_len)) ||
            (p_int && (p_int[s] < 0 || p_int[s] + 2 + kBlock > A.hist_len)))
            return set_error(EF_EINVAL, "ef_audio_update: direct delay / predelay outside the history ring");
    }
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaSuccess;
    auto cp = [&](void* dst, const void* src, size_t bytes) {
        if (src && e == cudaSuccess) e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
    };
    cp(A.Y, Y, (size_t)S * kSh * 4);
    cp(A.d_int, d_int, (size_t)S * 4);
    cp(A.d_w, d_w, (size_t)S * 4);
    cp(A.gain, gain, (size_t)S * kBands * 4);
    cp(A.p_int, p_int, (size_t)S * 4);
    cp(A.p_w, p_w, (size_t)S * 4);
    cp(A.g, g_line, (size_t)S * kBands * kLines * 4);
    cp(A.M, M, (size_t)S * kBands * kSh * kLines * 4);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);   // the host arrays may be freed on return
    return e == cudaSuccess ? EF_OK : check_cuda(e, "ef_audio_update");
}

extern "C" int ef_audio_destroy(ef_audio* h) {
    free_audio(h);
    return EF_OK;
}

extern "C" int ef_audio_info(const ef_audio* h, int64_t* out4) {
    if (!h || !out4) return set_error(EF_EINVAL, "ef_audio_info: null argument");
    out4[0] = h->A.S;
    out4[1] = h->A.bytes;
    out4[2] = h->A.t;
    out4[3] = h->A.grid;
    return EF_OK;
}

extern "C" int ef_audio_process(ef_audio* h, const float* x, float* bus_out, float* out,
                                void* stream) {
    if (!h || !x || !out) return set_error(EF_EINVAL, "ef_audio_process: null argument");
    cudaStream_t st = (cudaStream_t)stream;
    AudioState& A = h->A;
    const int xg = (A.S + (kXoverThreads / kBands) - 1) / (kXoverThreads / kBands);
    xover_kernel<<<xg, kXoverThreads, 0, st>>>(A, x);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(render_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kRenderDynSmem);
        if (e != cudaSuccess) return check_cuda(e, "render_kernel attributes");
        attr = true;
    }
    render_kernel<<<A.grid, kRenderThreads, kRenderDynSmem, st>>>(A);
    reduce_kernel<<<kSh, kBlock, 0, st>>>(A, bus_out);
    bus_kernel<<<1, 512, 0, st>>>(A, out);
    count_launch(4);
    A.t += kBlock;
    return check_cuda(cudaGetLastError(), "ef_audio_process");
}
