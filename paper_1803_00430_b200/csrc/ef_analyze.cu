// K4: per-(source, band) decay-fit reducer.  One 256-thread CTA per
// (source, band); every reduction is a warp-shuffle + shared-memory sum in f64,
// the Schroeder integral a block-wide suffix scan over contiguous bin chunks.
//
// Replaces (SPEC-only in the reference, pinned in DESIGN.md 3.6):
//   estimate_rt60           SPEC.md:272-280 (decisions 344-346)
//   reverb_gain
//   estimate_predelay       SPEC.md:299-307 (decision 347)
//   average_directivity
//   mean free path
// and the reference's directional_loudness_matrix (sh.py:240-253) on
// design_for_order(order) (tdesigns.py:360-362).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <mutex>
#include <unordered_map>

#include "ef_device.cuh"

namespace ef {

constexpr unsigned kAll = 0xffffffffu;
#ifdef EF_PROFILE_PHASES
static __device__ long long g_t0;   // kernel start (block 0, thread 0)
#endif
constexpr double kY00 = 0.28209479177387814;   // sh.py:17
constexpr int kMaxDesign = 64;    // design_for_order(<=4) has 48 points

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kAll, v, o);
    return v;
}

struct AnalyzeParams {
    const float* H;
    const float* Dir;
    const unsigned long long* stats;
    const double* sum_t;
    const double* design;
    int32_t n_design, n_bins, nb;
    double bin_s, max_rt;
    double* params;
    double* src_params;
    double* avg_dir;
    double* loudness;
    int* counters;   // (n_sources) zeroed scratch, reset by the kernel
};

constexpr int kAThreads = 256;   // metrics_kernel
constexpr int kAWarps = kAThreads / 32;
constexpr int kKThreads = 512;   // analyze_kernel: 4 bins per thread at 2,000 bins
constexpr size_t kMaxSeriesSmem = 96 * 1024;   // I_b(t) staged in shared memory up to 12,288 bins

// block-wide sum of one double (all threads get the result)
template <int T = kAThreads>
__device__ __forceinline__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < T / 32; ++i) t += red[i];
    return t;
}

// block-wide sums of N doubles with one pair of barriers (red: N * T/32)
template <int N, int T>
__device__ __forceinline__ void block_sum_n(double (&v)[N], double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = warp_sum(v[i]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < N; ++i) red[i * (T / 32) + w] = v[i];
    __syncthreads();
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < T / 32; ++k) t += red[i * (T / 32) + k];
        v[i] = t;
    }
}

struct Fit {
    bool silent;
    double slope, nfit;
};

// Block-cooperative Schroeder integral from the last non-zero bin
// (truncation) and LS line over EDC in [-35,-5] dB, or
// [-25,-5] dB when the EDC does not reach -35 dB; every thread
// owns the contiguous chunk [lo, hi) of I(t).  DESIGN.md 3.6.
// s_red holds >= 10 * T/32 doubles.
template <int T, class F>
__device__ Fit schroeder_fit(F I, int lo, int hi, int last, int nnz, double bin_s, double* s_red,
                             double* s_dblast) {
    constexpr int W = T / 32;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // n, sx, sy, sxy, sxx for the [-35,-5] (0..4) and [-25,-5] (5..9) ranges;
    // a flat array indexed by constants only, so it stays in registers
    double fit[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    Fit out{true, 0.0, 0.0};
    if (nnz < 3) return out;
    const int h2 = min(hi, last + 1);
    double csum = 0.0;
    for (int t = h2 - 1; t >= lo; --t) csum += I(t);
    double suf = csum;   // block inclusive suffix scan of the chunk sums
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double v = __shfl_down_sync(kAll, suf, o);
        if (lane + o < 32) suf += v;
    }
    __syncthreads();
    if (lane == 0) s_red[w] = suf;   // warp total
    __syncthreads();
    double after = 0.0, edc0 = 0.0;
    for (int i = 0; i < W; ++i) {
        if (i > w) after += s_red[i];
        edc0 += s_red[i];
    }
    suf += after;
    double acc = suf - csum;   // energy after this thread's chunk
    for (int t = h2 - 1; t >= lo; --t) {
        acc += I(t);
        const double db = 10.0 * log10(acc / edc0);
        const double x = (double)t * bin_s;
        if (t == last) *s_dblast = db;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const double lim = r == 0 ? -35.0 : -25.0;
            if (db <= -5.0 && db >= lim) {
                fit[5 * r + 0] += 1.0;
                fit[5 * r + 1] += x;
                fit[5 * r + 2] += db;
                fit[5 * r + 3] += x * db;
                fit[5 * r + 4] += x * x;
            }
        }
    }
    __syncthreads();   // s_red is reused below
    block_sum_n<10, T>(fit, s_red);
    const double db_last = *s_dblast;
    const int r = db_last <= -35.0 ? 0 : (db_last <= -25.0 ? 1 : -1);
    if (r < 0) return out;
    const double n = r ? fit[5] : fit[0], sx = r ? fit[6] : fit[1], sy = r ? fit[7] : fit[2],
                 sxy = r ? fit[8] : fit[3], sxx = r ? fit[9] : fit[4];
    const double den = n * sxx - sx * sx;
    if (n < 2.0 || !(den > 0.0)) return out;
    const double slope = (n * sxy - sx * sy) / den;
    if (!(slope < 0.0)) return out;
    out.silent = false;
    out.slope = slope;
    out.nfit = n;
    return out;
}

template <int ORDER>
__global__ void __launch_bounds__(kKThreads) analyze_kernel(const AnalyzeParams P) {
    constexpr int NK = (ORDER + 1) * (ORDER + 1);
    constexpr int T = kKThreads, W = T / 32;
    extern __shared__ double s_I[];   // I_b(t), when n_bins fits (else read from H)
    __shared__ double s_B[kMaxDesign * NK];
    __shared__ double s_g[kMaxDesign];
    __shared__ double s_avg[NK];
    __shared__ double s_red[10 * W];
    __shared__ double s_wsum[W][NK];
    __shared__ int s_ired[3][W];
    __shared__ double s_dblast;
    __shared__ int s_done;
#ifdef EF_PROFILE_PHASES
    if (threadIdx.x == 0 && blockIdx.x == 0) g_t0 = clock64();
#endif
    const int nb = P.nb;
    const int s = blockIdx.x / nb, b = blockIdx.x % nb;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int nbins = P.n_bins;
    const bool staged = (size_t)nbins * sizeof(double) <= kMaxSeriesSmem;
    const float* Hs = P.H + (size_t)s * nbins * nb * NK + (size_t)b * NK;
    const size_t stride = (size_t)nb * NK;
    for (int j = tid; j < P.n_design; j += T) {
        double Y[NK];
        eval_sh<ORDER>(P.design[3 * j], P.design[3 * j + 1], P.design[3 * j + 2], Y);
#pragma unroll
        for (int k = 0; k < NK; ++k) s_B[j * NK + k] = Y[k];
    }
    if (tid == 0) s_dblast = 0.0;
    pdl_wait();   // the design table above is ready; H is final from here

#ifdef EF_PROFILE_PHASES
    const long long a0 = clock64();   // analysis phases (counters of the analysis TU)
#endif
    // ---- pass 1 (contiguous chunk per thread, all its rows' loads in
    // flight together): support of I_b(t) = H[t,b,0]/Y00, the directivity
    // sums, and I_b(t) staged in shared memory for the fit
    const int chunk = (nbins + T - 1) / T;
    const int lo = min(tid * chunk, nbins), hi = min(lo + chunk, nbins);
    int last = -1, first = INT_MAX, nnz = 0;
    double S[NK];
#pragma unroll
    for (int k = 0; k < NK; ++k) S[k] = 0.0;
#pragma unroll 4
    for (int t = lo; t < hi; ++t) {
        const float* row = Hs + t * stride;
        float r[NK];
        if constexpr (NK % 4 == 0) {   // rows are 16-byte aligned (stride and offset multiples of 4)
#pragma unroll
            for (int k = 0; k < NK; k += 4) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(row + k));
                r[k] = q.x; r[k + 1] = q.y; r[k + 2] = q.z; r[k + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < NK; ++k) r[k] = __ldg(row + k);
        }
        const double i0 = (double)r[0] / kY00;
        if (staged) s_I[t] = i0;
        if (i0 > 0.0) {
            last = t;
            first = min(first, t);
            ++nnz;
        }
#pragma unroll
        for (int k = 0; k < NK; ++k) S[k] += (double)r[k];
    }
#ifdef EF_PROFILE_PHASES
    if (tid == 0 && blockIdx.x == 0) atomicAdd(&g_phase[5], (unsigned long long)(clock64() - a0));
#endif
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        last = max(last, __shfl_xor_sync(kAll, last, o));
        first = min(first, __shfl_xor_sync(kAll, first, o));
        nnz += __shfl_xor_sync(kAll, nnz, o);
    }
#pragma unroll
    for (int k = 0; k < NK; ++k) S[k] = warp_sum(S[k]);
#ifdef EF_PROFILE_PHASES
    if (tid == 0 && blockIdx.x == 0) atomicAdd(&g_phase[6], (unsigned long long)(clock64() - a0));
#endif
    if (lane == 0) {
        s_ired[0][w] = last;
        s_ired[1][w] = first;
        s_ired[2][w] = nnz;
#pragma unroll
        for (int k = 0; k < NK; ++k) s_wsum[w][k] = S[k];
    }
    __syncthreads();
    last = -1; first = INT_MAX; nnz = 0;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        last = max(last, s_ired[0][i]);
        first = min(first, s_ired[1][i]);
        nnz += s_ired[2][i];
    }
    if (tid < NK) {
        double a = 0.0;
#pragma unroll
        for (int i = 0; i < W; ++i) a += s_wsum[i][tid];
        s_avg[tid] = a;   // raw sums for now
    }
    __syncthreads();
    const double total = s_avg[0] / kY00;

#ifdef EF_PROFILE_PHASES
    const long long a1 = clock64();
#endif
    // ---- pass 2: Schroeder fit (shared with the acoustic-metrics kernel)
    const Fit fit = staged
        ? schroeder_fit<T>([&](int t) { return s_I[t]; }, lo, hi, last, nnz, P.bin_s, s_red, &s_dblast)
        : schroeder_fit<T>([&](int t) { return (double)Hs[t * stride] / kY00; }, lo, hi, last, nnz,
                           P.bin_s, s_red, &s_dblast);
    const bool silent = fit.silent;
    const double slope = fit.slope, nfit = fit.nfit;
    double rt60 = 1.0;   // cold-start value for silent bands
    if (!silent) rt60 = fmin(fmax(-60.0 / slope, 0.05), P.max_rt);
    const double gain = (!silent && total > 0.0) ? sqrt(total / (rt60 / (6.0 * log(10.0)))) : 0.0;
    const double edir = (double)P.Dir[((size_t)s * nb + b) * NK] / kY00;
    double drr;
    if (!(edir > 0.0)) drr = -99.0;
    else if (!(total > 0.0)) drr = 99.0;
    else drr = fmin(fmax(10.0 * log10(edir / total), -99.0), 99.0);
    double* p = P.params + ((size_t)s * nb + b) * EF_P_COUNT;
    if (tid == 0) {
        p[EF_P_RT60] = rt60;
        p[EF_P_GAIN] = gain;
        p[EF_P_DRR_DB] = drr;
        p[EF_P_TOTAL] = total;
        p[EF_P_DIRECT] = edir;
        p[EF_P_SILENT] = silent ? 1.0 : 0.0;
        p[EF_P_FIT_N] = nfit;
        p[EF_P_SLOPE] = slope;
        p[EF_P_FIRST_BIN] = first == INT_MAX ? -1.0 : (double)first;
        p[EF_P_LAST_BIN] = (double)last;
    }

#ifdef EF_PROFILE_PHASES
    const long long a2 = clock64();
#endif
    // ---- average directivity and loudness (sh.py:240-253)
    __syncthreads();
    if (tid < NK) s_avg[tid] = total > 0.0 ? s_avg[tid] / total : 0.0;
    __syncthreads();
    if (tid < NK && P.avg_dir) P.avg_dir[((size_t)s * nb + b) * NK + tid] = s_avg[tid];
    if (P.loudness) {
        for (int j = tid; j < P.n_design; j += T) {
            double g = 0.0;
#pragma unroll
            for (int k = 0; k < NK; ++k) g += s_B[j * NK + k] * s_avg[k];
            s_g[j] = fmax(0.0, g);
        }
        __syncthreads();
        // D = (4 pi / N) B^T diag(g) B: two adjacent lanes per entry, each
        // summing half of the design, joined by one shuffle
        const double scale = 4.0 * M_PI / (double)P.n_design;
        double* D = P.loudness + ((size_t)s * nb + b) * NK * NK;
        const int half = (P.n_design + 1) / 2;
        for (int base = 0; base < 2 * NK * NK; base += T) {   // block-uniform trip count
            const int e2 = base + tid;
            const bool ok = e2 < 2 * NK * NK;
            const int e = e2 >> 1, k1 = e / NK, k2 = e % NK;
            const int j0 = (e2 & 1) * half, j1 = ok ? min(P.n_design, j0 + half) : j0;
            double acc = 0.0;
            for (int j = j0; j < j1; ++j) acc += s_B[j * NK + k1] * s_g[j] * s_B[j * NK + k2];
            acc += __shfl_xor_sync(kAll, acc, 1);
            if (ok && !(e2 & 1)) D[e] = scale * acc;
        }
    }

#ifdef EF_PROFILE_PHASES
    if (tid == 0 && blockIdx.x == 0) {
        const long long a3 = clock64();
        atomicAdd(&g_phase[0], (unsigned long long)(a1 - a0));
        atomicAdd(&g_phase[1], (unsigned long long)(a2 - a1));
        atomicAdd(&g_phase[2], (unsigned long long)(a3 - a2));
        atomicAdd(&g_phase[3], 1ull);
        atomicAdd(&g_phase[4], (unsigned long long)(a0 - g_t0));
    }
#endif
    // ---- per-source outputs: the last band block of a source finishes it
    // (the finisher reads only the FIRST_BIN entries, written by thread 0)
    if (tid == 0) {
        __threadfence();
        s_done = atomicAdd(P.counters + s, 1);
    }
    __syncthreads();
    if (s_done == nb - 1 && tid == 0) {
        __threadfence();
        double firstb = -1.0;
        for (int bb = 0; bb < nb; ++bb) {
            const double f = ((volatile double*)P.params)[((size_t)s * nb + bb) * EF_P_COUNT + EF_P_FIRST_BIN];
            if (f >= 0.0 && (firstb < 0.0 || f < firstb)) firstb = f;
        }
        double* q = P.src_params + (size_t)s * EF_S_COUNT;
        q[EF_S_PREDELAY] = firstb < 0.0 ? -1.0 : firstb * P.bin_s;
        const unsigned long long nrefl = P.stats[(size_t)s * EF_ST_COUNT + EF_ST_REFLECTIONS];
        q[EF_S_MFP] = nrefl ? P.sum_t[s] / (double)nrefl : 0.0;
        q[EF_S_SILENT] = firstb < 0.0 ? 1.0 : 0.0;
        q[3] = 0.0;
        P.counters[s] = 0;
    }
}

// Acoustic metrics of energy series: one CTA per series.
__global__ void __launch_bounds__(kAThreads) metrics_kernel(const double* E, int n_bins, double bin_s,
                                                            const int32_t* direct_index, double e_ref,
                                                            double max_rt, double* out) {
    __shared__ double s_red[10 * kAWarps];
    __shared__ double s_dblast;
    __shared__ int s_ired[2][kAWarps];
    const int sr = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const double* I = E + (size_t)sr * n_bins;
    const int d0 = direct_index ? max(0, min(direct_index[sr], n_bins - 1)) : 0;
    const int n80 = (int)llrint(0.080 / bin_s), n50 = (int)llrint(0.050 / bin_s);
    const int chunk = (n_bins + kAThreads - 1) / kAThreads;
    const int lo = min(tid * chunk, n_bins), hi = min(lo + chunk, n_bins);
    int last = -1, nnz = 0;
    double tot = 0.0, e80 = 0.0, e50 = 0.0, tsn = 0.0;
    for (int t = lo; t < hi; ++t) {
        const double v = I[t];
        if (v > 0.0) {
            last = t;
            ++nnz;
        }
        if (t >= d0) {
            tot += v;
            if (t < d0 + n80) e80 += v;
            if (t < d0 + n50) e50 += v;
            tsn += ((double)(t - d0) + 0.5) * bin_s * v;   // bin centres
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        last = max(last, __shfl_xor_sync(kAll, last, o));
        nnz += __shfl_xor_sync(kAll, nnz, o);
    }
    if (lane == 0) {
        s_ired[0][w] = last;
        s_ired[1][w] = nnz;
    }
    __syncthreads();
    last = -1;
    nnz = 0;
    for (int i = 0; i < kAWarps; ++i) {
        last = max(last, s_ired[0][i]);
        nnz += s_ired[1][i];
    }
    tot = block_sum(tot, s_red);
    e80 = block_sum(e80, s_red);
    e50 = block_sum(e50, s_red);
    tsn = block_sum(tsn, s_red);
    if (tid == 0) s_dblast = 0.0;
    __syncthreads();
    const Fit fit = schroeder_fit<kAThreads>([&](int t) { return I[t]; }, lo, hi, last, nnz, bin_s, s_red,
                                             &s_dblast);
    if (tid == 0) {
        double* o = out + (size_t)sr * 5;
        o[0] = fit.silent ? -1.0 : fmin(fmax(-60.0 / fit.slope, 0.05), max_rt);
        const double late = tot - e80;
        o[1] = late > 0.0 ? fmin(10.0 * log10(e80 / late), 99.0) : 99.0;   // C80, +99 dB sentinel
        o[2] = tot > 0.0 ? e50 / tot : 0.0;                                // D50
        o[3] = tot > 0.0 ? tsn / tot : 0.0;                                // TS, s
        o[4] = (tot > 0.0 && e_ref > 0.0) ? 10.0 * log10(tot / e_ref) : -99.0;   // G, dB
    }
}

__global__ void blend_kernel(const float* cache, const float* frame,
                             int64_t n, float a, float b, float* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = a * frame[i] + b * cache[i];
}

// Per-stream "source finished" counters for analyze_kernel: zeroed once when
// allocated and left zeroed by the kernel itself (its last CTA per source
// resets its entry), so a call needs no allocation or memset.  Calls on one
// stream are ordered; different streams get different buffers.
static int* analyze_counters(cudaStream_t st, int n, cudaError_t& e) {
    static std::mutex mu;
    static std::unordered_map<cudaStream_t, std::pair<int*, int>> bufs;
    std::lock_guard<std::mutex> lock(mu);
    auto& b = bufs[st];
    if (b.second < n) {
        if (b.first) {
            e = cudaFreeAsync(b.first, st);
            if (e != cudaSuccess) return nullptr;
        }
        b = {nullptr, 0};
        const int cap = std::max(n, 256);
        e = cudaMallocAsync((void**)&b.first, sizeof(int) * cap, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(b.first, 0, sizeof(int) * cap, st);
        if (e != cudaSuccess) return nullptr;
        b.second = cap;
    }
    e = cudaSuccess;
    return b.first;
}

#ifdef EF_PROFILE_PHASES
}  // namespace ef
// debug builds: [0] pass 1, [1] fit, [2] directivity + loudness, [3] calls,
// [4] start -> pass 1, [5] pass-1 rows done, [6] pass-1 warp sums done
extern "C" int ef_debug_analysis_phases(unsigned long long* out7, int reset) {
    cudaMemcpyFromSymbol(out7, ef::g_phase, sizeof(unsigned long long) * 7);
    if (reset) {
        unsigned long long z[ef::kPhaseSlots] = {0};
        cudaMemcpyToSymbol(ef::g_phase, z, sizeof z);
    }
    return EF_OK;
}
namespace ef {
#endif

template <int ORDER>
static void analyze_set_smem() {
    cudaFuncSetAttribute(analyze_kernel<ORDER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kMaxSeriesSmem);
}

}  // namespace ef

using namespace ef;

extern "C" int ef_acoustic_metrics(const double* energy, int64_t n_series, int32_t n_bins,
                                   double bin_s, const int32_t* direct_index, double e_ref,
                                   double max_rt, double* out, void* stream) {
    if (n_series < 0 || n_bins < 1 || !(bin_s > 0.0)) return set_error(EF_EINVAL, "ef_acoustic_metrics: bad sizes");
    if (n_series == 0) return EF_OK;
    if (!energy || !out) return set_error(EF_EINVAL, "ef_acoustic_metrics: null argument");
    metrics_kernel<<<(unsigned)n_series, kAThreads, 0, (cudaStream_t)stream>>>(energy, n_bins, bin_s, direct_index,
                                                                              e_ref, max_rt, out);
    count_launch();
    return check_cuda(cudaGetLastError(), "metrics_kernel");
}

extern "C" int ef_blend(const float* cache, const float* frame, int64_t n, double alpha, float* out,
                        void* stream) {
    if (n < 0 || !(alpha >= 0.0 && alpha <= 1.0)) return set_error(EF_EINVAL, "ef_blend: bad n or alpha");
    if (n == 0) return EF_OK;
    if (!cache || !frame || !out) return set_error(EF_EINVAL, "ef_blend: null argument");
    const long long g = std::min<long long>((n + 255) / 256, 148LL * 16);
    blend_kernel<<<(int)g, 256, 0, (cudaStream_t)stream>>>(cache, frame, n, (float)alpha,
                                                           (float)(1.0 - alpha), out);
    count_launch();
    return check_cuda(cudaGetLastError(), "blend_kernel");
}

extern "C" int ef_analyze(const ef_analysis_config* cfg, const float* H, const float* Dir,
                          const unsigned long long* stats, const double* sum_t,
                          const double* design, int32_t n_design, double* params,
                          double* src_params, double* avg_dir, double* loudness, void* stream) {
    if (!cfg || !H || !Dir || !stats || !sum_t || !params || !src_params)
        return set_error(EF_EINVAL, "ef_analyze: null argument");
    if (cfg->order < 0 || cfg->order > kMaxOrder) return set_error(EF_EINVAL, "ef_analyze: order must be in [0, 4]");
    if (cfg->n_bands < 1 || cfg->n_bands > kMaxBands) return set_error(EF_EINVAL, "ef_analyze: n_bands must be in [1, 8]");
    if (cfg->n_sources < 1 || cfg->n_bins < 1) return set_error(EF_EINVAL, "ef_analyze: empty histogram");
    if (loudness && (!design || n_design < 1 || n_design > kMaxDesign))
        return set_error(EF_EINVAL, "ef_analyze: loudness needs a t-design of 1..64 directions");
    if (!(cfg->bin_s > 0.0) || !(cfg->max_rt >= 0.05)) return set_error(EF_EINVAL, "ef_analyze: bad bin_s / max_rt");
    cudaStream_t st = (cudaStream_t)stream;
    keep_pool_memory();
    cudaError_t e = cudaSuccess;
    int* counters = analyze_counters(st, cfg->n_sources, e);
    if (!counters) return check_cuda(e, "ef_analyze scratch");
    AnalyzeParams P{H, Dir, stats, sum_t, design, loudness ? n_design : 0, cfg->n_bins, cfg->n_bands,
                    cfg->bin_s, cfg->max_rt, params, src_params, avg_dir, loudness, counters};
    const dim3 grid(cfg->n_sources * cfg->n_bands), block(kKThreads);
    const size_t smem = (size_t)cfg->n_bins * sizeof(double) <= kMaxSeriesSmem
                            ? (size_t)cfg->n_bins * sizeof(double) : 0;
    static bool attr_done = false;
    if (!attr_done) {   // the static shared tables plus up to 96 KB of series
        analyze_set_smem<0>(); analyze_set_smem<1>(); analyze_set_smem<2>();
        analyze_set_smem<3>(); analyze_set_smem<4>();
        attr_done = true;
    }
    // PDL: the kernel may be scheduled before the trace (or tail) kernel ends;
    // it evaluates its t-design table, then waits for the histograms
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaError_t le = cudaSuccess;
    switch (cfg->order) {
        case 0: le = cudaLaunchKernelEx(&lc, analyze_kernel<0>, P); break;
        case 1: le = cudaLaunchKernelEx(&lc, analyze_kernel<1>, P); break;
        case 2: le = cudaLaunchKernelEx(&lc, analyze_kernel<2>, P); break;
        case 3: le = cudaLaunchKernelEx(&lc, analyze_kernel<3>, P); break;
        default: le = cudaLaunchKernelEx(&lc, analyze_kernel<4>, P); break;
    }
    if (le == cudaSuccess) le = cudaGetLastError();
    count_launch();
    return check_cuda(le, "analyze_kernel");
}
