// Read bandwidth of the L1 and L2 caches on the whole GPU: the peaks behind
// bench.py's device-work roofline ("roofline_device"), whose working sets
// (BVH nodes, triangle records) are served from L1/L2, not HBM.
//
//   l2: every CTA streams a 32 MiB buffer (fits the 126 MB L2, ld.global.cg
//       so L1 is bypassed) with 16-byte loads, many passes, after one warm
//       pass; bytes = requested bytes.
//   l1: every CTA re-reads its own 16 KiB slice (ld.global.ca, L1-resident
//       after the first pass) with 16-byte loads.
//   l1_256: the same with 32-byte loads (ld.global.nc.v8, sm_100).
// Prints one JSON object: {"l2_read_gbs", "l1_read_gbs", "l1_read_256_gbs", "sms", "clock_mhz"}.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void l2_read(const float4* __restrict__ p, size_t n, int passes, float* sink) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < passes; ++r) {
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
            float4 v;
            asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p + i));
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 1234.5f) sink[0] = acc;
}

template <bool WIDE>
__global__ void l1_read(const float4* __restrict__ p, int per_cta, int passes, float* sink) {
    const float4* base = p + (size_t)blockIdx.x * per_cta;
    float acc = 0.f;
    for (int r = 0; r < passes; ++r) {
        if (WIDE) {
            for (int i = 2 * threadIdx.x; i < per_cta; i += 2 * blockDim.x) {
                float a0, a1, a2, a3, a4, a5, a6, a7;
                asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(a4), "=f"(a5), "=f"(a6),
                               "=f"(a7)
                             : "l"(base + i));
                acc += ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
            }
        } else {
            for (int i = threadIdx.x; i < per_cta; i += blockDim.x) {
                float4 v;
                asm volatile("ld.global.ca.v4.f32 {%0,%1,%2,%3}, [%4];"
                             : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(base + i));
                acc += v.x + v.y + v.z + v.w;
            }
        }
    }
    if (acc == 1234.5f) sink[0] = acc;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* sink;
    cudaMalloc(&sink, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0.f;

    // L2
    const size_t l2_bytes = 32u << 20;
    float4* buf;
    cudaMalloc(&buf, l2_bytes);
    cudaMemset(buf, 0, l2_bytes);
    const size_t n = l2_bytes / 16;
    const int passes = 50;
    l2_read<<<sms * 4, 512>>>(buf, n, 1, sink);
    cudaEventRecord(a);
    l2_read<<<sms * 4, 512>>>(buf, n, passes, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    const double l2 = (double)l2_bytes * passes / (ms * 1e-3) / 1e9;

    // L1 (16 KiB per CTA, 4 CTAs per SM)
    const int per_cta = (16 << 10) / 16;
    const int ctas = sms * 4;
    float4* l1buf;
    cudaMalloc(&l1buf, (size_t)ctas * per_cta * 16);
    cudaMemset(l1buf, 0, (size_t)ctas * per_cta * 16);
    const int p1 = 4000;
    double l1[2];
    for (int wide = 0; wide < 2; ++wide) {
        auto k = wide ? l1_read<true> : l1_read<false>;
        k<<<ctas, 256>>>(l1buf, per_cta, 2, sink);
        cudaEventRecord(a);
        k<<<ctas, 256>>>(l1buf, per_cta, p1, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        l1[wide] = (double)ctas * per_cta * 16 * p1 / (ms * 1e-3) / 1e9;
    }
    printf("{\"l2_read_gbs\": %.1f, \"l1_read_gbs\": %.1f, \"l1_read_256_gbs\": %.1f, \"sms\": %d, "
           "\"clock_mhz_attr\": %d, \"error\": \"%s\"}\n",
           l2, l1[0], l1[1], sms, clk / 1000, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
