// FP64 (and FP32) FMA throughput of the whole GPU: every SM full of warps,
// eight independent FMA chains per thread, CUDA events around the launch.
// Reported as TFLOP/s (2 flops per FMA) -- the FP64-pipe peak SURVEY.md 8(d)
// asks for, which MEASURED_PEAKS.json does not carry.
#include <cstdio>
#include <cuda_runtime.h>

template <class T>
__global__ void fma_kernel(T* out, T a, T b, int iters) {
    T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
      x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

template <class T>
double run(const char* name, int sms) {
    const int threads = 1024, blocks = sms * 2, iters = 4096;
    T* out;
    cudaMalloc(&out, sizeof(T) * threads * blocks);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    fma_kernel<T><<<blocks, threads>>>(out, (T)0.999999, (T)1e-7, 64);   // warm-up
    cudaEventRecord(e0);
    fma_kernel<T><<<blocks, threads>>>(out, (T)0.999999, (T)1e-7, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    const double tf = flops / (ms * 1e-3) / 1e12;
    printf("%s FMA: %.2f TFLOP/s (%.3f ms)\n", name, tf, ms);
    cudaFree(out);
    return tf;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double f64 = run<double>("FP64", sms);
    const double f32 = run<float>("FP32", sms);
    printf("{\"fp64_fma_tflops\": %.3f, \"fp32_fma_tflops\": %.3f, \"sms\": %d, "
           "\"fp64_fma_per_sm_per_clk_at_%d_mhz\": %.1f}\n",
           f64, f32, sms, clk / 1000, f64 * 1e12 / 2 / sms / (clk * 1e3));
    return 0;
}
