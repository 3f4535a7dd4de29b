// Dependent-chain latency microbenchmark (one warp, clock64 around N ops).
#include <cstdio>
#include <cuda_runtime.h>
#define RUN(k, o, a, name) for (int r = 0; r < 2; ++r) { k<<<1, 1>>>(o, a, t); } cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("%-10s %6.2f cycles/op\n", name, (double)h / N);
int main2();
#define N 4096
__global__ void k_dadd(double* o, double a, long long* t) {
    double x = a; long long s = clock64();
    #pragma unroll 64
    for (int i = 0; i < N; ++i) x = x + a;
    t[0] = clock64() - s; o[0] = x;
}
__global__ void k_dmul(double* o, double a, long long* t) {
    double x = a; long long s = clock64();
    #pragma unroll 64
    for (int i = 0; i < N; ++i) x = x * a;
    t[0] = clock64() - s; o[0] = x;
}
__global__ void k_dfma(double* o, double a, long long* t) {
    double x = a; long long s = clock64();
    #pragma unroll 64
    for (int i = 0; i < N; ++i) x = fma(x, a, a);
    t[0] = clock64() - s; o[0] = x;
}
__global__ void k_ddiv(double* o, double a, long long* t) {
    double x = a; long long s = clock64();
    for (int i = 0; i < N / 16; ++i) x = a / x;
    t[0] = (clock64() - s) * 16; o[0] = x;
}
__global__ void k_dsqrt(double* o, double a, long long* t) {
    double x = a; long long s = clock64();
    for (int i = 0; i < N / 16; ++i) x = sqrt(x + a);
    t[0] = (clock64() - s) * 16; o[0] = x;
}
__global__ void k_ffma(float* o, float a, long long* t) {
    float x = a; long long s = clock64();
    #pragma unroll 64
    for (int i = 0; i < N; ++i) x = fmaf(x, a, a);
    t[0] = clock64() - s; o[0] = x;
}
__global__ void k_imadhi(unsigned* o, unsigned a, long long* t) {
    unsigned x = a; long long s = clock64();
    #pragma unroll 64
    for (int i = 0; i < N; ++i) x = __umulhi(x, 0xD2511F53u) ^ a;
    t[0] = clock64() - s; o[0] = x;
}
__global__ void k_ldl(int* o, int a, long long* t) {
    volatile int st[64];
    for (int i = 0; i < 64; ++i) st[i] = (i * 7 + a) & 63;
    int x = a & 63; long long s = clock64();
    for (int i = 0; i < N / 16; ++i) x = st[x];
    t[0] = (clock64() - s) * 16; o[0] = x;
}
__global__ void k_lds(int* o, int a, long long* t) {
    __shared__ int st[64];
    for (int i = 0; i < 64; ++i) st[i] = (i * 7 + a) & 63;
    __syncwarp();
    int x = a & 63; long long s = clock64();
    for (int i = 0; i < N / 16; ++i) x = st[x];
    t[0] = (clock64() - s) * 16; o[0] = x;
}
int main() {
    double* od; float* of; unsigned* ou; int* oi; long long* t; long long h;
    cudaMalloc(&od, 8); cudaMalloc(&of, 4); cudaMalloc(&ou, 4); cudaMalloc(&oi, 4); cudaMalloc(&t, 8);
    RUN(k_dadd, od, 1.0000001, "DADD");
    RUN(k_dmul, od, 1.0000001, "DMUL");
    RUN(k_dfma, od, 0.5, "DFMA");
    RUN(k_ddiv, od, 1.5, "f64 div");
    RUN(k_dsqrt, od, 1.5, "f64 sqrt");
    RUN(k_ffma, of, 0.5f, "FFMA");
    RUN(k_imadhi, ou, 12345u, "IMAD.HI+LOP");
    RUN(k_ldl, oi, 5, "LDL chain");
    RUN(k_lds, oi, 5, "LDS chain");
    return main2();
}
__global__ void k_drcp(double* o, double a, long long* t) {
    double x = a; long long s = clock64();
    for (int i = 0; i < N / 16; ++i) x = __drcp_rn(x) + a;
    t[0] = (clock64() - s) * 16; o[0] = x;
}
__global__ void k_ddiv1(double* o, double a, long long* t) {
    double x = a; long long s = clock64();
    for (int i = 0; i < N / 16; ++i) x = 1.0 / x + a;
    t[0] = (clock64() - s) * 16; o[0] = x;
}
__global__ void k_check(double* o, double a, long long* t) {
    // bit-identity of __drcp_rn(x) and 1.0/x over many x
    unsigned long long bad = 0; double x = a;
    for (int i = 0; i < 1 << 20; ++i) {
        x = x * 1.0000001 + 1e-3 * (double)(i & 7) - 0.002;
        if (__double_as_longlong(__drcp_rn(x)) != __double_as_longlong(1.0 / x)) ++bad;
    }
    t[0] = bad; o[0] = x;
}
int main2() {
    double* od; long long* t; long long h;
    cudaMalloc(&od, 8); cudaMalloc(&t, 8);
    RUN(k_drcp, od, 1.5, "drcp+add");
    RUN(k_ddiv1, od, 1.5, "1/x+add");
    k_check<<<1,1>>>(od, 0.37, t); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("drcp vs div mismatches: %lld of %d\n", h, 1<<20);
    return 0;
}
