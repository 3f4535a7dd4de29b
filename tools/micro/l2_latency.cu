// Dependent-load latency (pointer chase, one thread) over working sets that
// live in L1, L2 and HBM: the cost of one "round trip" in the latency-bound
// kernels (analysis pass 1, the tail sweep's candidates).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chase(const unsigned* __restrict__ next, unsigned start, int steps, long long* t,
                      unsigned* out) {
    unsigned i = start;
    for (int k = 0; k < 64; ++k) i = next[i];   // warm the path
    const long long s = clock64();
    for (int k = 0; k < steps; ++k) i = __ldg(next + i);
    t[0] = clock64() - s;
    out[0] = i;
}

int main() {
    const size_t sizes[] = {16u << 10, 128u << 10, 4u << 20, 32u << 20, 1024u << 20};
    long long* t;
    unsigned* out;
    cudaMalloc(&t, 8);
    cudaMalloc(&out, 4);
    for (size_t bytes : sizes) {
        const size_t n = bytes / 4;
        unsigned* h = new unsigned[n];
        // one random cycle over 128-byte lines (Sattolo), one word per line
        const size_t lines = n / 32;
        unsigned* perm = new unsigned[lines];
        for (size_t i = 0; i < lines; ++i) perm[i] = (unsigned)i;
        unsigned long long x = 88172645463325252ull;
        for (size_t i = lines - 1; i > 0; --i) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            const size_t j = x % i;
            const unsigned tmp = perm[i]; perm[i] = perm[j]; perm[j] = tmp;
        }
        for (size_t i = 0; i < lines; ++i) h[32 * (size_t)perm[i]] = 32 * perm[(i + 1) % lines];
        delete[] perm;
        unsigned* d;
        cudaMalloc(&d, bytes);
        cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
        const int steps = 4096;
        chase<<<1, 1>>>(d, 0, steps, t, out);   // warm L2
        chase<<<1, 1>>>(d, 0, steps, t, out);
        long long c;
        cudaMemcpy(&c, t, 8, cudaMemcpyDeviceToHost);
        printf("working set %8zu KB: %6.0f cycles per dependent load\n", bytes >> 10, (double)c / steps);
        cudaFree(d);
        delete[] h;
    }
    return 0;
}
