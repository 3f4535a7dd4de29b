// Trace-kernel instantiations: BVH kernels and the frame-tail kernel
// for 4-band scenes (see ef_trace_kernels.cuh).  One translation unit per
// family so the build compiles them in parallel.
#include "ef_trace_kernels.cuh"

namespace ef {

cudaError_t trace_dispatch_bvh_nb4(bool big, int order, const TraceParams& P, cudaStream_t st) {
    return dispatch_bvh<4>(big, order, P, st);
}

cudaError_t tail_dispatch_nb4(int order, const TraceParams& P, cudaStream_t st) {
    return launch_tail<4>(order, P, st);
}

#ifdef EF_PROFILE_PHASES
void debug_phases_bvh_nb4(unsigned long long* acc, int reset) {
    unsigned long long v[kPhaseSlots];
    cudaMemcpyFromSymbol(v, g_phase, sizeof v);
    for (int i = 0; i < kPhaseSlots; ++i) acc[i] += v[i];
    if (reset) {
        unsigned long long z[kPhaseSlots] = {0};
        cudaMemcpyToSymbol(g_phase, z, sizeof z);
    }
}
#endif

}  // namespace ef
