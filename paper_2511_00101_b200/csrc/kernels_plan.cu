// kernels_plan.cu -- per-call plan upload through kernel parameters.
//
// Every SMLM call stages a few KB of plan records (tiles, pairs, adapter blocks) into its
// workspace.  A cudaMemcpyAsync H2D for that would go to a copy engine, where it queues behind
// whatever bulk transfers the application has in flight (measured in the end-to-end bench:
// 14 small uploads per layer-step behind 1 GB of activation copies stretched a 6.7 ms step to
// 25 ms).  Instead the bytes ride in the parameters of a one-CTA copy kernel: the upload is
// stream-ordered compute work, never blocked by the DMA queues, and capturable into CUDA graphs
// by value.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "pdl.cuh"

namespace smlm {
namespace {

template <int N>
struct PlanBlob {
    uint32_t n;
    uint32_t pad[3];
    uint4 data[N / 16];
};

template <int N>
__global__ void __launch_bounds__(256) plan_copy_kernel(uint4 *__restrict__ dst, const __grid_constant__ PlanBlob<N> b) {
    // the parameter reads go ahead of the grid-dependency wait (they touch no global memory):
    // only the stores wait for the previous call's kernels, which may still read this workspace
    constexpr int kPer = (N / 16 + 255) / 256;
    const uint32_t n16 = (b.n + 15) / 16;
    uint4 v[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const uint32_t i = threadIdx.x + 256u * k;
        if (i < n16) v[k] = b.data[i];
    }
    pdl_wait();
    pdl_trigger();
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
        const uint32_t i = threadIdx.x + 256u * k;
        if (i < n16) dst[i] = v[k];
    }
}

template <int N>
int launch_blob(void *dst, const void *src, size_t n, cudaStream_t st) {
    static thread_local PlanBlob<N> blob;
    blob.n = (uint32_t)n;
    memcpy(blob.data, src, n);
    return (int)launch_pdl(plan_copy_kernel<N>, dim3(1), dim3(256), 0, st, reinterpret_cast<uint4 *>(dst), blob);
}

}  // namespace

constexpr size_t kPlanBlobMax = 32000;

// Copies n bytes (host) to dst (device, 16-byte aligned) in stream order through kernel
// parameters.  Returns -1 if n is too large for one parameter block (caller falls back).
int launch_plan_copy(void *dst, const void *src, size_t n, cudaStream_t st) {
    if (n == 0) return 0;
    if (reinterpret_cast<uintptr_t>(dst) % 16) return -1;
    if (n <= 1024) return launch_blob<1024>(dst, src, n, st);
    if (n <= 4096) return launch_blob<4096>(dst, src, n, st);
    if (n <= 16384) return launch_blob<16384>(dst, src, n, st);
    if (n <= kPlanBlobMax) return launch_blob<kPlanBlobMax>(dst, src, n, st);
    return -1;
}

}  // namespace smlm
