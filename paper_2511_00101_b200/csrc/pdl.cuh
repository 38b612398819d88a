// pdl.cuh -- programmatic dependent launch (PDL) helpers.  Every kernel of a call chain is
// launched with programmatic stream serialization; inside, griddepcontrol.wait precedes the first
// global-memory access (the prologue -- barrier init, TMEM allocation, descriptor prefetch --
// overlaps the predecessor's tail) and griddepcontrol.launch_dependents lets the successor start
// its own prologue early.
#pragma once
#include <cuda_runtime.h>

#include <utility>

namespace smlm {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace smlm
