// Microbenchmark: the C2 decode layer-step's streaming ceiling.
// Two kernels per "layer-step" that do nothing but stream the bytes of the q/k/v call (~69 MB) and
// of the o call (~42 MB) from HBM into shared memory with 1-D bulk copies (a ring of stages per
// CTA), over 8 rotated buffer sets (every set > L2 / 8), replayed in a CUDA graph.  Variants:
//   pdl=0/1      programmatic stream serialisation between the two kernels
//   trig=0/1     griddepcontrol.launch_dependents at the start (1) or implicit at exit (0)
//   cps=1/2      CTAs per SM (2: half the ring per CTA, so the next kernel's CTAs fit beside the
//                current one's and start streaming before griddepcontrol.wait)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_ceiling stream_ceiling.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint32_t b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory"); }
__device__ __forceinline__ void mwait(uint32_t b, uint32_t ph) {
    uint32_t d;
    do { asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}" : "=r"(d) : "r"(b), "r"(ph) : "memory"); } while (!d);
}
__device__ __forceinline__ void bulk1d(uint32_t dst, const void *src, uint32_t n, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst), "l"(src), "r"(n), "r"(bar) : "memory");
}

constexpr uint32_t kChunk = 16384;
constexpr int STMAX = 16;
__device__ int g_sink;

// CTA b streams chunks b, b + grid, b + 2 grid, ... of [0, bytes)
__global__ void __launch_bounds__(32) kstream(const char *src, size_t bytes, int ST, int trig, int pre, const char *xb, int xr) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bars[STMAX];
    const uint32_t base = (su32(sm) + 1023) & ~1023u;
    if (trig) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) mbar_init(su32(&bars[s]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const size_t nch = bytes / kChunk;
    int n = 0;
    bool waited = false;
    for (size_t c = blockIdx.x; c < nch; c += gridDim.x, ++n) {
        // the first `pre` stages are issued before the grid-dependency wait (weights do not depend
        // on the previous kernel); the rest after it
        if (!waited && n >= pre) { asm volatile("griddepcontrol.wait;" ::: "memory"); waited = true; }
        const int s = n % ST;
        const uint32_t bar = su32(&bars[s]);
        if (n >= ST) mwait(bar, ((n / ST) & 1) ^ 1);
        // xr > 0: with every W chunk, xr chunks of the L2-resident 2 MiB "X" buffer (the A operand
        // copies every CTA pair of a split-K decode GEMM pulls from L2)
        expect_tx(bar, kChunk * (1 + xr));
        bulk1d(base + s * kChunk * (1 + xr), src + c * kChunk, kChunk, bar);
        for (int j = 0; j < xr; ++j)
            bulk1d(base + s * kChunk * (1 + xr) + (j + 1) * kChunk, xb + ((c * xr + j) % 128) * kChunk, kChunk, bar);
    }
    if (!waited) asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int m = n > ST ? n - ST : 0; m < n; ++m) mwait(su32(&bars[m % ST]), (m / ST) & 1);
    if (n == 0) g_sink = 1;
}

static const char *g_xb;
static void launch(const char *src, size_t bytes, int grid, int ST, int pdl, int trig, int pre, cudaStream_t st, int xr = 0) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32);
    cfg.dynamicSmemBytes = ST * kChunk * (1 + xr) + 1024;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, kstream, src, bytes, ST, trig, pre, g_xb, xr));
}

int main(int argc, char **argv) {
    const size_t b1 = 69ull << 20, b2 = 42ull << 20;   // q/k/v call, o call (rounded up to MiB)
    const int NS = 8;
    char *buf;
    CK(cudaMalloc(&buf, NS * (b1 + b2)));
    CK(cudaMemset(buf, 1, NS * (b1 + b2)));
    CK(cudaFuncSetAttribute(kstream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaMalloc((void **)&g_xb, 2 << 20));
    struct V { int cps, ST, pdl, trig, pre, xr; } vs[] = {
        {1, 12, 0, 0, 0}, {1, 12, 1, 0, 0}, {1, 12, 1, 1, 0}, {1, 12, 1, 1, 12},
        {2, 6, 0, 0, 0}, {2, 6, 1, 1, 0}, {2, 6, 1, 1, 6}, {2, 6, 1, 1, 1000},
        {1, 6, 1, 1, 6}, {3, 4, 1, 1, 4},
        {1, 6, 1, 1, 6, 1}, {1, 4, 1, 1, 4, 1}, {1, 3, 1, 1, 3, 2}, {2, 3, 1, 1, 3, 1}, {1, 6, 1, 1, 0, 1},
    };
    for (auto v : vs) {
        const int grid = 148 * v.cps;
        cudaGraph_t g;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
        for (int i = 0; i < NS; ++i) {
            const char *s = buf + i * (b1 + b2);
            launch(s, b1, grid, v.ST, v.pdl, v.trig, v.pre, st, v.xr);
            launch(s + b1, b2, grid, v.ST, v.pdl, v.trig, v.pre, st, v.xr);
        }
        CK(cudaStreamEndCapture(st, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        for (int w = 0; w < 5; ++w) CK(cudaGraphLaunch(ge, st));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        const int R = 20;
        CK(cudaEventRecord(e0, st));
        for (int r = 0; r < R; ++r) CK(cudaGraphLaunch(ge, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaStreamSynchronize(st));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = 1e3 * ms / (R * NS);
        const double roof = (b1 + b2) / 6.55e6 * 1.0;   // us at 6.55 TB/s
        printf("xr=%d cps=%d ST=%2d pdl=%d trig=%d pre=%4d : layer-step %.2f us  (%.2f TB/s, %.2f of 6.55 TB/s)\n", v.xr, v.cps, v.ST,
               v.pdl, v.trig, v.pre, us, (b1 + b2) / us / 1e6, roof / us);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
    }
    // isolated single launches of each size (no graph)
    for (int i = 0; i < 3; ++i) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        CK(cudaEventRecord(e0, st));
        launch(buf, b1, 148, 12, 0, 0, 0, st);
        CK(cudaEventRecord(e1, st));
        CK(cudaStreamSynchronize(st));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("isolated q/k/v-size stream: %.2f us\n", ms * 1e3);
    }
    return 0;
}
