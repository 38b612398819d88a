// kernels_opt.cu -- the step after the path: AdamW over the fine-tune adapters'
// parameters, one flat fp32 buffer (master weights, exp_avg, exp_avg_sq, gradient) plus the bf16
// working copy the SMLM pools borrow.
//
// PAPER.md Table 5 trains with the HF Trainer at learning_rate 2e-5; its optimizer
// defaults (AdamW with decoupled weight decay, global gradient-norm clipping) are DESIGN.md R12.
// The fused cross-rank variant (smlm_adamw_step_reduce) sums the gradient slots the
// ranks wrote into each other's staging buffers (smlm_pool_set_grad_fanout) in rank order before
// the update -- the collective and the optimizer in one pass over HBM, deterministic, and
// identical on every rank.
// Masking: only the adapters whose parameters the caller placed in the buffer move.
//
// HBM-bound elementwise work (30 B/element: read g, p, m, v; write p, m, v and bf16 p; +4 B
// when the gradient is zeroed), so the design is about streaming: float4 loads/stores, a
// grid of a few CTAs per SM (grid-stride), no shared-memory staging.  With clipping on, a first
// pass reduces sum(g^2) into one fp32 partial per CTA (fixed grid -> fixed order); every CTA of
// the step kernel sums the partials in the same order in fp64, so the coefficient is identical
// everywhere and bitwise reproducible.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "device_types.h"
#include "pdl.cuh"

namespace smlm {

namespace {

constexpr int kOptT = 256;

__device__ __forceinline__ float block_sum(float x, float *red) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = x;
    __syncthreads();
    float s = 0.f;
    if (threadIdx.x == 0)
        for (int i = 0; i < kOptT / 32; ++i) s += red[i];
    return s;
}

// wait until the peers' gradient slots are complete (system-scope counter, see smlm_fanout_signal)
__device__ __forceinline__ void wait_ready(const int *ready, int target) {
    if (!ready) return;
    if (threadIdx.x == 0) {
        int v;
        do {
            asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(ready) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// gradient element i: the sum of the slots in rank order (one slot: the buffer itself)
__device__ __forceinline__ float4 grad4(const float4 *g4, int n_slots, size_t stride4, size_t i) {
    float4 x = __ldcs(g4 + i);
    for (int q = 1; q < n_slots; ++q) {
        const float4 y = __ldcs(g4 + (size_t)q * stride4 + i);
        x.x += y.x; x.y += y.y; x.z += y.z; x.w += y.w;
    }
    return x;
}
__device__ __forceinline__ float grad1(const float *g, int n_slots, size_t stride, size_t i) {
    float x = g[i];
    for (int q = 1; q < n_slots; ++q) x += g[(size_t)q * stride + i];
    return x;
}

__global__ void __launch_bounds__(kOptT) adamw_sumsq_kernel(const float *__restrict__ g, size_t n, float gscale,
                                                            float *__restrict__ partial, int n_slots, size_t slot_stride,
                                                            const int *ready, int ready_target) {
    __shared__ float red[kOptT / 32];
    pdl_wait();
    pdl_trigger();
    wait_ready(ready, ready_target);
    const size_t n4 = n / 4, stride = (size_t)gridDim.x * kOptT;
    const float4 *g4 = reinterpret_cast<const float4 *>(g);
    float acc = 0.f;
    for (size_t i = (size_t)blockIdx.x * kOptT + threadIdx.x; i < n4; i += stride) {
        float4 x = grad4(g4, n_slots, slot_stride / 4, i);
        x.x *= gscale; x.y *= gscale; x.z *= gscale; x.w *= gscale;
        acc = fmaf(x.x, x.x, acc);
        acc = fmaf(x.y, x.y, acc);
        acc = fmaf(x.z, x.z, acc);
        acc = fmaf(x.w, x.w, acc);
    }
    for (size_t i = 4 * n4 + (size_t)blockIdx.x * kOptT + threadIdx.x; i < n; i += stride) {
        const float x = grad1(g, n_slots, slot_stride, i) * gscale;
        acc = fmaf(x, x, acc);
    }
    const float s = block_sum(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__device__ __forceinline__ void adam1(float &p, float &m, float &v, float g, const AdamwArgs &a) {
    p *= a.decay;
    m = fmaf(a.beta1, m, (1.f - a.beta1) * g);
    v = fmaf(a.beta2, v, (1.f - a.beta2) * g * g);
    const float denom = sqrtf(v) * a.inv_bc2_sqrt + a.eps;
    p -= a.step_size * m / denom;
}

__global__ void __launch_bounds__(kOptT) adamw_step_kernel(const AdamwArgs a) {
    __shared__ float coef_s;
    pdl_wait();
    pdl_trigger();
    wait_ready(a.ready, a.ready_target);
    float coef = 1.f;
    if (a.partial) {
        // every CTA reduces the partials the same way (strided fp64 sums, then a fixed tree), so
        // the coefficient is the same everywhere and run to run
        __shared__ double red[kOptT];
        double s = 0.0;
        for (int i = threadIdx.x; i < a.n_partial; i += kOptT) s += (double)a.partial[i];
        red[threadIdx.x] = s;
        __syncthreads();
#pragma unroll
        for (int h = kOptT / 2; h > 0; h >>= 1) {
            if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const double c = (double)a.max_norm / (sqrt(red[0]) + 1e-6);
            coef_s = (float)(c < 1.0 ? c : 1.0);
        }
        __syncthreads();
        coef = coef_s;
    }
    const float gmul = a.gscale * coef;
    const size_t n4 = a.n / 4, stride = (size_t)gridDim.x * kOptT;
    float4 *p4 = reinterpret_cast<float4 *>(a.p), *m4 = reinterpret_cast<float4 *>(a.m);
    float4 *v4 = reinterpret_cast<float4 *>(a.v), *g4 = reinterpret_cast<float4 *>(a.g);
    float4 *z4 = g4 + (size_t)a.zero_slot * (a.slot_stride / 4);   // the slot zero_grad clears
    for (size_t i = (size_t)blockIdx.x * kOptT + threadIdx.x; i < n4; i += stride) {
        const float4 g = grad4(g4, a.n_slots, a.slot_stride / 4, i);
        float4 p = __ldcs(p4 + i), m = __ldcs(m4 + i), v = __ldcs(v4 + i);
        adam1(p.x, m.x, v.x, g.x * gmul, a);
        adam1(p.y, m.y, v.y, g.y * gmul, a);
        adam1(p.z, m.z, v.z, g.z * gmul, a);
        adam1(p.w, m.w, v.w, g.w * gmul, a);
        __stcs(p4 + i, p);
        __stcs(m4 + i, m);
        __stcs(v4 + i, v);
        if (a.zero_grad) __stcs(z4 + i, make_float4(0.f, 0.f, 0.f, 0.f));
        if (a.pb) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(p.x, p.y), hi = __floats2bfloat162_rn(p.z, p.w);
            uint2 u;
            u.x = *reinterpret_cast<uint32_t *>(&lo);
            u.y = *reinterpret_cast<uint32_t *>(&hi);
            __stcs(reinterpret_cast<uint2 *>(a.pb) + i, u);
        }
    }
    for (size_t i = 4 * n4 + (size_t)blockIdx.x * kOptT + threadIdx.x; i < a.n; i += stride) {
        float p = a.p[i], m = a.m[i], v = a.v[i];
        adam1(p, m, v, grad1(a.g, a.n_slots, a.slot_stride, i) * gmul, a);
        a.p[i] = p;
        a.m[i] = m;
        a.v[i] = v;
        if (a.zero_grad) a.g[(size_t)a.zero_slot * a.slot_stride + i] = 0.f;
        if (a.pb) reinterpret_cast<__nv_bfloat16 *>(a.pb)[i] = __float2bfloat16_rn(p);
    }
}

}  // namespace

// grid of the two passes: a few CTAs per SM, fewer for small buffers
int adamw_grid(int num_sms, size_t n) {
    const size_t want = (n / 4 + kOptT - 1) / kOptT;
    const size_t cap = (size_t)num_sms * 8;
    return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

int launch_adamw_sumsq(const AdamwArgs &a, float *partial, int grid, cudaStream_t st) {
    return (int)launch_pdl(adamw_sumsq_kernel, dim3(grid), dim3(kOptT), 0, st, (const float *)a.g, a.n, a.gscale,
                           partial, a.n_slots, a.slot_stride, a.ready, a.ready_target);
}

// fan-out completion: after this rank's gradient kernels (stream order), a system-scope release
// increment of every rank's ready counter (its own included)
__global__ void fanout_signal_kernel(FanoutFlags f) {
    pdl_wait();
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int q = 0; q < f.n; ++q)
            asm volatile("red.release.sys.global.add.s32 [%0], 1;" ::"l"(f.flag[q]) : "memory");
    }
}

// the consumer side without an optimizer: the stream waits until every rank's slots are complete
__global__ void fanout_wait_kernel(const int *ready, int target) {
    pdl_wait();
    pdl_trigger();
    wait_ready(ready, target);
}

int launch_fanout_wait(const int *ready, int target, cudaStream_t st) {
    return (int)launch_pdl(fanout_wait_kernel, dim3(1), dim3(32), 0, st, ready, target);
}

int launch_fanout_signal(const FanoutFlags &f, cudaStream_t st) {
    return (int)launch_pdl(fanout_signal_kernel, dim3(1), dim3(32), 0, st, f);
}

int launch_adamw_step(const AdamwArgs &a, int grid, cudaStream_t st) {
    return (int)launch_pdl(adamw_step_kernel, dim3(grid), dim3(kOptT), 0, st, a);
}

}  // namespace smlm
