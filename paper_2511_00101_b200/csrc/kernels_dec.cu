// kernels_dec.cu -- K-split SIMT shrink for the short rows of MIXED batches.
//
// Short rows (decode / short segments) that ride in the CTA-pair GEMM next to long tiles get their
// rank-r intermediate here: V = A_u x per short row, split over 512-column chunks of `in`
// (128-bit loads, lane partials + shuffle trees), partials combined in fixed chunk order into the
// block-diagonal s*V operand of the GEMM's per-adapter expand K-blocks.  Pure decode batches take
// the single-launch kernel in kernels_dec3.cu instead.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "device_types.h"
#include "dropout.cuh"
#include "pdl.cuh"
#include "sm100.cuh"

namespace smlm {
using namespace sm100;

namespace {

__device__ __forceinline__ float warp_sum_d(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void bf16x8_f32(const uint4 &u, float (&f)[8]) {
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

// ------------------------------------------------------------------------------------------
// K-split shrink: CTA (block, chunk) computes partial V[i][j] = sum_{k in chunk} A_u[j][k] x_i[k]
// for the block's rows.  A warp covers the whole 512-column chunk (lane l owns columns
// [16 l, 16 l + 16): two 128-bit loads); warps take rows round-robin; a xor-shuffle tree reduces.
// The decomposition depends only on `in`, so a row's V never depends on its batch position.
// ------------------------------------------------------------------------------------------
constexpr int kChunk = 512;
constexpr int kRowsPerPass = 32;

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

// combine partials in chunk order -> block-diagonal s*V (bf16 [128, RP]) and V_save of block bi
// (256 threads; idx_of[128] and vals[128 * RP] in shared memory)
template <int RP>
__device__ __forceinline__ void shrink_combine_block(int bi, const DevBlock *__restrict__ blocks,
                                                     const DevShortRow *__restrict__ srows, int nch, int r,
                                                     const float *__restrict__ part, __nv_bfloat16 *__restrict__ Vbd,
                                                     __nv_bfloat16 *__restrict__ Vsave, int *idx_of, float *vals,
                                                     const DropArgs &drop) {
    const DevBlock blk = blocks[bi];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) idx_of[i] = -1;
    __syncthreads();
    for (int i = threadIdx.x; i < blk.nrows; i += blockDim.x) idx_of[srows[blk.row_begin + i].pos] = i;
    const float *src = part + (size_t)bi * nch * 128 * RP;
    for (int e = threadIdx.x; e < blk.nrows * RP; e += blockDim.x) {
        const int i = e / RP, j = e % RP;
        float v = 0.f;
        if (j < r) {
            float t[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) t[c] = c < nch ? __ldcg(src + (size_t)c * 128 * RP + i * RP + j) : 0.f;
            for (int c = 0; c < nch && c < 16; ++c) v += t[c];   // chunk order
            for (int c = 16; c < nch; ++c) v += __ldcg(src + (size_t)c * 128 * RP + i * RP + j);
            if (drop.on && srows[blk.row_begin + i].ft) v *= drop.scale;   // V~ of a dropout row
        }
        vals[i * RP + j] = v;
    }
    __syncthreads();
    __nv_bfloat16 *dst = Vbd + (size_t)bi * 128 * RP;
    for (int e = threadIdx.x; e < 128 * RP; e += blockDim.x) {
        const int p = e / RP, j = e % RP;
        const int i = idx_of[p];
        dst[e] = __float2bfloat16_rn(i < 0 ? 0.f : srows[blk.row_begin + i].scale * vals[i * RP + j]);
    }
    if (Vsave) {
        for (int e = threadIdx.x; e < blk.nrows * r; e += blockDim.x) {
            const int i = e / r, j = e % r;
            const DevShortRow sr = srows[blk.row_begin + i];
            if (sr.ft) Vsave[(size_t)sr.row * r + j] = __float2bfloat16_rn(vals[i * RP + j]);
        }
    }
}

template <int RP>
__global__ void __launch_bounds__(256) shrink_partial_kernel(const __nv_bfloat16 *__restrict__ X,
                                                             const SlotDev *__restrict__ slots,
                                                             const DevBlock *__restrict__ blocks,
                                                             const DevShortRow *__restrict__ srows, int in_f,
                                                             int r, float *__restrict__ part, int *ctr,
                                                             __nv_bfloat16 *__restrict__ Vbd,
                                                             __nv_bfloat16 *__restrict__ Vsave, const DropArgs drop) {
    // A_u[:, chunk] and the block's x rows [:, chunk] are staged in shared memory with coalesced
    // 128-bit loads (every byte read once); then warp w computes outputs (i, j) = w, w+8, ...:
    // lane l reduces columns [16 l, 16 l + 16) and a xor-shuffle tree finishes.
    extern __shared__ __align__(16) uint8_t sm[];
    __nv_bfloat16 *As = reinterpret_cast<__nv_bfloat16 *>(sm);                   // [RP][512]
    __nv_bfloat16 *Xs = As + RP * kChunk;                                         // [32][512]
    pdl_wait();
    pdl_trigger();
    const DevBlock blk = blocks[blockIdx.x];
    const int c = blockIdx.y, nch = gridDim.y;
    const __nv_bfloat16 *A = reinterpret_cast<const __nv_bfloat16 *>(slots[blk.slot].A);
    const int ra = slots[blk.slot].r;   // rows of A past the adapter's own rank are zero
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k0 = c * kChunk;
    for (int e = threadIdx.x; e < r * (kChunk / 8); e += 256) {
        const int j = e / (kChunk / 8), v = e % (kChunk / 8);
        if (j < ra)
            cp_async16(reinterpret_cast<uint4 *>(As) + e, reinterpret_cast<const uint4 *>(A + (size_t)j * in_f + k0) + v);
        else
            reinterpret_cast<uint4 *>(As)[e] = make_uint4(0, 0, 0, 0);
    }
    float *dst = part + ((size_t)blockIdx.x * nch + c) * 128 * RP;
    for (int rb = 0; rb < blk.nrows; rb += kRowsPerPass) {
        const int nr = min(kRowsPerPass, blk.nrows - rb);
        __syncthreads();
        for (int e = threadIdx.x; e < nr * (kChunk / 8); e += 256) {
            const int i = e / (kChunk / 8), v = e % (kChunk / 8);
            const int row = srows[blk.row_begin + rb + i].row;
            cp_async16(reinterpret_cast<uint4 *>(Xs) + e, reinterpret_cast<const uint4 *>(X + (size_t)row * in_f + k0) + v);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        if (drop.on) {   // LoRA dropout of FINETUNE rows: zero the dropped elements of the staged x rows
            for (int e = threadIdx.x; e < nr * (kChunk / 8); e += 256) {
                const int i = e / (kChunk / 8), v = e % (kChunk / 8);
                const DevShortRow sr = srows[blk.row_begin + rb + i];
                if (sr.ft) {
                    uint4 *p = reinterpret_cast<uint4 *>(Xs) + e;
                    *p = drop_mask8(drop, (uint32_t)sr.row, (uint32_t)(k0 + 8 * v), *p);
                }
            }
            __syncthreads();
        }
        for (int o = warp; o < nr * r; o += 8) {
            const int i = o / r, j = o % r;
            const uint4 *ap = reinterpret_cast<const uint4 *>(As + j * kChunk + 16 * lane);
            const uint4 *xp = reinterpret_cast<const uint4 *>(Xs + i * kChunk + 16 * lane);
            float a0[8], a1[8], x0[8], x1[8];
            bf16x8_f32(ap[0], a0);
            bf16x8_f32(ap[1], a1);
            bf16x8_f32(xp[0], x0);
            bf16x8_f32(xp[1], x1);
            float acc = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = fmaf(a0[e], x0[e], acc);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = fmaf(a1[e], x1[e], acc);
            acc = warp_sum_d(acc);
            if (lane == 0) dst[(rb + i) * RP + j] = acc;
        }
    }
    if (ctr) {
        // the last chunk of the block to finish combines it (no second launch): barrier, then one
        // gpu-scope fence + counter by thread 0 (split-K semaphore); the counter returns to 0
        __shared__ int s_last;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const int old = atomicAdd(ctr + blockIdx.x, 1);
            s_last = old == nch - 1;
            if (s_last) {
                ctr[blockIdx.x] = 0;
                __threadfence();
            }
        }
        __syncthreads();
        if (s_last) {
            // the staged A / X tiles are no longer needed: reuse the dynamic shared memory
            int *idx_of = reinterpret_cast<int *>(sm);
            float *vals = reinterpret_cast<float *>(sm + 512);
            shrink_combine_block<RP>(blockIdx.x, blocks, srows, nch, r, part, Vbd, Vsave, idx_of, vals, drop);
        }
    }
}

template <int RP>
__global__ void __launch_bounds__(256) shrink_combine_kernel(const DevBlock *__restrict__ blocks,
                                                             const DevShortRow *__restrict__ srows, int nch,
                                                             int r, const float *__restrict__ part,
                                                             __nv_bfloat16 *__restrict__ Vbd,
                                                             __nv_bfloat16 *__restrict__ Vsave, const DropArgs drop) {
    pdl_wait();
    pdl_trigger();
    __shared__ int idx_of[128];
    __shared__ float vals[128 * RP];
    shrink_combine_block<RP>(blockIdx.x, blocks, srows, nch, r, part, Vbd, Vsave, idx_of, vals, drop);
}

}  // namespace

int dec_chunks(int in_f) { return in_f / kChunk > 0 && in_f % kChunk == 0 ? in_f / kChunk : 0; }

int launch_shrink_split(const __nv_bfloat16 *X, const SlotDev *slots, const DevBlock *blocks,
                        const DevShortRow *srows, int n_blocks, int in_f, int r, int r_pad, float *part,
                        __nv_bfloat16 *Vbd, __nv_bfloat16 *Vsave, int *ctr, const DropArgs &drop, cudaStream_t st) {
    if (n_blocks == 0) return 0;
    const int nch = dec_chunks(in_f);
    dim3 g1(n_blocks, nch);
    cudaError_t e = cudaSuccess;
    switch (r_pad) {
        case 16:
            cudaFuncSetAttribute(shrink_partial_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (16 + kRowsPerPass) * kChunk * 2);
            e = launch_pdl(shrink_partial_kernel<16>, g1, dim3(256), (16 + kRowsPerPass) * kChunk * 2, st, X, slots, blocks, srows, in_f, r, part, ctr, Vbd, Vsave, drop);
            if (e != cudaSuccess || ctr) break;
            e = launch_pdl(shrink_combine_kernel<16>, dim3(n_blocks), dim3(256), 0, st, blocks, srows, nch, r, part, Vbd, Vsave, drop);
            break;
        case 32:
            cudaFuncSetAttribute(shrink_partial_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (32 + kRowsPerPass) * kChunk * 2);
            e = launch_pdl(shrink_partial_kernel<32>, g1, dim3(256), (32 + kRowsPerPass) * kChunk * 2, st, X, slots, blocks, srows, in_f, r, part, ctr, Vbd, Vsave, drop);
            if (e != cudaSuccess || ctr) break;
            e = launch_pdl(shrink_combine_kernel<32>, dim3(n_blocks), dim3(256), 0, st, blocks, srows, nch, r, part, Vbd, Vsave, drop);
            break;
        case 64:
            cudaFuncSetAttribute(shrink_partial_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (64 + kRowsPerPass) * kChunk * 2);
            e = launch_pdl(shrink_partial_kernel<64>, g1, dim3(256), (64 + kRowsPerPass) * kChunk * 2, st, X, slots, blocks, srows, in_f, r, part, ctr, Vbd, Vsave, drop);
            if (e != cudaSuccess || ctr) break;
            e = launch_pdl(shrink_combine_kernel<64>, dim3(n_blocks), dim3(256), 0, st, blocks, srows, nch, r, part, Vbd, Vsave, drop);
            break;
        default: return (int)cudaErrorInvalidValue;
    }
    return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}

}  // namespace smlm
