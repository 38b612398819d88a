// kernels_simt.cu -- CUDA-core kernels of the SMLM path.
//
//  * shrink_short  (a3): V = A_a x for short/decode rows, grouped by adapter (each A_a streamed
//                        once per short tile); writes the block-diagonal s*V operand that the
//                        tensor-core kernel folds in, plus V_save of fine-tune rows.
//                        HBM-bound: 128-bit loads, lane partials + warp-shuffle trees.
//  * rows_shrink / rows_u: per-row V = A_a x and U = B_a^T dy for tile lists (backward without
//                        dX or without V_save, and the fp32 test mode).
//  * dA / dB     (a5): per-adapter token contractions dA = s U^T X, dB = s dY^T V, each adapter's
//                        fine-tune tiles visited in the canonical order (bitwise deterministic,
//                        no atomics).  PAPER.md P:420 (shared backward), P:422 (masking).
//  * fp32 test mode: warp-per-output kernels with chunked (lane partial + tree) accumulation.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "device_types.h"
#include "dropout.cuh"
#include "pdl.cuh"

namespace smlm {

namespace {

template <typename T> __device__ __forceinline__ float ld_f(const T *p);
template <> __device__ __forceinline__ float ld_f<float>(const float *p) { return __ldg(p); }
template <> __device__ __forceinline__ float ld_f<__nv_bfloat16>(const __nv_bfloat16 *p) {
    return __bfloat162float(*p);
}
template <typename T> __device__ __forceinline__ void st_f(T *p, float v);
template <> __device__ __forceinline__ void st_f<float>(float *p, float v) { *p = v; }
template <> __device__ __forceinline__ void st_f<__nv_bfloat16>(__nv_bfloat16 *p, float v) {
    *p = __float2bfloat16_rn(v);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4 &u, float (&f)[8]) {
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

// --------------------------------------------------------------------------------------
// shrink_short: one CTA per (short tile, adapter) block.  8 warps split K = in into 8 slices;
// lane l of a warp owns 16-byte chunks l, l+32, ... of its slice.  For <= 4 rows at a time and
// 16 ranks at a time, lane partials are reduced by a xor-shuffle tree and then across warps in
// fixed order (position independent: a row's V depends only on its data).
// --------------------------------------------------------------------------------------
template <int RP>
__global__ void __launch_bounds__(256) shrink_short_kernel(const __nv_bfloat16 *__restrict__ X,
                                                           const SlotDev *__restrict__ slots,
                                                           const DevBlock *__restrict__ blocks,
                                                           const DevShortRow *__restrict__ srows, int in_f, int r,
                                                           __nv_bfloat16 *__restrict__ Vbd,
                                                           __nv_bfloat16 *__restrict__ Vsave, const DropArgs drop) {
    const DevBlock blk = blocks[blockIdx.x];
    const __nv_bfloat16 *A = reinterpret_cast<const __nv_bfloat16 *>(slots[blk.slot].A);
    const int ra = slots[blk.slot].r;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ float part[8][4][16];
    __shared__ float vbuf[128][RP + 1];
    __shared__ int pos_of[128];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) pos_of[i] = -1;
    __syncthreads();
    const int slice = in_f / 8;          // multiple of 8 (in % 64 == 0)
    const int k0 = warp * slice;
    const int nvec = slice / 8;          // 16-byte vectors in this warp's slice
    for (int rb = 0; rb < blk.nrows; rb += 4) {
        const int nr = min(4, blk.nrows - rb);
        int rows[4];
        bool dmask[4];   // LoRA dropout on this (FINETUNE) row
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const DevShortRow sr = srows[blk.row_begin + rb + min(i, nr - 1)];
            rows[i] = sr.row;
            dmask[i] = drop.on && sr.ft;
        }
        for (int jg = 0; jg < r; jg += 16) {
            float acc[4][16];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[i][j] = 0.f;
            for (int v = lane; v < nvec; v += 32) {
                const int k = k0 + 8 * v;
                float xf[4][8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    uint4 xu = *reinterpret_cast<const uint4 *>(X + (size_t)rows[i] * in_f + k);
                    if (dmask[i]) xu = drop_mask8(drop, (uint32_t)rows[i], (uint32_t)k, xu);
                    bf16x8_to_f32(xu, xf[i]);
                }
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    if (jg + j < ra) {   // rows past the adapter's own rank are zero
                        float af[8];
                        uint4 au = *reinterpret_cast<const uint4 *>(A + (size_t)(jg + j) * in_f + k);
                        bf16x8_to_f32(au, af);
#pragma unroll
                        for (int i = 0; i < 4; ++i)
#pragma unroll
                            for (int e = 0; e < 8; ++e) acc[i][j] = fmaf(af[e], xf[i][e], acc[i][j]);
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    float s = warp_sum(acc[i][j]);
                    if (lane == 0) part[warp][i][j] = s;
                }
            __syncthreads();
            if (threadIdx.x < 64) {
                const int i = threadIdx.x >> 4, j = threadIdx.x & 15;
                float s = 0.f;
#pragma unroll
                for (int w = 0; w < 8; ++w) s += part[w][i][j];
                if (i < nr && jg + j < RP)
                    vbuf[rb + i][jg + j] = (drop.on && srows[blk.row_begin + rb + i].ft) ? s * drop.scale : s;
            }
            __syncthreads();
        }
    }
    // zero ranks r..RP-1 (TMA-padded lanes of the MMA operand must be 0)
    for (int e = threadIdx.x; e < blk.nrows * RP; e += blockDim.x) {
        int i = e / RP, j = e % RP;
        if (j >= r) vbuf[i][j] = 0.f;
    }
    for (int i = threadIdx.x; i < blk.nrows; i += blockDim.x) pos_of[srows[blk.row_begin + i].pos] = i;
    __syncthreads();
    // block-diagonal operand: row p of this block = s*V of the block's row at position p, else 0
    __nv_bfloat16 *dst = Vbd + (size_t)blockIdx.x * 128 * RP;
    for (int e = threadIdx.x; e < 128 * RP; e += blockDim.x) {
        const int p = e / RP, j = e % RP;
        const int i = pos_of[p];
        float v = 0.f;
        if (i >= 0) v = srows[blk.row_begin + i].scale * vbuf[i][j];
        dst[e] = __float2bfloat16_rn(v);
    }
    if (Vsave) {
        for (int e = threadIdx.x; e < blk.nrows * r; e += blockDim.x) {
            const int i = e / r, j = e % r;
            const DevShortRow sr = srows[blk.row_begin + i];
            if (sr.ft) Vsave[(size_t)sr.row * r + j] = __float2bfloat16_rn(vbuf[i][j]);
        }
    }
}

// --------------------------------------------------------------------------------------
// Per-row kernels over a tile list (warp per row).  Lanes split the reduction dimension with
// stride 32; each lane keeps RP partials; a xor-shuffle tree finishes (chunked accumulation).
// --------------------------------------------------------------------------------------
// V[t][j] = sum_k A[j][k] x[t][k]   (tiles with slot >= 0)
template <typename T, int RP>
__global__ void __launch_bounds__(256) rows_shrink_kernel(const DevTile *__restrict__ tiles,
                                                          const SlotDev *__restrict__ slots,
                                                          const T *__restrict__ X, int in_f, int r,
                                                          float *__restrict__ Vf, T *__restrict__ Vsave,
                                                          int ft_only_vsave, const DropArgs drop) {
    const DevTile t = tiles[blockIdx.x];
    if (t.slot < 0) return;
    const bool dm = drop.on && (t.flags & kTileFT);   // LoRA dropout: V~ = A (keep * x) / (1 - p)
    const T *A = reinterpret_cast<const T *>(slots[t.slot].A);
    const int ra = slots[t.slot].r;   // rows of A past the adapter's own rank are zero
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int m = blockIdx.y * 8 + warp; m < t.rows; m += gridDim.y * 8) {
        const int row = t.row0 + m;
        const T *x = X + (size_t)row * in_f;
        float acc[RP];
#pragma unroll
        for (int j = 0; j < RP; ++j) acc[j] = 0.f;
        for (int k = lane; k < in_f; k += 32) {
            float xv = ld_f(x + k);
            if (dm && !drop_keep(drop, (uint32_t)row, (uint32_t)k)) xv = 0.f;
#pragma unroll
            for (int j = 0; j < RP; ++j)
                if (j < ra) acc[j] = fmaf(ld_f(A + (size_t)j * in_f + k), xv, acc[j]);
        }
#pragma unroll
        for (int j = 0; j < RP; ++j) {
            float s = warp_sum(acc[j]);
            if (dm) s *= drop.scale;
            if (lane == 0 && j < r) {
                if (Vf) Vf[(size_t)row * r + j] = s;
                if (Vsave && (!ft_only_vsave || (t.flags & kTileFT))) st_f(Vsave + (size_t)row * r + j, s);
            }
        }
    }
}

// U[t][j] = sum_o dy[t][o] B[o][j]   (tiles with slot >= 0)
// Writes fp32 U [S,r] (Uf) and/or the tile-compact bf16 s*U [n_tiles*128, RP] (sUt, zero-padded).
template <typename T, int RP>
__global__ void __launch_bounds__(256) rows_u_kernel(const DevTile *__restrict__ tiles,
                                                     const SlotDev *__restrict__ slots,
                                                     const T *__restrict__ dY, int out_f, int r,
                                                     float *__restrict__ Uf, __nv_bfloat16 *__restrict__ sUt) {
    const DevTile t = tiles[blockIdx.x];
    if (t.slot < 0) return;
    const T *B = reinterpret_cast<const T *>(slots[t.slot].B);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int m = blockIdx.y * 8 + warp; m < 128; m += gridDim.y * 8) {
        if (m >= t.rows) {
            if (sUt)
                for (int j = lane; j < RP; j += 32) sUt[((size_t)blockIdx.x * 128 + m) * RP + j] = __float2bfloat16_rn(0.f);
            continue;
        }
        const int row = t.row0 + m;
        const T *dy = dY + (size_t)row * out_f;
        float acc[RP];
#pragma unroll
        for (int j = 0; j < RP; ++j) acc[j] = 0.f;
        for (int o = lane; o < out_f; o += 32) {
            const float g = ld_f(dy + o);
#pragma unroll
            for (int j = 0; j < RP; ++j)
                if (j < r) acc[j] = fmaf(ld_f(B + (size_t)o * r + j), g, acc[j]);
        }
#pragma unroll
        for (int j = 0; j < RP; ++j) {
            float s = warp_sum(acc[j]);
            if (lane == 0) {
                if (Uf && j < r) Uf[(size_t)row * r + j] = s;
                if (sUt) sUt[((size_t)blockIdx.x * 128 + m) * RP + j] = __float2bfloat16_rn(j < r ? t.scale * s : 0.f);
            }
        }
    }
}

// tile-compact bf16 s*V [n_tiles*128, RP] from V_save (bf16) or the fp32 recompute, zero-padded
template <typename TV, int RP>
__global__ void __launch_bounds__(128) prep_sv_kernel(const DevTile *__restrict__ tiles, const TV *__restrict__ V,
                                                      int r, __nv_bfloat16 *__restrict__ sVt) {
    pdl_wait();
    pdl_trigger();
    const DevTile t = tiles[blockIdx.x];
    const int m = threadIdx.x;
    __nv_bfloat16 *dst = sVt + ((size_t)blockIdx.x * 128 + m) * RP;
#pragma unroll
    for (int j = 0; j < RP; ++j) {
        float v = 0.f;
        if (t.slot >= 0 && m < t.rows && j < r) v = t.scale * ld_f(V + (size_t)(t.row0 + m) * r + j);
        dst[j] = __float2bfloat16_rn(v);
    }
}

// --------------------------------------------------------------------------------------
// dA_a[j][k] = sum over a's fine-tune tiles (canonical order) and rows: (s U[t][j]) x[t][k]
// grid (ceil(in/128), n_groups), 128 threads; thread owns column k.
// --------------------------------------------------------------------------------------
template <typename T, int RP>
__global__ void __launch_bounds__(128) dA_kernel(const DevTile *__restrict__ tiles,
                                                 const GradGroup *__restrict__ groups,
                                                 const T *__restrict__ X, const float *__restrict__ Uf,
                                                 int in_f, int r, int accumulate, const DropArgs drop) {
    const GradGroup g = groups[blockIdx.y];
    if (!g.dA) return;
    const int k = blockIdx.x * 128 + threadIdx.x;
    __shared__ float su[64][RP];  // (s * U) rows, staged 64 at a time
    float acc[RP];
#pragma unroll
    for (int j = 0; j < RP; ++j) acc[j] = 0.f;
    for (int ti = 0; ti < g.n_tiles; ++ti) {
        const DevTile t = tiles[g.tile_begin + ti];
        for (int m0 = 0; m0 < t.rows; m0 += 64) {
            const int nm = min(64, t.rows - m0);
            __syncthreads();
            for (int e = threadIdx.x; e < nm * RP; e += 128) {
                const int i = e / RP, j = e % RP;
                su[i][j] = j < r ? t.scale * Uf[(size_t)(t.row0 + m0 + i) * r + j] : 0.f;
            }
            __syncthreads();
            if (k < in_f) {
                for (int i = 0; i < nm; ++i) {
                    float xv = ld_f(X + (size_t)(t.row0 + m0 + i) * in_f + k);
                    if (drop.on && !drop_keep(drop, (uint32_t)(t.row0 + m0 + i), (uint32_t)k)) xv = 0.f;
#pragma unroll
                    for (int j = 0; j < RP; ++j) acc[j] = fmaf(su[i][j], xv, acc[j]);
                }
            }
        }
    }
    if (k < in_f) {
#pragma unroll
        for (int j = 0; j < RP; ++j) {
            if (j < r) {
                float *p = g.dA + (size_t)j * in_f + k;
                const float v = drop.on ? acc[j] * drop.scale : acc[j];   // x~ = keep * x / (1 - p)
                *p = accumulate ? *p + v : v;
            }
        }
    }
}

// dB_a[o][j] = sum_t (s V[t][j]) dy[t][o];  V from V_save (type TV) or fp32 workspace
template <typename T, typename TV, int RP>
__global__ void __launch_bounds__(128) dB_kernel(const DevTile *__restrict__ tiles,
                                                 const GradGroup *__restrict__ groups,
                                                 const T *__restrict__ dY, const TV *__restrict__ V,
                                                 int out_f, int r, int accumulate) {
    const GradGroup g = groups[blockIdx.y];
    if (!g.dB) return;
    const int o = blockIdx.x * 128 + threadIdx.x;
    __shared__ float sv[64][RP];
    float acc[RP];
#pragma unroll
    for (int j = 0; j < RP; ++j) acc[j] = 0.f;
    for (int ti = 0; ti < g.n_tiles; ++ti) {
        const DevTile t = tiles[g.tile_begin + ti];
        for (int m0 = 0; m0 < t.rows; m0 += 64) {
            const int nm = min(64, t.rows - m0);
            __syncthreads();
            for (int e = threadIdx.x; e < nm * RP; e += 128) {
                const int i = e / RP, j = e % RP;
                sv[i][j] = j < r ? t.scale * ld_f(V + (size_t)(t.row0 + m0 + i) * r + j) : 0.f;
            }
            __syncthreads();
            if (o < out_f) {
                for (int i = 0; i < nm; ++i) {
                    const float gv = ld_f(dY + (size_t)(t.row0 + m0 + i) * out_f + o);
#pragma unroll
                    for (int j = 0; j < RP; ++j) acc[j] = fmaf(sv[i][j], gv, acc[j]);
                }
            }
        }
    }
    if (o < out_f) {
        float *p = g.dB + (size_t)o * r;
#pragma unroll
        for (int j = 0; j < RP; ++j)
            if (j < r) p[j] = accumulate ? p[j] + acc[j] : acc[j];
    }
}

// --------------------------------------------------------------------------------------
// fp32 test mode: warp per output element.
// --------------------------------------------------------------------------------------
// y[t][n] = (W ? sum_k x[t][k] W[n][k] : y[t][n]) + s * sum_j B[n][j] V[t][j]
__global__ void __launch_bounds__(256) f32_fwd_kernel(const DevTile *__restrict__ tiles,
                                                      const SlotDev *__restrict__ slots,
                                                      const float *__restrict__ X, const float *__restrict__ W,
                                                      float *__restrict__ Y, const float *__restrict__ Vf,
                                                      int in_f, int out_f, int r) {
    const DevTile t = tiles[blockIdx.x >> 7];
    const int m = blockIdx.x & 127;
    if (m >= t.rows) return;
    const int row = t.row0 + m;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = blockIdx.y * 8 + warp;
    if (n >= out_f) return;
    float base;
    if (W) {
        float acc = 0.f;
        for (int k = lane; k < in_f; k += 32) acc = fmaf(X[(size_t)row * in_f + k], W[(size_t)n * in_f + k], acc);
        base = warp_sum(acc);
    } else {
        base = Y[(size_t)row * out_f + n];
    }
    if (lane == 0) {
        float lora = 0.f;
        if (t.slot >= 0) {
            const float *B = reinterpret_cast<const float *>(slots[t.slot].B);
            for (int j = 0; j < r; ++j) lora = fmaf(B[(size_t)n * r + j], Vf[(size_t)row * r + j], lora);
        }
        Y[(size_t)row * out_f + n] = base + t.scale * lora;
    }
}

// dx[t][k] = sum_o dy[t][o] W[o][k] + s * sum_j U[t][j] A[j][k]
__global__ void __launch_bounds__(256) f32_dx_kernel(const DevTile *__restrict__ tiles,
                                                     const SlotDev *__restrict__ slots,
                                                     const float *__restrict__ dY, const float *__restrict__ W,
                                                     float *__restrict__ dX, const float *__restrict__ Uf,
                                                     int in_f, int out_f, int r, const DropArgs drop) {
    const DevTile t = tiles[blockIdx.x >> 7];
    const int m = blockIdx.x & 127;
    if (m >= t.rows) return;
    const int row = t.row0 + m;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = blockIdx.y * 8 + warp;
    if (k >= in_f) return;
    float acc = 0.f;
    for (int o = lane; o < out_f; o += 32) acc = fmaf(dY[(size_t)row * out_f + o], W[(size_t)o * in_f + k], acc);
    const float base = warp_sum(acc);
    if (lane == 0) {
        float lora = 0.f;
        if (t.slot >= 0) {
            const float *A = reinterpret_cast<const float *>(slots[t.slot].A);
            for (int j = 0; j < r; ++j) lora = fmaf(Uf[(size_t)row * r + j], A[(size_t)j * in_f + k], lora);
            if (drop.on) lora *= drop_keep(drop, (uint32_t)row, (uint32_t)k) ? drop.scale : 0.f;   // d dropout(x)/dx
        }
        dX[(size_t)row * in_f + k] = base + t.scale * lora;
    }
}

inline int rp_of(int r) { return r <= 16 ? 16 : (r <= 32 ? 32 : 64); }

}  // namespace

int launch_shrink_short(const __nv_bfloat16 *X, const SlotDev *slots, const DevBlock *blocks,
                        const DevShortRow *srows, int n_blocks, int in_f, int r, int r_pad,
                        __nv_bfloat16 *Vbd, __nv_bfloat16 *Vsave, const DropArgs &drop, cudaStream_t st) {
    if (n_blocks == 0) return 0;
    switch (r_pad) {
        case 16: shrink_short_kernel<16><<<n_blocks, 256, 0, st>>>(X, slots, blocks, srows, in_f, r, Vbd, Vsave, drop); break;
        case 32: shrink_short_kernel<32><<<n_blocks, 256, 0, st>>>(X, slots, blocks, srows, in_f, r, Vbd, Vsave, drop); break;
        case 64: shrink_short_kernel<64><<<n_blocks, 256, 0, st>>>(X, slots, blocks, srows, in_f, r, Vbd, Vsave, drop); break;
        default: return (int)cudaErrorInvalidValue;
    }
    return (int)cudaGetLastError();
}

template <typename T>
int launch_rows_shrink(const DevTile *tiles, int n_tiles, const SlotDev *slots, const T *X, int in_f, int r,
                       float *Vf, T *Vsave, int ft_only, const DropArgs &drop, cudaStream_t st) {
    if (n_tiles == 0) return 0;
    dim3 grid(n_tiles, 16);
    switch (rp_of(r)) {
        case 16: rows_shrink_kernel<T, 16><<<grid, 256, 0, st>>>(tiles, slots, X, in_f, r, Vf, Vsave, ft_only, drop); break;
        case 32: rows_shrink_kernel<T, 32><<<grid, 256, 0, st>>>(tiles, slots, X, in_f, r, Vf, Vsave, ft_only, drop); break;
        default: rows_shrink_kernel<T, 64><<<grid, 256, 0, st>>>(tiles, slots, X, in_f, r, Vf, Vsave, ft_only, drop); break;
    }
    return (int)cudaGetLastError();
}
template int launch_rows_shrink<float>(const DevTile *, int, const SlotDev *, const float *, int, int, float *,
                                       float *, int, const DropArgs &, cudaStream_t);
template int launch_rows_shrink<__nv_bfloat16>(const DevTile *, int, const SlotDev *, const __nv_bfloat16 *, int,
                                               int, float *, __nv_bfloat16 *, int, const DropArgs &, cudaStream_t);

template <typename T>
int launch_rows_u(const DevTile *tiles, int n_tiles, const SlotDev *slots, const T *dY, int out_f, int r, float *Uf,
                  __nv_bfloat16 *sUt, int r_pad, cudaStream_t st) {
    if (n_tiles == 0) return 0;
    dim3 grid(n_tiles, 16);
    switch (sUt ? r_pad : rp_of(r)) {
        case 16: rows_u_kernel<T, 16><<<grid, 256, 0, st>>>(tiles, slots, dY, out_f, r, Uf, sUt); break;
        case 32: rows_u_kernel<T, 32><<<grid, 256, 0, st>>>(tiles, slots, dY, out_f, r, Uf, sUt); break;
        default: rows_u_kernel<T, 64><<<grid, 256, 0, st>>>(tiles, slots, dY, out_f, r, Uf, sUt); break;
    }
    return (int)cudaGetLastError();
}
template int launch_rows_u<float>(const DevTile *, int, const SlotDev *, const float *, int, int, float *,
                                  __nv_bfloat16 *, int, cudaStream_t);
template int launch_rows_u<__nv_bfloat16>(const DevTile *, int, const SlotDev *, const __nv_bfloat16 *, int, int,
                                          float *, __nv_bfloat16 *, int, cudaStream_t);

template <typename TV>
int launch_prep_sv(const DevTile *tiles, int n_tiles, const TV *V, int r, int r_pad, __nv_bfloat16 *sVt,
                   cudaStream_t st) {
    if (n_tiles == 0) return 0;
    switch (r_pad) {
        case 16: return (int)launch_pdl(prep_sv_kernel<TV, 16>, dim3(n_tiles), dim3(128), 0, st, tiles, V, r, sVt);
        case 32: return (int)launch_pdl(prep_sv_kernel<TV, 32>, dim3(n_tiles), dim3(128), 0, st, tiles, V, r, sVt);
        default: return (int)launch_pdl(prep_sv_kernel<TV, 64>, dim3(n_tiles), dim3(128), 0, st, tiles, V, r, sVt);
    }
}
template int launch_prep_sv<float>(const DevTile *, int, const float *, int, int, __nv_bfloat16 *, cudaStream_t);
template int launch_prep_sv<__nv_bfloat16>(const DevTile *, int, const __nv_bfloat16 *, int, int, __nv_bfloat16 *,
                                           cudaStream_t);

size_t grad_group_bytes() { return sizeof(GradGroup); }
void fill_grad_group(void *dst, int slot, int tile_begin, int n_tiles, int r, float *dA, float *dB) {
    GradGroup g{slot, tile_begin, n_tiles, r, dA, dB};
    *reinterpret_cast<GradGroup *>(dst) = g;
}

template <typename T, typename TV>
int launch_dadb(const DevTile *tiles, const void *groups, int n_groups, const T *X, const T *dY, const float *Uf,
                const TV *V, int in_f, int out_f, int r, int accumulate, const DropArgs &drop, cudaStream_t st) {
    if (n_groups == 0) return 0;
    const GradGroup *g = reinterpret_cast<const GradGroup *>(groups);
    dim3 ga((in_f + 127) / 128, n_groups), gb((out_f + 127) / 128, n_groups);
    switch (rp_of(r)) {
        case 16:
            dA_kernel<T, 16><<<ga, 128, 0, st>>>(tiles, g, X, Uf, in_f, r, accumulate, drop);
            dB_kernel<T, TV, 16><<<gb, 128, 0, st>>>(tiles, g, dY, V, out_f, r, accumulate);
            break;
        case 32:
            dA_kernel<T, 32><<<ga, 128, 0, st>>>(tiles, g, X, Uf, in_f, r, accumulate, drop);
            dB_kernel<T, TV, 32><<<gb, 128, 0, st>>>(tiles, g, dY, V, out_f, r, accumulate);
            break;
        default:
            dA_kernel<T, 64><<<ga, 128, 0, st>>>(tiles, g, X, Uf, in_f, r, accumulate, drop);
            dB_kernel<T, TV, 64><<<gb, 128, 0, st>>>(tiles, g, dY, V, out_f, r, accumulate);
            break;
    }
    return (int)cudaGetLastError();
}
template int launch_dadb<float, float>(const DevTile *, const void *, int, const float *, const float *,
                                       const float *, const float *, int, int, int, int, const DropArgs &, cudaStream_t);
template int launch_dadb<__nv_bfloat16, __nv_bfloat16>(const DevTile *, const void *, int, const __nv_bfloat16 *,
                                                       const __nv_bfloat16 *, const float *, const __nv_bfloat16 *,
                                                       int, int, int, int, const DropArgs &, cudaStream_t);
template int launch_dadb<__nv_bfloat16, float>(const DevTile *, const void *, int, const __nv_bfloat16 *,
                                               const __nv_bfloat16 *, const float *, const float *, int, int, int,
                                               int, const DropArgs &, cudaStream_t);

int launch_f32_fwd(const DevTile *tiles, int n_tiles, const SlotDev *slots, const float *X, const float *W, float *Y,
                   const float *Vf, int in_f, int out_f, int r, cudaStream_t st) {
    if (n_tiles == 0) return 0;
    dim3 grid(n_tiles * 128, (out_f + 7) / 8);
    f32_fwd_kernel<<<grid, 256, 0, st>>>(tiles, slots, X, W, Y, Vf, in_f, out_f, r);
    return (int)cudaGetLastError();
}

int launch_f32_dx(const DevTile *tiles, int n_tiles, const SlotDev *slots, const float *dY, const float *W, float *dX,
                  const float *Uf, int in_f, int out_f, int r, const DropArgs &drop, cudaStream_t st) {
    if (n_tiles == 0) return 0;
    dim3 grid(n_tiles * 128, (in_f + 7) / 8);
    f32_dx_kernel<<<grid, 256, 0, st>>>(tiles, slots, dY, W, dX, Uf, in_f, out_f, r, drop);
    return (int)cudaGetLastError();
}

}  // namespace smlm
