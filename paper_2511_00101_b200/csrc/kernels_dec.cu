// kernels_dec.cu -- the decode / short-row path, HBM-bound.
//
// PAPER.md P:687 (§4.2): decode throughput plateaus "indicating that the GPU memory access
// bottleneck has been hit" -- a decode batch is a skinny product (few hundred rows) that must
// stream W at HBM speed.  Orientation is transposed so the tensor core's M dimension runs over
// W rows and N over the decode rows:
//     D[n, m] = sum_k W[n0+n, k] x_m[k]  +  sum_u B_u[n0+n, :] (s V)_u[m, :]^T
// One work item = (128 W rows, group of <= 2 short tiles = <= 256 decode rows, K split).  W is
// streamed once from HBM (A operand, K-major), the decode rows' X tiles come from L2 (B operand).
// Split K spreads the stream over >= 148 CTAs; each split writes an fp32 partial tile and the
// last-arriving CTA of an item sums the partials in split order (deterministic) and stores bf16
// Y = base + LoRA in one pass (the base output is fused with the expand, no read-modify-write).
// The shrink runs first as a K-split SIMT pass (128-bit loads, lane partials + shuffle trees)
// whose partials are combined in fixed order into the block-diagonal s*V operand.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "device_types.h"
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

template <int RP>
__global__ void __launch_bounds__(256) shrink_partial_kernel(const __nv_bfloat16 *__restrict__ X,
                                                             const SlotDev *__restrict__ slots,
                                                             const DevBlock *__restrict__ blocks,
                                                             const DevShortRow *__restrict__ srows, int in_f,
                                                             int r, float *__restrict__ part) {
    const DevBlock blk = blocks[blockIdx.x];
    const int c = blockIdx.y, nch = gridDim.y;
    const __nv_bfloat16 *A = reinterpret_cast<const __nv_bfloat16 *>(slots[blk.slot].A);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = c * kChunk + 16 * lane;
    float *dst = part + ((size_t)blockIdx.x * nch + c) * 128 * RP;
    for (int i = warp; i < blk.nrows; i += 8) {
        const int row = srows[blk.row_begin + i].row;
        float xf[16];
        {
            const uint4 *xp = reinterpret_cast<const uint4 *>(X + (size_t)row * in_f + k);
            float t[8];
            bf16x8_f32(__ldg(xp), t);
#pragma unroll
            for (int e = 0; e < 8; ++e) xf[e] = t[e];
            bf16x8_f32(__ldg(xp + 1), t);
#pragma unroll
            for (int e = 0; e < 8; ++e) xf[8 + e] = t[e];
        }
#pragma unroll 4
        for (int j = 0; j < r; ++j) {
            const uint4 *ap = reinterpret_cast<const uint4 *>(A + (size_t)j * in_f + k);
            float a0[8], a1[8];
            bf16x8_f32(__ldg(ap), a0);
            bf16x8_f32(__ldg(ap + 1), a1);
            float acc = 0.f;
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = fmaf(a0[e], xf[e], acc);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = fmaf(a1[e], xf[8 + e], acc);
            acc = warp_sum_d(acc);
            if (lane == 0) dst[i * RP + j] = acc;
        }
    }
}

// combine partials in chunk order -> block-diagonal s*V (bf16 [128, RP]) and V_save
template <int RP>
__global__ void __launch_bounds__(128) shrink_combine_kernel(const DevBlock *__restrict__ blocks,
                                                             const DevShortRow *__restrict__ srows, int nch,
                                                             int r, const float *__restrict__ part,
                                                             __nv_bfloat16 *__restrict__ Vbd,
                                                             __nv_bfloat16 *__restrict__ Vsave) {
    const DevBlock blk = blocks[blockIdx.x];
    __shared__ int idx_of[128];
    idx_of[threadIdx.x] = -1;
    __syncthreads();
    for (int i = threadIdx.x; i < blk.nrows; i += blockDim.x) idx_of[srows[blk.row_begin + i].pos] = i;
    __syncthreads();
    const int p = threadIdx.x;  // row position inside the short tile
    const int i = idx_of[p];
    __nv_bfloat16 *dst = Vbd + ((size_t)blockIdx.x * 128 + p) * RP;
    if (i < 0) {
#pragma unroll
        for (int j = 0; j < RP; ++j) dst[j] = __float2bfloat16_rn(0.f);
        return;
    }
    const DevShortRow sr = srows[blk.row_begin + i];
    const float *src = part + (size_t)blockIdx.x * nch * 128 * RP + (size_t)i * RP;
#pragma unroll
    for (int j = 0; j < RP; ++j) {
        float v = 0.f;
        if (j < r)
            for (int c = 0; c < nch; ++c) v += src[(size_t)c * 128 * RP + j];
        dst[j] = __float2bfloat16_rn(sr.scale * v);
        if (Vsave && sr.ft && j < r) Vsave[(size_t)sr.row * r + j] = __float2bfloat16_rn(v);
    }
}

// ------------------------------------------------------------------------------------------
// transposed decode GEMM with split K
// ------------------------------------------------------------------------------------------
constexpr int kDThreads = 256;
constexpr uint32_t kDA = 128 * 128;   // W tile 128 rows x 64 k
constexpr uint32_t kDB = 256 * 128;   // X tiles: up to 256 decode rows x 64 k
constexpr uint32_t kDStage = kDA + kDB;

__device__ __forceinline__ void dec_item(const DecArgs &a, int w, int &nt, int &grp, int &split) {
    split = w % a.ksplit;
    const int rest = w / a.ksplit;
    grp = rest % a.n_groups;
    nt = rest / a.n_groups;
}

template <int RP>
__global__ void __launch_bounds__(kDThreads, 1) smlm_dec_kernel(const __grid_constant__ DecArgs args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    constexpr uint32_t RB = RP * 2;
    constexpr uint32_t kSwR = RB >= 128 ? kSw128 : (RB == 64 ? kSw64 : kSw32);
    const int ST = args.stages;
    const uint32_t bar = base + ST * kDStage;
    auto full_bar = [&](int s) { return bar + 8u * s; };
    auto empty_bar = [&](int s) { return bar + 8u * (ST + s); };
    const uint32_t accf0 = bar + 16u * ST;   // acc_full[2] then acc_empty[2]
    const uint32_t tmem_slot = accf0 + 32;
    auto a_addr = [&](int s) { return base + s * kDStage; };
    auto b_addr = [&](int s) { return base + s * kDStage + kDA; };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        mbar_init(accf0 + 0, 1);
        mbar_init(accf0 + 8, 1);
        mbar_init(accf0 + 16, 128);
        mbar_init(accf0 + 24, 128);
        fence_mbar_init();
        tma_prefetch_desc(&args.tmW);
        tma_prefetch_desc(&args.tmX);
        tma_prefetch_desc(&args.tmV);
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t *>(base_ptr + (tmem_slot - base));
    const int total = args.n_nt * args.n_groups * args.ksplit;
    const int nkb = args.K / kBK;

    auto kb_range = [&](int split, int &kb0, int &kb1) {
        const int q = nkb / args.ksplit, rm = nkb % args.ksplit;
        kb0 = split * q + min(split, rm);
        kb1 = kb0 + q + (split < rm ? 1 : 0);
    };

    if (warp == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            int nt, grp, split;
            dec_item(args, w, nt, grp, split);
            const int n0 = nt * 128;
            const int t0 = 2 * grp, nt_in = min(2, args.n_tiles - t0);
            int kb0, kb1;
            kb_range(split, kb0, kb1);
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(empty_bar(stage), phase ^ 1);
                if (lane == 0) {
                    mbar_expect_tx(full_bar(stage), kDA + 16384u * nt_in);
                    tma_load_2d(a_addr(stage), &args.tmW, full_bar(stage), kb * kBK, n0);
                    for (int t = 0; t < nt_in; ++t)
                        tma_load_2d(b_addr(stage) + 16384u * t, &args.tmX, full_bar(stage), kb * kBK,
                                    args.tiles[t0 + t].row0);
                }
                __syncwarp();
                if (++stage == ST) { stage = 0; phase ^= 1; }
            }
            if (split == 0) {
                for (int t = 0; t < nt_in; ++t) {
                    const DevTile tl = args.tiles[t0 + t];
                    for (int bi = 0; bi < tl.nblk; ++bi) {
                        const DevBlock blk = args.blocks[tl.blk0 + bi];
                        const SlotDev *sd = args.slots + blk.slot;
                        mbar_wait(empty_bar(stage), phase ^ 1);
                        if (lane == 0) {
                            mbar_expect_tx(full_bar(stage), 256u * RB);
                            tma_load_2d(a_addr(stage), &sd->tmBk, full_bar(stage), 0, n0);
                            tma_load_2d(a_addr(stage) + 64u * RB, &sd->tmBk, full_bar(stage), 0, n0 + 64);
                            tma_load_2d(b_addr(stage), &args.tmV, full_bar(stage), 0, (tl.blk0 + bi) * 128);
                        }
                        __syncwarp();
                        if (++stage == ST) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        int stage = 0;
        uint32_t phase = 0;
        uint32_t it = 0;
        constexpr uint32_t idesc128 = idesc_bf16(128, 128, 0, 0);
        constexpr uint32_t idesc256 = idesc_bf16(128, 256, 0, 0);
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            int nt, grp, split;
            dec_item(args, w, nt, grp, split);
            const int t0 = 2 * grp, nt_in = min(2, args.n_tiles - t0);
            int kb0, kb1;
            kb_range(split, kb0, kb1);
            const uint32_t b = it & 1, u = it >> 1;
            const uint32_t acc = tmem_base + 256u * b;
            mbar_wait(accf0 + 16 + 8 * b, (u & 1) ^ 1);
            tc_fence_after();
            uint32_t acc_on = 0;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(full_bar(stage), phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t ab = a_addr(stage), bb = b_addr(stage);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        mma_bf16(acc, smem_desc(ab + 32u * k, 16, 1024, kSw128),
                                 smem_desc(bb + 32u * k, 16, 1024, kSw128), nt_in == 2 ? idesc256 : idesc128,
                                 acc_on);
                        acc_on = 1;
                    }
                    mma_commit(empty_bar(stage));
                }
                __syncwarp();
                if (++stage == ST) { stage = 0; phase ^= 1; }
            }
            if (split == 0) {
                for (int t = 0; t < nt_in; ++t) {
                    const DevTile tl = args.tiles[t0 + t];
                    for (int bi = 0; bi < tl.nblk; ++bi) {
                        mbar_wait(full_bar(stage), phase);
                        tc_fence_after();
                        if (lane == 0) {
                            const uint32_t ab = a_addr(stage), bb = b_addr(stage);
#pragma unroll
                            for (int kk = 0; kk < RP / 16; ++kk)
                                mma_bf16(acc + 128u * t, smem_desc(ab + 32u * kk, 16, 8u * RB, kSwR),
                                         smem_desc(bb + 32u * kk, 16, 8u * RB, kSwR), idesc128, 1);
                            mma_commit(empty_bar(stage));
                        }
                        __syncwarp();
                        if (++stage == ST) { stage = 0; phase ^= 1; }
                    }
                }
            }
            if (lane == 0) mma_commit(accf0 + 8 * b);
            __syncwarp();
            ++it;
        }
    } else if (warp >= 4) {
        const int q = warp - 4;
        const int n = q * 32 + lane;               // W row inside the n-tile (TMEM lane)
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        __nv_bfloat16 *Y = reinterpret_cast<__nv_bfloat16 *>(args.Y);
        uint32_t it = 0;
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            int nt, grp, split;
            dec_item(args, w, nt, grp, split);
            const int n0 = nt * 128;
            const int t0 = 2 * grp, nt_in = min(2, args.n_tiles - t0);
            const int pair = nt * args.n_groups + grp;
            const uint32_t b = it & 1, u = it >> 1;
            mbar_wait(accf0 + 8 * b, u & 1);
            tc_fence_after();
            float *mypart = args.part + ((size_t)pair * args.ksplit + split) * 256 * 128;
            const int ncol = 128 * nt_in;
            for (int c = 0; c < ncol; c += 32) {
                uint32_t rr[32];
                tmem_ld32(tmem_base + 256u * b + lane_base + c, rr);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; ++j) mypart[(size_t)(c + j) * 128 + n] = __uint_as_float(rr[j]);
            }
            tc_fence_before();
            mbar_arrive(accf0 + 16 + 8 * b);   // TMEM buffer free for the next item
            // Every split of an item has its own co-resident CTA (grid == items <= #SMs, 1 CTA/SM),
            // so the splits can wait for each other: once all partials are written, split s sums
            // rows [s*M/ks, (s+1)*M/ks) over the splits in split order (deterministic).
            __threadfence();
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (q == 0 && lane == 0) {
                atomicAdd(args.counters + pair, 1);
                unsigned v;
                do {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(args.counters + pair) : "memory");
                    if ((int)v < args.ksplit) __nanosleep(32);
                } while ((int)v < args.ksplit);
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            __threadfence();
            {
                const float *pp = args.part + (size_t)pair * args.ksplit * 256 * 128;
                const bool col_ok = n0 + n < args.N;
                const int mtot = ncol;
                const int m_lo = split * mtot / args.ksplit, m_hi = (split + 1) * mtot / args.ksplit;
                for (int m = m_lo; m < m_hi; ++m) {
                    const int t = m >> 7, mm = m & 127;
                    const DevTile tl = args.tiles[t0 + t];
                    if (mm >= tl.rows) continue;
                    float acc = 0.f;
                    for (int s2 = 0; s2 < args.ksplit; ++s2) acc += __ldcg(pp + ((size_t)s2 * 256 + m) * 128 + n);
                    if (col_ok) Y[(size_t)(tl.row0 + mm) * args.N + n0 + n] = __float2bfloat16_rn(acc);
                }
            }
            ++it;
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

template <int RP>
int launch_dec_impl(const DecArgs &a, int num_sms, cudaStream_t st) {
    auto kern = smlm_dec_kernel<RP>;
    const size_t smem = 1024 + (size_t)a.stages * kDStage + 256;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        attr_done = true;
    }
    const int total = a.n_nt * a.n_groups * a.ksplit;
    if (total > num_sms) return (int)cudaErrorInvalidValue;  // the split handshake needs co-residency
    kern<<<total, kDThreads, smem, st>>>(a);
    return (int)cudaGetLastError();
}

}  // namespace

int dec_stages() { return 4; }

int dec_chunks(int in_f) { return in_f / kChunk > 0 && in_f % kChunk == 0 ? in_f / kChunk : 0; }

int launch_shrink_split(const __nv_bfloat16 *X, const SlotDev *slots, const DevBlock *blocks,
                        const DevShortRow *srows, int n_blocks, int in_f, int r, int r_pad, float *part,
                        __nv_bfloat16 *Vbd, __nv_bfloat16 *Vsave, cudaStream_t st) {
    if (n_blocks == 0) return 0;
    const int nch = dec_chunks(in_f);
    dim3 g1(n_blocks, nch);
    switch (r_pad) {
        case 16:
            shrink_partial_kernel<16><<<g1, 256, 0, st>>>(X, slots, blocks, srows, in_f, r, part);
            shrink_combine_kernel<16><<<n_blocks, 128, 0, st>>>(blocks, srows, nch, r, part, Vbd, Vsave);
            break;
        case 32:
            shrink_partial_kernel<32><<<g1, 256, 0, st>>>(X, slots, blocks, srows, in_f, r, part);
            shrink_combine_kernel<32><<<n_blocks, 128, 0, st>>>(blocks, srows, nch, r, part, Vbd, Vsave);
            break;
        case 64:
            shrink_partial_kernel<64><<<g1, 256, 0, st>>>(X, slots, blocks, srows, in_f, r, part);
            shrink_combine_kernel<64><<<n_blocks, 128, 0, st>>>(blocks, srows, nch, r, part, Vbd, Vsave);
            break;
        default: return (int)cudaErrorInvalidValue;
    }
    return (int)cudaGetLastError();
}

int launch_dec(const DecArgs &a, int num_sms, cudaStream_t st) {
    switch (a.r_pad) {
        case 16: return launch_dec_impl<16>(a, num_sms, st);
        case 32: return launch_dec_impl<32>(a, num_sms, st);
        case 64: return launch_dec_impl<64>(a, num_sms, st);
    }
    return (int)cudaErrorInvalidValue;
}

}  // namespace smlm
