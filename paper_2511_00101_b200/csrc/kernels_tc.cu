// kernels_tc.cu -- the fused SMLM GEMM on 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// One persistent, warp-specialised kernel serves both directions:
//   forward  (a2/a3): Y[tile, n-tile] = X_tile W^T  +  (s V) B_a^T,   V = X_tile A_a^T on-chip
//   backward (a4)   : dX[tile, n-tile] = dY_tile W  +  (s U) A_a,     U = dY_tile B_a  on-chip
// PAPER.md P:379-384 (§3.3): all input-LoRA pairs of one linear layer in a single kernel call,
// per-request scale applied "during the forward pass"; P:415 / P:696: the LoRA backward, which
// the paper left to per-linear autograd calls, is fused here.
//
// Work item = (128-row tile, 256-column n-tile).  Long tiles (one segment, one adapter) compute
// the rank-r intermediate with an extra N=r_pad MMA that reuses the X (dY) tile already staged
// in shared memory; the epilogue warps scale it by s, round to bf16 into shared memory, and the
// MMA warp folds it in as one more K-block of depth r (the rank-r intermediate never leaves the
// SM).  Short tiles (rows of many decode/short segments) fold each distinct adapter
// in as a K=r_pad block whose A operand is the block-diagonal s*V prepared by the shrink kernel.
//
// Warp roles (256 threads): warp 0 TMA producer, warp 1 MMA issuer, warp 2 TMEM allocator,
// warps 4..7 epilogue (TMEM lanes 32*(warp%4) ...).  TMEM: accumulator columns [0,256),
// rank-r accumulator columns [256, 256+r_pad).
#include <cuda_runtime.h>

#include "device_types.h"
#include "pdl.cuh"
#include "sm100.cuh"
#include "dropout.cuh"

namespace smlm {
using namespace sm100;

namespace {

constexpr int kThreads = 256;
constexpr uint32_t kABytes = 128 * 128;   // X/dY tile: 128 rows x 64 bf16
constexpr uint32_t kBBytes = 256 * 128;   // W tile: 256 x 64 bf16

__device__ __forceinline__ void decode_work(int w, int n_tiles, int n_nt, int group_m, int &ti, int &nt) {
    const int gsz = group_m * n_nt;
    const int g = w / gsz;
    const int first = g * group_m;
    const int gm = min(group_m, n_tiles - first);
    const int local = w - g * gsz;
    ti = first + local % gm;
    nt = local / gm;
}

template <bool BWD, int RP>
__global__ void __launch_bounds__(kThreads, 1) smlm_gemm_kernel(const __grid_constant__ GemmArgs args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);

    constexpr uint32_t RB = RP * 2;             // bytes per row of an r_pad-wide bf16 tile
    // Forward: the shrink is fused into the main MMA.  The B operand of one N=256 MMA is the W
    // n-tile (BNW = 256 - RP rows) stacked on A_a (RP rows), so the accumulator columns
    // [BNW, 256) receive V = X_tile A_a^T while [0, BNW) receive X_tile W^T, and the X tile is
    // read from shared memory once per K-step.  Backward: U = dY B_a comes precomputed (tile-compact
    // s*U from smlm_u_kernel, also needed by the dA contraction) and is TMA-loaded as the A operand
    // of the expand K-block; the main loop is a plain dY W with W as the MN-major operand.
    constexpr int BNW = BWD ? kBN : kBN - RP;   // output columns per n-tile
    constexpr uint32_t kStage = kABytes + kBBytes;
    constexpr uint32_t kSwR = RB >= 128 ? kSw128 : (RB == 64 ? kSw64 : kSw32);
    const int stages = args.stages;
    const uint32_t sv_addr = base + stages * kStage;
    const uint32_t bar = sv_addr + 128 * RB;
    auto full_bar = [&](int s) { return bar + 8u * s; };
    auto empty_bar = [&](int s) { return bar + 8u * (stages + s); };
    const uint32_t acc_full0 = bar + 16u * stages;   // acc_full[2]
    const uint32_t acc_empty0 = acc_full0 + 16;      // acc_empty[2]
    const uint32_t v_full = acc_full0 + 48;
    const uint32_t sv_ready = acc_full0 + 56;
    const uint32_t tmem_slot = acc_full0 + 64;
    auto a_addr = [&](int s) { return base + s * kStage; };
    auto b_addr = [&](int s) { return base + s * kStage + kABytes; };

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(acc_full0 + 8 * b, 1);
            mbar_init(acc_empty0 + 8 * b, 128);
        }
        mbar_init(v_full, 1);
        mbar_init(sv_ready, 128);
        fence_mbar_init();
        tma_prefetch_desc(&args.tmA);
        tma_prefetch_desc(&args.tmB);
        if (!BWD) tma_prefetch_desc(&args.tmV);
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t *>(base_ptr + (tmem_slot - base));
    // two accumulator buffers ACC_b = TMEM columns [256 b, 256 b + 256)
    auto acc_col = [&](uint32_t b) { return tmem_base + 256u * b; };
    auto v_col = [&](uint32_t b) { return tmem_base + 256u * b + BNW; };   // forward V columns
    pdl_wait();
    pdl_trigger();

    const int total = args.n_tiles * args.n_ntiles;
    const int nkb = args.K / kBK;

    if (warp == 0) {
        // ============================ TMA producer ============================
        int stage = 0;
        uint32_t phase = 0;
        auto advance = [&]() {
            if (++stage == stages) { stage = 0; phase ^= 1; }
        };
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            int ti, nt;
            decode_work(w, args.n_tiles, args.n_ntiles, args.group_m, ti, nt);
            const DevTile t = args.tiles[ti];
            const int n0 = nt * BNW;
            const bool is_short = (t.flags & kTileShort) != 0;
            const bool lora = (t.flags & kTileLora) != 0;
            const SlotDev *sd = lora ? args.slots + t.slot : nullptr;
            if (!is_short || args.has_w) {
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(empty_bar(stage), phase ^ 1);
                    if (lane == 0) {
                        uint32_t bytes = kABytes;
                        if (args.has_w) {
                            if (BWD) {
                                int nb = 0;
                                for (int i = 0; i < 4; ++i) nb += (n0 + 64 * i < args.N);
                                bytes += 8192u * nb;
                            } else {
                                bytes += BNW * 128u;
                            }
                        }
                        if (lora && !BWD) bytes += RP * 128u;
                        mbar_expect_tx(full_bar(stage), bytes);
                        tma_load_2d(a_addr(stage), &args.tmA, full_bar(stage), kb * kBK, t.row0);
                        if (args.has_w) {
                            if (BWD) {
                                for (int i = 0; i < 4; ++i)
                                    if (n0 + 64 * i < args.N)
                                        tma_load_2d(b_addr(stage) + 8192u * i, &args.tmB, full_bar(stage),
                                                    n0 + 64 * i, kb * kBK);
                            } else {
                                tma_load_2d(b_addr(stage), &args.tmB, full_bar(stage), kb * kBK, n0);
                            }
                        }
                        if (lora && !BWD)  // A_a [r_pad rows] x 64 k, stacked under the W rows
                            tma_load_2d(b_addr(stage) + BNW * 128u, &sd->tmA, full_bar(stage), kb * kBK, 0);
                    }
                    __syncwarp();
                    advance();
                }
            }
            if (lora) {
                mbar_wait(empty_bar(stage), phase ^ 1);
                if (lane == 0) {
                    if (BWD) {  // s*U rows of the tile (K-major) + A_a [r_pad rows, n0 + 64 i ...] (MN-major)
                        mbar_expect_tx(full_bar(stage), 256u * RB + 128u * RB);
                        tma_load_2d(a_addr(stage), &args.tmV, full_bar(stage), 0, ti * 128);
                        for (int i = 0; i < 4; ++i)
                            tma_load_2d(b_addr(stage) + (uint32_t)RP * 128u * i, &sd->tmA, full_bar(stage),
                                        n0 + 64 * i, 0);
                    } else {    // B_a [n0 .. n0 + BNW, r_pad] K-major expand operand
                        mbar_expect_tx(full_bar(stage), (uint32_t)BNW * RB);
                        tma_load_2d(b_addr(stage), &sd->tmBn, full_bar(stage), 0, n0);
                    }
                }
                __syncwarp();
                advance();
            } else if (is_short) {
                for (int bi = 0; bi < t.nblk; ++bi) {
                    const DevBlock blk = args.blocks[t.blk0 + bi];
                    const SlotDev *bs = args.slots + blk.slot;
                    mbar_wait(empty_bar(stage), phase ^ 1);
                    if (lane == 0) {
                        mbar_expect_tx(full_bar(stage), 128u * RB + (uint32_t)BNW * RB);
                        tma_load_2d(a_addr(stage), &args.tmV, full_bar(stage), 0, (t.blk0 + bi) * 128);
                        tma_load_2d(b_addr(stage), &bs->tmBn, full_bar(stage), 0, n0);
                    }
                    __syncwarp();
                    advance();
                }
            }
        }
    } else if (warp == 1) {
        // ============================ MMA issuer ============================
        int stage = 0;
        uint32_t phase = 0;
        auto advance = [&]() {
            if (++stage == stages) { stage = 0; phase ^= 1; }
        };
        constexpr uint32_t idesc_full = idesc_bf16(128, kBN, 0, BWD ? 1 : 0);   // W (+ stacked A_a)
        constexpr uint32_t idesc_out = idesc_bf16(128, BNW, 0, BWD ? 1 : 0);    // output columns only
        uint32_t it = 0, lora_it = 0;
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            int ti, nt;
            decode_work(w, args.n_tiles, args.n_ntiles, args.group_m, ti, nt);
            const DevTile t = args.tiles[ti];
            const bool is_short = (t.flags & kTileShort) != 0;
            const bool lora = (t.flags & kTileLora) != 0;
            const uint32_t b = it & 1, u = it >> 1;
            const uint32_t acc_tmem = acc_col(b), v_tmem = v_col(b);
            mbar_wait(acc_empty0 + 8 * b, (u & 1) ^ 1);
            tc_fence_after();
            uint32_t acc_on = 0;  // 1 once the accumulator holds data
            if (!is_short || args.has_w) {
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(full_bar(stage), phase);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t ab = a_addr(stage), bb = b_addr(stage);
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k) {
                            const uint64_t ad = smem_desc(ab + 32u * k, 16, 1024, kSw128);
                            if (BWD) {
                                const uint64_t bd = smem_desc(bb + 2048u * k, 8192, 1024, kSw128);
                                mma_bf16(acc_tmem, ad, bd, idesc_full, (kb | k) != 0);
                            } else if (args.has_w) {
                                const uint64_t bd = smem_desc(bb + 32u * k, 16, 1024, kSw128);
                                mma_bf16(acc_tmem, ad, bd, lora ? idesc_full : idesc_out, (kb | k) != 0);
                            } else {
                                // delta-only forward: only the stacked A_a rows (V columns)
                                const uint64_t vd = smem_desc(bb + BNW * 128u + 32u * k, 16, 1024, kSw128);
                                mma_bf16(v_tmem, ad, vd, idesc_bf16(128, RP, 0, 0), (kb | k) != 0);
                            }
                        }
                        mma_commit(empty_bar(stage));
                    }
                    __syncwarp();
                    advance();
                }
                acc_on = args.has_w ? 1u : 0u;
            }
            if (lora) {
                if (!BWD) {
                    if (lane == 0) mma_commit(v_full);
                    __syncwarp();
                }
                mbar_wait(full_bar(stage), phase);
                if (!BWD) mbar_wait(sv_ready, lora_it & 1);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t bb = b_addr(stage);
                    const uint32_t aop = BWD ? a_addr(stage) : sv_addr;   // s*U via TMA / s*V from the epilogue
#pragma unroll
                    for (int kk = 0; kk < RP / 16; ++kk) {
                        const uint64_t ad = smem_desc(aop + 32u * kk, 16, 8u * RB, kSwR);
                        const uint64_t bd = BWD ? smem_desc(bb + 2048u * kk, (uint32_t)RP * 128u, 1024, kSw128)
                                                : smem_desc(bb + 32u * kk, 16, 8u * RB, kSwR);
                        mma_bf16(acc_tmem, ad, bd, idesc_out, acc_on | (kk != 0));
                    }
                    mma_commit(empty_bar(stage));
                }
                __syncwarp();
                advance();
                ++lora_it;
            } else if (is_short) {
                for (int bi = 0; bi < t.nblk; ++bi) {
                    mbar_wait(full_bar(stage), phase);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t ab = a_addr(stage), bb = b_addr(stage);
#pragma unroll
                        for (int kk = 0; kk < RP / 16; ++kk) {
                            const uint64_t ad = smem_desc(ab + 32u * kk, 16, 8u * RB, kSwR);
                            const uint64_t bd = smem_desc(bb + 32u * kk, 16, 8u * RB, kSwR);
                            mma_bf16(acc_tmem, ad, bd, idesc_out, acc_on | (uint32_t)(bi | kk));
                        }
                        mma_commit(empty_bar(stage));
                    }
                    __syncwarp();
                    advance();
                }
            }
            if (lane == 0) mma_commit(acc_full0 + 8 * b);
            __syncwarp();
            ++it;
        }
    } else if (warp >= 4) {
        // ============================ epilogue ============================
        const int q = warp - 4;
        const int m = q * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        uint32_t it = 0, lora_it = 0;
        __nv_bfloat16 *Y = reinterpret_cast<__nv_bfloat16 *>(args.Y);
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            int ti, nt;
            decode_work(w, args.n_tiles, args.n_ntiles, args.group_m, ti, nt);
            const DevTile t = args.tiles[ti];
            const int n0 = nt * BNW;
            const bool lora = (t.flags & kTileLora) != 0;
            const bool row_ok = m < t.rows;
            const int row = t.row0 + m;
            const uint32_t b = it & 1, u = it >> 1;
            if (lora && !BWD) {
                mbar_wait(v_full, lora_it & 1);
                tc_fence_after();
                uint32_t v[RP];
#pragma unroll
                for (int c = 0; c < RP; c += 16) {
                    uint32_t tmp[16];
                    tmem_ld16(v_col(b) + lane_base + c, tmp);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[c + j] = tmp[j];
                }
                if (!BWD && nt == 0 && row_ok && (t.flags & kTileFT) && args.Vsave) {
                    __nv_bfloat16 *vs = reinterpret_cast<__nv_bfloat16 *>(args.Vsave) + (size_t)row * args.r;
#pragma unroll
                    for (int j = 0; j < RP; ++j)
                        if (j < args.r) vs[j] = __float2bfloat16_rn(__uint_as_float(v[j]));
                }
                const float s = t.scale;
                uint8_t *sv = base_ptr + (sv_addr - base);
#pragma unroll
                for (int c = 0; c < RP / 8; ++c) {
                    uint4 pk;
                    pk.x = pack_bf16x2(s * __uint_as_float(v[8 * c + 0]), s * __uint_as_float(v[8 * c + 1]));
                    pk.y = pack_bf16x2(s * __uint_as_float(v[8 * c + 2]), s * __uint_as_float(v[8 * c + 3]));
                    pk.z = pack_bf16x2(s * __uint_as_float(v[8 * c + 4]), s * __uint_as_float(v[8 * c + 5]));
                    pk.w = pack_bf16x2(s * __uint_as_float(v[8 * c + 6]), s * __uint_as_float(v[8 * c + 7]));
                    *reinterpret_cast<uint4 *>(sv + swz((uint32_t)m * RB + 16u * c, RB)) = pk;
                }
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(sv_ready);
                ++lora_it;
            }
            mbar_wait(acc_full0 + 8 * b, u & 1);
            tc_fence_after();
            // drain the accumulator in 16-column chunks
#pragma unroll 1
            for (int c = BNW / 16 - 1; c >= 0; --c) {
                uint32_t r[16];
                tmem_ld16(acc_col(b) + lane_base + 16u * c, r);
                tmem_wait_ld();
                const int col = n0 + 16 * c;
                if (row_ok && col < args.N) {
                    uint4 *dst = reinterpret_cast<uint4 *>(Y + (size_t)row * args.N + col);
                    if (!BWD && !args.has_w) {
#pragma unroll
                        for (int q4 = 0; q4 < 2; ++q4) {
                            uint4 old = dst[q4];
                            const __nv_bfloat162 *o2 = reinterpret_cast<const __nv_bfloat162 *>(&old);
                            uint4 pk;
                            uint32_t *pw = reinterpret_cast<uint32_t *>(&pk);
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                float2 f = __bfloat1622float2(o2[e]);
                                pw[e] = pack_bf16x2(f.x + __uint_as_float(r[8 * q4 + 2 * e]),
                                                    f.y + __uint_as_float(r[8 * q4 + 2 * e + 1]));
                            }
                            dst[q4] = pk;
                        }
                    } else {
#pragma unroll
                        for (int q4 = 0; q4 < 2; ++q4) {
                            uint4 pk;
                            pk.x = pack_bf16x2(__uint_as_float(r[8 * q4 + 0]), __uint_as_float(r[8 * q4 + 1]));
                            pk.y = pack_bf16x2(__uint_as_float(r[8 * q4 + 2]), __uint_as_float(r[8 * q4 + 3]));
                            pk.z = pack_bf16x2(__uint_as_float(r[8 * q4 + 4]), __uint_as_float(r[8 * q4 + 5]));
                            pk.w = pack_bf16x2(__uint_as_float(r[8 * q4 + 6]), __uint_as_float(r[8 * q4 + 7]));
                            dst[q4] = pk;
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(acc_empty0 + 8 * b);
            ++it;
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

template <bool BWD, int RP>
int launch_impl(const GemmArgs &a, int num_sms, size_t smem, cudaStream_t st) {
    auto kern = smlm_gemm_kernel<BWD, RP>;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
        if (e != cudaSuccess) return (int)e;
        attr_done = true;
    }
    const int total = a.n_tiles * a.n_ntiles;
    const int grid = total < num_sms ? total : num_sms;
    return (int)launch_pdl(kern, dim3(grid), dim3(kThreads), smem, st, a);
}


// ==========================================================================================
// Token-contraction GEMM (a5): for every adapter with fine-tune rows and bound gradients,
//   dA_a^T [in x r]  = X^T (s U)   and   dB_a [out x r] = dY^T (s V)
// contracted over the adapter's fine-tune tokens, visiting its tiles in the canonical order
// (bitwise deterministic, no atomics; PAPER.md P:420 shared backward, P:422 masking).
// Work item = (adapter, 128-row M tile of in or out).  A operand = 64 tokens x 128 columns of
// X or dY (MN-major, two 64-column SW128 boxes); B operand = 64 tokens x r_pad of the
// tile-compact s*U / s*V (MN-major).  Token rows past a segment's end are zeroed in shared
// memory before the MMA (isolation from other requests' rows).  Two TMEM accumulators of r_pad
// columns let the epilogue of one item overlap the main loop of the next.
// ==========================================================================================
// pipeline depth: as many stages as shared memory holds (HBM-bound stream of 64-token K-blocks;
// bytes in flight per SM are what keep the memory system busy), at most 12
template <int RP, int NH = 1>
constexpr int tok_stages() {
    return (int)((232448u - 1536u) / (16384u * NH + ((64u * RP * 2u + 1023u) & ~1023u))) > 12
               ? 12
               : (int)((232448u - 1536u) / (16384u * NH + ((64u * RP * 2u + 1023u) & ~1023u)));
}

__device__ __forceinline__ bool tok_item(const TokArgs &a, int w, int &g, int &mt, bool &is_b) {
    const int na = a.n_groups * a.mt_a;
    if (w < na) {
        g = w / a.mt_a;
        mt = w % a.mt_a;
        is_b = false;
        return a.groups[g].dA != nullptr;
    }
    w -= na;
    g = w / a.mt_b;
    mt = w % a.mt_b;
    is_b = true;
    return a.groups[g].dB != nullptr;
}

// NH = 2: an item covers 256 columns (two 128-column halves, two accumulators sharing the s*U /
// s*V operand): each token row is read as 512 contiguous bytes per K-block instead of 256
template <int RP, int NH>
__global__ void __launch_bounds__(kThreads, 1) smlm_tok_kernel(const __grid_constant__ TokArgs args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    constexpr uint32_t RB = RP * 2;
    constexpr uint32_t kA = 16384 * NH;         // 64 tokens x 128*NH columns bf16 (2*NH boxes of 8 KB)
    constexpr uint32_t kB = 64 * RB;            // 64 tokens x r_pad
    constexpr uint32_t kStage = kA + ((kB + 1023u) & ~1023u);
    constexpr uint32_t kSwR = RB >= 128 ? kSw128 : (RB == 64 ? kSw64 : kSw32);
    constexpr int ST = tok_stages<RP, NH>();
    constexpr uint32_t kTm = 2 * NH * RP <= 128 ? 128 : 256;
    const uint32_t bar = base + ST * kStage;
    auto full_bar = [&](int s) { return bar + 8u * s; };
    auto empty_bar = [&](int s) { return bar + 8u * (ST + s); };
    const uint32_t accf0 = bar + 16u * ST;      // acc_full[2], acc_empty[2]
    const uint32_t tmem_slot = accf0 + 32;
    auto mask_bar = [&](int s) { return accf0 + 48u + 8u * s; };   // dropout: the X stage is masked
    auto a_addr = [&](int s) { return base + s * kStage; };
    auto b_addr = [&](int s) { return base + s * kStage + kA; };

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
        for (int s = 0; s < ST; ++s) mbar_init(mask_bar(s), 64);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, kTm);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t *>(base_ptr + (tmem_slot - base));
    pdl_wait();
    pdl_trigger();
    const int total = args.n_groups * (args.mt_a + args.mt_b);

    if (warp == 2 || warp == 3) {
        // LoRA dropout (dA items): zero the dropped X elements of each staged token block -- the
        // forward's mask (same counter-based hash of (seed, token, column)); dA is scaled by
        // 1/(1-p) in the epilogue
        if (args.drop.on) {
            int stage = 0;
            uint32_t phase = 0;
            const int tid = threadIdx.x - 64;
            for (int w = blockIdx.x; w < total; w += gridDim.x) {
                int g, mt;
                bool is_b;
                if (!tok_item(args, w, g, mt, is_b)) continue;
                const GradGroup grp = args.groups[g];
                const int m0 = mt * 128 * NH;
                int nbox = 0;
#pragma unroll
                for (int bx = 0; bx < 2 * NH; ++bx) nbox += (m0 + 64 * bx < args.in_f);
                for (int ti = 0; ti < grp.n_tiles; ++ti) {
                    const DevTile t = args.tiles[grp.tile_begin + ti];
                    for (int kb = 0; kb * 64 < t.rows; ++kb) {
                        if (!is_b) {
                            mbar_wait(full_bar(stage), phase);
                            for (int bx = 0; bx < nbox; ++bx)
                                drop_mask_box_sw128(args.drop, base_ptr + (a_addr(stage) - base) + 8192 * bx, 64,
                                                    (uint32_t)(t.row0 + 64 * kb), (uint32_t)(m0 + 64 * bx), tid, 64);
                            fence_proxy_async_smem();
                            mbar_arrive(mask_bar(stage));
                        }
                        if (++stage == ST) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            int g, mt;
            bool is_b;
            if (!tok_item(args, w, g, mt, is_b)) continue;
            const GradGroup grp = args.groups[g];
            const int M = is_b ? args.out_f : args.in_f;
            const int m0 = mt * 128 * NH;
            int nbox = 0;   // 64-column boxes of this item inside M (in/out are multiples of 64)
#pragma unroll
            for (int bx = 0; bx < 2 * NH; ++bx) nbox += (m0 + 64 * bx < M);
            const CUtensorMap *ma = is_b ? &args.tmDY : &args.tmX;
            const CUtensorMap *mb = is_b ? &args.tmSV : &args.tmSU;
            for (int ti = 0; ti < grp.n_tiles; ++ti) {
                const int tix = grp.tile_begin + ti;
                const DevTile t = args.tiles[tix];
                for (int kb = 0; kb * 64 < t.rows; ++kb) {
                    mbar_wait(empty_bar(stage), phase ^ 1);
                    if (lane == 0) {
                        mbar_expect_tx(full_bar(stage), (uint32_t)nbox * 8192u + kB);
                        for (int bx = 0; bx < nbox; ++bx)
                            tma_load_2d(a_addr(stage) + 8192u * bx, ma, full_bar(stage), m0 + 64 * bx, t.row0 + 64 * kb);
                        tma_load_2d(b_addr(stage), mb, full_bar(stage), 0, tix * 128 + 64 * kb);
                    }
                    __syncwarp();
                    if (++stage == ST) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        int stage = 0;
        uint32_t phase = 0, mph = 0;
        uint32_t it = 0;
        constexpr uint32_t idesc = idesc_bf16(128, RP, 1, 1);
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            int g, mt;
            bool is_b;
            if (!tok_item(args, w, g, mt, is_b)) continue;
            const GradGroup grp = args.groups[g];
            const uint32_t buf = it & 1;
            mbar_wait(accf0 + 16 + 8 * buf, ((it >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t acc = tmem_base + buf * NH * RP;
            const int nh = (NH == 2 && mt * 256 + 128 < (is_b ? args.out_f : args.in_f)) ? 2 : 1;
            uint32_t acc_on = 0;
            for (int ti = 0; ti < grp.n_tiles; ++ti) {
                const DevTile t = args.tiles[grp.tile_begin + ti];
                for (int kb = 0; kb * 64 < t.rows; ++kb) {
                    if (args.drop.on && !is_b) {
                        mbar_wait(mask_bar(stage), (mph >> stage) & 1u);
                        mph ^= 1u << stage;
                    } else {
                        mbar_wait(full_bar(stage), phase);
                    }
                    const int valid = min(64, t.rows - 64 * kb);
                    if (valid < 64) {
                        // zero token rows past the segment end in both 64-column boxes
                        uint8_t *ap = base_ptr + (a_addr(stage) - base);
                        for (int e = lane; e < (64 - valid) * 8 * 2 * NH; e += 32) {
                            const int row = valid + e / (16 * NH), box = (e >> 3) % (2 * NH), ch = e & 7;
                            *reinterpret_cast<uint4 *>(ap + box * 8192 + row * 128 + ch * 16) = make_uint4(0, 0, 0, 0);
                        }
                        fence_proxy_async_smem();
                        __syncwarp();
                    }
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t ab = a_addr(stage), bb = b_addr(stage);
                        for (int k = 0; k * 16 < valid; ++k) {
                            const uint64_t bd = smem_desc(bb + 16u * RB * k, 64u * RB, 8u * RB, kSwR);
                            for (int h = 0; h < nh; ++h) {
                                const uint64_t ad = smem_desc(ab + 16384u * h + 2048u * k, 8192, 1024, kSw128);
                                mma_bf16(acc + (uint32_t)h * RP, ad, bd, idesc, acc_on);
                            }
                            acc_on = 1;
                        }
                        mma_commit(empty_bar(stage));
                    }
                    __syncwarp();
                    if (++stage == ST) { stage = 0; phase ^= 1; }
                }
            }
            if (lane == 0) mma_commit(accf0 + 8 * buf);
            __syncwarp();
            ++it;
        }
    } else if (warp >= 4) {
        const int q = warp - 4;
        const int m = q * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        uint32_t it = 0;
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            int g, mt;
            bool is_b;
            if (!tok_item(args, w, g, mt, is_b)) continue;
            const GradGroup grp = args.groups[g];
            const uint32_t buf = it & 1;
            mbar_wait(accf0 + 8 * buf, (it >> 1) & 1);
            tc_fence_after();
            uint32_t vv[NH][RP];
#pragma unroll
            for (int h = 0; h < NH; ++h)
#pragma unroll
                for (int c = 0; c < RP; c += 16) {
                    uint32_t tmp[16];
                    tmem_ld16(tmem_base + buf * NH * RP + h * RP + lane_base + c, tmp);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; ++j) vv[h][c + j] = tmp[j];
                }
            tc_fence_before();
            mbar_arrive(accf0 + 16 + 8 * buf);
            const int M = is_b ? args.out_f : args.in_f;
#pragma unroll
            for (int h = 0; h < NH; ++h) {
            const uint32_t *v = vv[h];
            const int col = mt * 128 * NH + 128 * h + m;
            if (col < M) {
                if (is_b) {
                    float *p = grp.dB + (size_t)col * grp.r;   // the adapter's own rank
#pragma unroll
                    for (int j = 0; j < RP; ++j)
                        if (j < grp.r) {
                            const float dv = args.accumulate ? p[j] + __uint_as_float(v[j]) : __uint_as_float(v[j]);
                            p[j] = dv;
                            for (int q = 0; q < args.n_fanout; ++q)   // peers' copies of this rank's slot
                                *reinterpret_cast<float *>(reinterpret_cast<char *>(p + j) + args.fanout_delta[q]) = dv;
                        }
                } else {
                    const float ds = args.drop.on ? args.drop.scale : 1.f;   // x~ = keep * x / (1 - p)
#pragma unroll
                    for (int j = 0; j < RP; ++j)
                        if (j < grp.r) {
                            float *p = grp.dA + (size_t)j * args.in_f + col;
                            const float dv = ds * __uint_as_float(v[j]);
                            const float nv = args.accumulate ? *p + dv : dv;
                            *p = nv;
                            for (int q = 0; q < args.n_fanout; ++q)   // peers' copies of this rank's slot
                                *reinterpret_cast<float *>(reinterpret_cast<char *>(p) + args.fanout_delta[q]) = nv;
                        }
                }
            }
            }
            ++it;
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTm);
    }
}

template <int RP, int NH>
int launch_tok_impl(const TokArgs &a, int num_sms, cudaStream_t st) {
    auto kern = smlm_tok_kernel<RP, NH>;
    constexpr size_t kStage = 16384 * NH + ((64 * RP * 2 + 1023) & ~1023);
    const size_t smem = 1024 + tok_stages<RP, NH>() * kStage + 512;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        attr_done = true;
    }
    const int total = a.n_groups * (a.mt_a + a.mt_b);
    const int grid = total < num_sms ? total : num_sms;
    return (int)launch_pdl(kern, dim3(grid), dim3(kThreads), smem, st, a);
}


// ==========================================================================================
// U = dY B_a for the fine-tune tiles (backward), split K over `out`:
//   item = (fine-tune tile with an adapter, K split); D[128 rows x r_pad] on tcgen05 with the dY
//   tile as the K-major A operand and B_a k-rows as the MN-major B operand; fp32 partials
//   [tile][split][128][r_pad]; the last split of a tile to arrive (per-item counter) sums them in
//   split order and writes the tile-compact s*U (bf16, zero rows past the segment) consumed by the
//   dX expand and the dA contraction.
// The same kernel is the forward PRE-SHRINK (vf = 1, DESIGN K1a): V = X A_a^T of every long tile
//   with an adapter, A_a as the K-major B operand, -> tile-compact s*V + V_save; with NPJ > 1 the
//   A_a of several projections that share X are stacked (N = NPJ * r_pad) so X is read once.
// ==========================================================================================
// pipeline depth of the U / pre-shrink pass: as many 16 KB + r_pad-row stages as shared memory
// holds (the pass is a latency-bound stream of small K-blocks: depth is what keeps HBM busy)
template <int RP, int NPJ = 1>
constexpr uint32_t u_stage_bytes() { return kABytes + ((64u * RP * 2u * NPJ + 1023u) & ~1023u); }
template <int RP, int NPJ = 1, int KW = 1>
constexpr int u_stages() {
    return (int)((232448u - 1536u) / (KW * u_stage_bytes<RP, NPJ>())) > 12
               ? 12
               : (int)((232448u - 1536u) / (KW * u_stage_bytes<RP, NPJ>()));
}

// sUt[tile*128 + m][j] = bf16(s * sum_split part) (zero rows past the segment), split order fixed
// NPJ > 1 (forward pre-shrink of several projections sharing X): the partial rows hold NPJ x RP
// columns; projection p's columns go to sUt_p[p] / Vsave_p[p]
template <int RP, int NPJ = 1>
__device__ __forceinline__ void u_reduce_row(const UArgs &args, int item, int m) {
    const int ti = args.items[item];
    const DevTile t = args.tiles[ti];
#pragma unroll 1
    for (int pj = 0; pj < NPJ; ++pj) {
    void *sut = NPJ == 1 ? args.sUt : args.sUt_p[pj];
    void *vsave = NPJ == 1 ? args.Vsave : args.Vsave_p[pj];
    uint4 *dst = reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(sut) + ((size_t)ti * 128 + m) * RP);
    float acc[RP];
#pragma unroll
    for (int j = 0; j < RP; ++j) acc[j] = 0.f;
    if (m < t.rows) {
        for (int s = 0; s < args.ksplit; ++s) {
            const float4 *src = reinterpret_cast<const float4 *>(args.part + (((size_t)item * args.ksplit + s) * 128 + m) * (NPJ * RP) + pj * RP);
#pragma unroll
            for (int j4 = 0; j4 < RP / 4; ++j4) {
                const float4 v = __ldcg(src + j4);
                acc[4 * j4] += v.x; acc[4 * j4 + 1] += v.y; acc[4 * j4 + 2] += v.z; acc[4 * j4 + 3] += v.w;
            }
        }
        if (args.vf && args.drop.on && (t.flags & kTileFT)) {   // V~ = A_a (keep * x) / (1 - p)
#pragma unroll
            for (int j = 0; j < RP; ++j) acc[j] *= args.drop.scale;
        }
    }
    if (args.vf && vsave && (t.flags & kTileFT) && m < t.rows) {
        __nv_bfloat16 *vs = reinterpret_cast<__nv_bfloat16 *>(vsave) + (size_t)(t.row0 + m) * args.r;
#pragma unroll
        for (int j = 0; j < RP; ++j)
            if (j < args.r) vs[j] = __float2bfloat16_rn(acc[j]);
    }
#pragma unroll
    for (int c = 0; c < RP / 8; ++c) {
        uint4 pk;
        pk.x = pack_bf16x2(t.scale * acc[8 * c + 0], t.scale * acc[8 * c + 1]);
        pk.y = pack_bf16x2(t.scale * acc[8 * c + 2], t.scale * acc[8 * c + 3]);
        pk.z = pack_bf16x2(t.scale * acc[8 * c + 4], t.scale * acc[8 * c + 5]);
        pk.w = pack_bf16x2(t.scale * acc[8 * c + 6], t.scale * acc[8 * c + 7]);
        dst[c] = pk;
    }
    }
    if (!args.vf && args.sVt) {
        const __nv_bfloat16 *vin = reinterpret_cast<const __nv_bfloat16 *>(args.Vsave_in);
        __nv_bfloat16 *dv = reinterpret_cast<__nv_bfloat16 *>(args.sVt) + ((size_t)ti * 128 + m) * RP;
#pragma unroll
        for (int j = 0; j < RP; ++j) {
            float v = 0.f;
            if (m < t.rows && j < args.r) v = t.scale * __bfloat162float(vin[(size_t)(t.row0 + m) * args.r + j]);
            dv[j] = __float2bfloat16_rn(v);
        }
    }
}

// stand-alone reduce (when the kernel has no arrival counters)
template <int RP, int NPJ>
__global__ void __launch_bounds__(128) u_reduce_kernel(const __grid_constant__ UArgs args) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    u_reduce_row<RP, NPJ>(args, blockIdx.x, threadIdx.x);
}

// KW = 2: a ring stage holds two consecutive 64-wide K-blocks (sub-stages), so each token row is
// requested as 256 contiguous bytes at a time
template <int RP, int NPJ, int KW>
__global__ void __launch_bounds__(kThreads, 1) smlm_u_kernel(const __grid_constant__ UArgs args) {
    // VF (args.vf): the forward pre-shrink V = X A_a^T of long tiles -- same split-K contraction,
    // the adapter operand A_a [r, in] K-major (tmA box {64, r_pad}) instead of B_a MN-major
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    constexpr uint32_t RB = RP * 2;
    constexpr uint32_t kSwR = RB >= 128 ? kSw128 : (RB == 64 ? kSw64 : kSw32);
    constexpr uint32_t kStg1 = u_stage_bytes<RP, NPJ>();   // one 64-wide K-block (sub-stage)
    constexpr uint32_t kStg = KW * kStg1;
    constexpr int ST = u_stages<RP, NPJ, KW>();
    constexpr int NC = NPJ * RP;                        // accumulator columns (one TMEM buffer)
    constexpr uint32_t kTm = 2 * NC <= 128 ? 128 : 256; // two buffers
    const uint32_t bar = base + ST * kStg;
    auto full_bar = [&](int s) { return bar + 8u * s; };
    auto empty_bar = [&](int s) { return bar + 8u * (ST + s); };
    const uint32_t accf0 = bar + 16u * ST;   // acc_full[2], acc_empty[2]
    const uint32_t tmem_slot = accf0 + 32;
    auto mask_bar = [&](int s) { return accf0 + 48u + 8u * s; };   // dropout: the X stage is masked
    auto a_addr = [&](int s, int i = 0) { return base + s * kStg + i * kStg1; };
    auto b_addr = [&](int s, int i = 0) { return base + s * kStg + i * kStg1 + kABytes; };
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
        for (int s = 0; s < ST; ++s) mbar_init(mask_bar(s), 64);
        fence_mbar_init();
        tma_prefetch_desc(&args.tmDY);
    }
    if (warp == 2) tmem_alloc(tmem_slot, kTm);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t *>(base_ptr + (tmem_slot - base));
    pdl_wait();
    pdl_trigger();
    const int total = args.n_items * args.ksplit;
    const int nkb = args.K / kBK;
    auto kb_range = [&](int split, int &kb0, int &kb1) {
        const int q = nkb / args.ksplit, rm = nkb % args.ksplit;
        kb0 = split * q + min(split, rm);
        kb1 = kb0 + q + (split < rm ? 1 : 0);
    };
    // forward pre-shrink of a FINETUNE tile with LoRA dropout: warps 2-3 zero the dropped X
    // elements of each staged K-block before the MMA reads it (the 1/(1-p) is applied in the reduce)
    auto masked_item = [&](int w) {
        return args.vf && args.drop.on && (args.tiles[args.items[w / args.ksplit]].flags & kTileFT);
    };
    if (warp == 2 || warp == 3) {
        if (args.vf && args.drop.on) {
            int stage = 0;
            uint32_t phase = 0, mph = 0;
            const int tid = threadIdx.x - 64;
            for (int w = blockIdx.x; w < total; w += gridDim.x) {
                const int split = w % args.ksplit;
                int kb0, kb1;
                kb_range(split, kb0, kb1);
                const bool mk = masked_item(w);
                const DevTile t = args.tiles[args.items[w / args.ksplit]];
                for (int kb = kb0; kb < kb1; kb += KW) {
                    if (mk) {
                        const int nb = min(KW, kb1 - kb);
                        mbar_wait(full_bar(stage), phase);
                        for (int i = 0; i < nb; ++i)
                            drop_mask_box_sw128(args.drop, base_ptr + (a_addr(stage, i) - base), 128, (uint32_t)t.row0,
                                                (uint32_t)(kb + i) * kBK, tid, 64);
                        fence_proxy_async_smem();
                        mbar_arrive(mask_bar(stage));
                        mph ^= 1u << stage;
                    }
                    if (++stage == ST) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            const int item = w / args.ksplit, split = w % args.ksplit;
            const DevTile t = args.tiles[args.items[item]];
            const SlotDev *sd = args.slots + t.slot;
            int kb0, kb1;
            kb_range(split, kb0, kb1);
            for (int kb = kb0; kb < kb1; kb += KW) {
                const int nb = min(KW, kb1 - kb);
                mbar_wait(empty_bar(stage), phase ^ 1);
                if (lane == 0) {
                    mbar_expect_tx(full_bar(stage), (uint32_t)nb * (kABytes + 64u * RB * NPJ));
                    for (int i = 0; i < nb; ++i)   // the X rows of both sub-stages back to back
                        tma_load_2d(a_addr(stage, i), &args.tmDY, full_bar(stage), (kb + i) * kBK, t.row0);
                    for (int i = 0; i < nb; ++i) {
                        if (NPJ > 1) {
                            // the A_a of every projection stacked: N = NPJ * r_pad rows of the B operand
#pragma unroll
                            for (int pj = 0; pj < NPJ; ++pj)
                                tma_load_2d(b_addr(stage, i) + (uint32_t)pj * RP * 128u, &args.slots_p[pj][t.slot].tmA,
                                            full_bar(stage), (kb + i) * kBK, 0);
                        } else if (args.vf) {
                            tma_load_2d(b_addr(stage, i), &sd->tmA, full_bar(stage), (kb + i) * kBK, 0);
                        } else {
                            tma_load_2d(b_addr(stage, i), &sd->tmBk, full_bar(stage), 0, (kb + i) * kBK);
                        }
                    }
                }
                __syncwarp();
                if (++stage == ST) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        int stage = 0;
        uint32_t phase = 0, it = 0, mph = 0;
        constexpr uint32_t idesc_u = idesc_bf16(128, RP, 0, 1), idesc_v = idesc_bf16(128, NC, 0, 0);
        const bool vf = args.vf != 0;
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            const int split = w % args.ksplit;
            int kb0, kb1;
            kb_range(split, kb0, kb1);
            const uint32_t b = it & 1, u = it >> 1;
            const uint32_t acc = tmem_base + b * NC;
            mbar_wait(accf0 + 16 + 8 * b, (u & 1) ^ 1);
            tc_fence_after();
            uint32_t acc_on = 0;
            const bool mk = masked_item(w);
            for (int kb = kb0; kb < kb1; kb += KW) {
                const int nb = min(KW, kb1 - kb);
                if (mk) {
                    mbar_wait(mask_bar(stage), (mph >> stage) & 1u);
                    mph ^= 1u << stage;
                } else {
                    mbar_wait(full_bar(stage), phase);
                }
                tc_fence_after();
                if (lane == 0) {
                    for (int i = 0; i < nb; ++i) {
                        const uint32_t ab = a_addr(stage, i), bb = b_addr(stage, i);
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k) {
                            if (vf)
                                mma_bf16(acc, smem_desc(ab + 32u * k, 16, 1024, kSw128),
                                         smem_desc(bb + 32u * k, 16, 1024, kSw128), idesc_v, acc_on);
                            else
                                mma_bf16(acc, smem_desc(ab + 32u * k, 16, 1024, kSw128),
                                         smem_desc(bb + 16u * RB * k, 64u * RB, 8u * RB, kSwR), idesc_u, acc_on);
                            acc_on = 1;
                        }
                    }
                    mma_commit(empty_bar(stage));
                }
                __syncwarp();
                if (++stage == ST) { stage = 0; phase ^= 1; }
            }
            if (lane == 0) mma_commit(accf0 + 8 * b);
            __syncwarp();
            ++it;
        }
    } else if (warp >= 4) {
        const int q = warp - 4;
        const int m = q * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        uint32_t it = 0;
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            const int item = w / args.ksplit, split = w % args.ksplit;
            const uint32_t b = it & 1, u = it >> 1;
            mbar_wait(accf0 + 8 * b, u & 1);
            tc_fence_after();
            float *dst = args.part + (((size_t)item * args.ksplit + split) * 128 + m) * NC;
#pragma unroll
            for (int c = 0; c < NC; c += 16) {
                uint32_t v[16];
                tmem_ld16(tmem_base + b * NC + lane_base + c, v);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 16; j += 4)
                    *reinterpret_cast<float4 *>(dst + c + j) =
                        make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                                    __uint_as_float(v[j + 3]));
            }
            tc_fence_before();
            mbar_arrive(accf0 + 16 + 8 * b);
            if (args.ctr) {
                // the last split of the item to arrive reduces it (split order, as u_reduce_kernel);
                // the counter returns to 0 for the next launch
                __shared__ int s_last;
                __threadfence();
                named_bar_sync(1, 128);
                if (threadIdx.x == 128) {
                    const int old = atomicAdd(args.ctr + item, 1);
                    s_last = old == args.ksplit - 1;
                    if (s_last) args.ctr[item] = 0;
                }
                named_bar_sync(1, 128);
                if (s_last) {
                    __threadfence();
                    u_reduce_row<RP, NPJ>(args, item, m);
                }
            }
            ++it;
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTm);
    }
}

template <int RP, int NPJ = 1, int KW = 2>
int launch_u_impl(const UArgs &a, int num_sms, cudaStream_t st) {
    auto kern = smlm_u_kernel<RP, NPJ, KW>;
    constexpr size_t kStg = KW * u_stage_bytes<RP, NPJ>();
    const size_t smem = 1024 + u_stages<RP, NPJ, KW>() * kStg + 512;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        attr_done = true;
    }
    const int total = a.n_items * a.ksplit;
    cudaError_t e = launch_pdl(kern, dim3(total < num_sms ? total : num_sms), dim3(kThreads), smem, st, a);
    if (e != cudaSuccess || a.ctr) return (int)e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.n_items);
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, u_reduce_kernel<RP, NPJ>, a);
}

}  // namespace

// Shared-memory bytes and pipeline depth for a given r_pad.
int gemm_stages(int r_pad, size_t *smem_bytes) {
    const size_t stage = kABytes + kBBytes;
    const size_t fixed = 1024 + (size_t)128 * r_pad * 2 + 256;
    int stages = (int)((232448 - fixed) / stage);
    if (stages > 6) stages = 6;
    if (smem_bytes) *smem_bytes = fixed + stage * stages;
    return stages;
}

int launch_u(const UArgs &a, int num_sms, cudaStream_t st) {
    if (a.n_items == 0) return 0;
    if (a.npj > 1) {   // forward pre-shrink of several projections (npj * r_pad <= 128)
        switch (a.r_pad * 8 + a.npj) {
            case 16 * 8 + 2: return launch_u_impl<16, 2>(a, num_sms, st);
            case 16 * 8 + 3: return launch_u_impl<16, 3>(a, num_sms, st);
            case 16 * 8 + 4: return launch_u_impl<16, 4>(a, num_sms, st);
            case 32 * 8 + 2: return launch_u_impl<32, 2>(a, num_sms, st);
            case 32 * 8 + 3: return launch_u_impl<32, 3>(a, num_sms, st);
            case 32 * 8 + 4: return launch_u_impl<32, 4>(a, num_sms, st);
            case 64 * 8 + 2: return launch_u_impl<64, 2>(a, num_sms, st);
        }
        return (int)cudaErrorInvalidValue;
    }
    switch (a.r_pad) {
        case 16: return launch_u_impl<16>(a, num_sms, st);
        case 32: return launch_u_impl<32>(a, num_sms, st);
        case 64: return launch_u_impl<64>(a, num_sms, st);
    }
    return (int)cudaErrorInvalidValue;
}

int launch_tok(const TokArgs &a, int num_sms, cudaStream_t st) {
    if (a.n_groups == 0) return 0;
    if (a.nh != 2) return (int)cudaErrorInvalidValue;   // 256-column items only
    switch (a.r_pad) {
        case 16: return launch_tok_impl<16, 2>(a, num_sms, st);
        case 32: return launch_tok_impl<32, 2>(a, num_sms, st);
        case 64: return launch_tok_impl<64, 2>(a, num_sms, st);
    }
    return (int)cudaErrorInvalidValue;
}

int launch_gemm(const GemmArgs &a, bool bwd, int num_sms, cudaStream_t st) {
    size_t smem = 0;
    gemm_stages(a.r_pad, &smem);
    if (a.n_tiles == 0 || a.n_ntiles == 0) return 0;
    if (bwd) {
        switch (a.r_pad) {
            case 16: return launch_impl<true, 16>(a, num_sms, smem, st);
            case 32: return launch_impl<true, 32>(a, num_sms, smem, st);
            case 64: return launch_impl<true, 64>(a, num_sms, smem, st);
        }
    } else {
        switch (a.r_pad) {
            case 16: return launch_impl<false, 16>(a, num_sms, smem, st);
            case 32: return launch_impl<false, 32>(a, num_sms, smem, st);
            case 64: return launch_impl<false, 64>(a, num_sms, smem, st);
        }
    }
    return (int)cudaErrorInvalidValue;
}

}  // namespace smlm
