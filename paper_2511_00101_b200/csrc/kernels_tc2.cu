// kernels_tc2.cu -- the SMLM GEMM on CTA pairs (tcgen05 cta_group::2, M = 256): the long-segment
// forward, the base + expand of short (decode) tiles inside mixed batches (a3), and
// the backward dX (a4).
//
// Work item = (pair of 128-row tiles, projection, 256-column n-tile).  The two tiles of a pair
// are any two consecutive tiles of the plan -- of the same segment or not: each CTA stages its
// own 128 rows of X (dY) and HALF of the 256-row B tile (W rows [n0, n0+128) in CTA 0, [n0+128,
// n0+256) in CTA 1), and the leader issues one M=256 N=256 K=16 MMA per K-step.  After the K loop
// the LoRA term lands in the same accumulator as extra K-blocks of depth r_pad ("expand"):
//   forward  : A = s*V rows (pre-shrunk once per long tile, DESIGN K1a; block-diagonal s*V of a
//              short tile's adapter block), B = B_a rows of the n-tile;
//   backward : A = s*U rows (DESIGN K5), B = A_a columns of the n-tile (MN-major).
// One expand block per distinct adapter of the pair: when the two tiles belong to different
// adapters (or one has none), each block zero-fills the other CTA's A rows (a fully out-of-bounds
// TMA box), so every row only receives its own adapter's term.  Pairing tiles across segments
// leaves only the partial 128-row tile at each segment end as padding (instead of a 256-row pair).
// Several projections that share X (q/k/v, gate/up: smlm_forward_multi) ride in ONE launch: the
// n-tiles of all projections form one persistent work list (no per-projection wave tail).
// Only the leader CTA (rank 0) issues MMAs; completions are multicast to both CTAs; two 256-column
// TMEM accumulators let the epilogue of item i overlap the main loop of item i+1.
// Backward with LoRA dropout (DESIGN R13): dx = W^T dy + keep * scale * (s A_a^T u) -- the mask
// multiplies only the LoRA term, so the expand blocks accumulate into the SECOND accumulator and
// the epilogue combines the two with the keep mask (one item in flight: no epilogue overlap).
#include <cuda_runtime.h>
#include <cstdio>

#include "device_types.h"
#include "dropout.cuh"
#include "pdl.cuh"
#include "sm100.cuh"

namespace smlm {
using namespace sm100;

namespace {

constexpr int kThreads2 = 256;
constexpr uint32_t kA2 = 128 * 128;   // own 128 X rows x 64 k
constexpr uint32_t kB2 = 128 * 128;   // half of the 256 B rows x 64 k
constexpr uint32_t kStage2 = kA2 + kB2;

// item w -> (pair pi, global n-tile gnt): raster groups of group_m pairs x every n-tile of every
// projection (the group's X tiles stay L2-resident while the W tiles stream)
__device__ __forceinline__ void decode_pair(int w, int n_pairs, int n_nt, int group_m, int &pi, int &gnt) {
    const int gsz = group_m * n_nt;
    const int g = w / gsz;
    const int first = g * group_m;
    const int gm = min(group_m, n_pairs - first);
    const int local = w - g * gsz;
    pi = first + local % gm;
    gnt = local / gm;
}

__device__ __forceinline__ int proj_of(const Gemm2Args &a, int gnt) {
    int p = 0;
#pragma unroll
    for (int i = 1; i < kGemm2MaxProj; ++i)
        if (i < a.n_proj && gnt >= a.proj[i].nt0) p = i;
    return p;
}

// expand blocks of a pair: one per adapter block of each half (a long tile with an adapter: 1;
// a short tile: its adapter blocks); two long halves with the same adapter share one block
__device__ __forceinline__ bool merged(const DevPair &pr) {
    const DevHalf &a = pr.h[0], &b = pr.h[1];
    return !(a.flags & kPairShort) && !(b.flags & kPairShort) && a.slot >= 0 && a.slot == b.slot && b.rows > 0;
}
__device__ __forceinline__ int half_blocks(const DevHalf &h) {
    if (h.rows <= 0) return 0;
    return (h.flags & kPairShort) ? h.nblk : (h.slot >= 0 ? 1 : 0);
}
__device__ __forceinline__ int n_expand(const DevPair &pr) {
    return merged(pr) ? 1 : half_blocks(pr.h[0]) + half_blocks(pr.h[1]);
}

template <bool BWD, int RP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    smlm_gemm2_kernel(const __grid_constant__ Gemm2Args args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    constexpr uint32_t RB = RP * 2;
    constexpr uint32_t kSwR = RB >= 128 ? kSw128 : (RB == 64 ? kSw64 : kSw32);
    const int stages = args.stages;
    const uint32_t bar = base + stages * kStage2;
    auto full_bar = [&](int s) { return bar + 8u * s; };
    auto empty_bar = [&](int s) { return bar + 8u * (stages + s); };
    const uint32_t acc_full0 = bar + 16u * stages;
    const uint32_t acc_empty0 = acc_full0 + 16;
    const uint32_t tmem_slot = acc_full0 + 32;
    auto a_addr = [&](int s) { return base + s * kStage2; };
    auto b_addr = [&](int s) { return base + s * kStage2 + kA2; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(acc_full0 + 8 * b, 1);
            mbar_init(acc_empty0 + 8 * b, 256);   // both CTAs' epilogue threads (leader's copy is used)
        }
        fence_mbar_init();
        for (int p = 0; p < args.n_proj; ++p) {
            tma_prefetch_desc(&args.proj[p].tmA);
            tma_prefetch_desc(&args.proj[p].tmW);
            if (args.proj[p].has_u) tma_prefetch_desc(&args.proj[p].tmU);
            if (args.proj[p].has_v) tma_prefetch_desc(&args.proj[p].tmV);
        }
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t *>(base_ptr + (tmem_slot - base));
    auto acc_col = [&](uint32_t b) { return tmem_base + 256u * b; };
    pdl_wait();
    pdl_trigger();

    const int n_clusters = gridDim.x / 2;
    const int cid = blockIdx.x / 2;
    const int total = args.n_pairs * args.n_nt;
    const bool drop = BWD && args.drop.on;

    if (warp == 0) {
        // ========================= TMA producer (both CTAs) =========================
        int stage = 0;
        uint32_t phase = 0;
        auto advance = [&]() {
            if (++stage == stages) { stage = 0; phase ^= 1; }
        };
        // X tiles are re-read for every n-tile of their raster group: keep them in L2
        uint64_t pol_keep;
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
        for (int w = cid; w < total; w += n_clusters) {
            int pi, gnt;
            decode_pair(w, args.n_pairs, args.n_nt, args.group_m, pi, gnt);
            const int p = proj_of(args, gnt);
            const Gemm2Proj &P = args.proj[p];
            const DevPair pr = args.pairs[pi];
            const DevHalf &mine = pr.h[rank];
            const int n0 = (gnt - P.nt0) * kBN;
            const int nkb = P.K / kBK;
            // backward: W column boxes past N are skipped (in is a multiple of 64)
            auto nbox = [&](int rk) {
                int nb = 0;
                for (int i = 0; i < 2; ++i) nb += (n0 + 128 * rk + 64 * i < P.N);
                return nb;
            };
            const uint32_t bytes_pair = BWD ? 2u * kA2 + 8192u * (nbox(0) + nbox(1)) : 2u * kStage2;
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(empty_bar(stage), phase ^ 1);
                if (lane == 0) {
                    const uint32_t fb = map_to_rank(full_bar(stage), 0);   // the leader's barrier
                    if (leader) mbar_expect_tx(full_bar(stage), bytes_pair);
                    tma_load_2d_pair_hint(a_addr(stage), &P.tmA, fb, kb * kBK, mine.row0, pol_keep);
                    if (BWD) {
                        for (int i = 0; i < 2; ++i) {
                            const int c0 = n0 + 128 * (int)rank + 64 * i;
                            if (c0 < P.N) tma_load_2d_pair(b_addr(stage) + 8192u * i, &P.tmW, fb, c0, kb * kBK);
                        }
                    } else {
                        tma_load_2d_pair(b_addr(stage), &P.tmW, fb, kb * kBK, n0 + 128 * (int)rank);
                    }
                }
                __syncwarp();
                advance();
            }
            // expand blocks: A = this CTA's s*V / s*U rows of the block (zeros if the block belongs
            // to the other half), B = the block adapter's B_a rows (fwd) / A_a columns (bwd)
            const int nb0 = merged(pr) ? 1 : half_blocks(pr.h[0]);
            const int nexp = n_expand(pr);
            for (int j = 0; j < nexp; ++j) {
                const int owner = merged(pr) ? (int)rank : (j < nb0 ? 0 : 1);
                const DevHalf &h = pr.h[owner];
                const int jj = (merged(pr) || owner == 0) ? j : j - nb0;
                const bool is_short = (h.flags & kPairShort) != 0;
                const int slot = is_short ? args.blocks[h.blk0 + jj].slot : h.slot;
                const SlotDev *sd = P.slots + slot;
                // long tiles: tile-compact s*V (fwd, tmV) / s*U (bwd, tmU); short: block-diagonal s*V (tmU)
                const CUtensorMap *amap = (!BWD && !is_short) ? &P.tmV : &P.tmU;
                const int arow = owner == (int)rank ? (is_short ? (h.blk0 + jj) * 128 : h.tile * 128)
                                                    : ((!BWD && !is_short) ? P.v_rows : P.u_rows);   // OOB: zeros
                mbar_wait(empty_bar(stage), phase ^ 1);
                if (lane == 0) {
                    const uint32_t fb = map_to_rank(full_bar(stage), 0);
                    if (leader) mbar_expect_tx(full_bar(stage), 2u * 256u * RB);
                    tma_load_2d_pair(a_addr(stage), amap, fb, 0, arow);
                    if (BWD) {
                        for (int i = 0; i < 2; ++i)
                            tma_load_2d_pair(b_addr(stage) + (uint32_t)i * RP * 128u, &sd->tmA, fb,
                                             n0 + 128 * (int)rank + 64 * i, 0);
                    } else {
                        const int rb0 = n0 + 128 * (int)rank;
                        tma_load_2d_pair(b_addr(stage), &sd->tmBk, fb, 0, rb0);
                        tma_load_2d_pair(b_addr(stage) + 64u * RB, &sd->tmBk, fb, 0, rb0 + 64);
                    }
                }
                __syncwarp();
                advance();
            }
        }
    } else if (warp == 1 && leader) {
        // ========================= MMA issuer (leader CTA) =========================
        int stage = 0;
        uint32_t phase = 0;
        auto advance = [&]() {
            if (++stage == stages) { stage = 0; phase ^= 1; }
        };
        constexpr uint32_t idesc = idesc_bf16(256, 256, 0, BWD ? 1 : 0);
        uint32_t it = 0;
#ifdef SMLM_MEASURE
        long long t_full = 0, t_acc = 0, n_full = 0;
        const long long t_begin = clock64();
        auto timed_wait = [&](uint32_t bar_, uint32_t ph_, long long &acc_) {
            const long long t0 = clock64();
            mbar_wait(bar_, ph_);
            acc_ += clock64() - t0;
        };
#define SMLM_WAIT_FULL(b_, p_) timed_wait(b_, p_, t_full)
#define SMLM_WAIT_ACC(b_, p_) timed_wait(b_, p_, t_acc)
#else
#define SMLM_WAIT_FULL(b_, p_) mbar_wait(b_, p_)
#define SMLM_WAIT_ACC(b_, p_) mbar_wait(b_, p_)
#endif
        for (int w = cid; w < total; w += n_clusters) {
            int pi, gnt;
            decode_pair(w, args.n_pairs, args.n_nt, args.group_m, pi, gnt);
            const DevPair pr = args.pairs[pi];
            const int nkb = args.proj[proj_of(args, gnt)].K / kBK;
            const uint32_t b = drop ? 0u : (it & 1), u = drop ? it : (it >> 1);
            const uint32_t acc = acc_col(b);
            SMLM_WAIT_ACC(acc_empty0 + 8 * b, (u & 1) ^ 1);
            if (drop) mbar_wait(acc_empty0 + 8, (u & 1) ^ 1);   // the LoRA accumulator
            tc_fence_after();
            for (int kb = 0; kb < nkb; ++kb) {
                SMLM_WAIT_FULL(full_bar(stage), phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t ab = a_addr(stage), bb = b_addr(stage);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                        mma2_bf16(acc, smem_desc(ab + 32u * k, 16, 1024, kSw128),
                                  BWD ? smem_desc(bb + 2048u * k, 8192, 1024, kSw128)
                                      : smem_desc(bb + 32u * k, 16, 1024, kSw128),
                                  idesc, (kb | k) != 0);
                    mma2_commit_mc(empty_bar(stage));
                }
                __syncwarp();
                advance();
            }
            const int nexp = n_expand(pr);
            for (int j = 0; j < nexp; ++j) {
                mbar_wait(full_bar(stage), phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t ab = a_addr(stage), bb = b_addr(stage);
#pragma unroll
                    for (int kk = 0; kk < RP / 16; ++kk)
                        mma2_bf16(drop ? acc_col(1) : acc, smem_desc(ab + 32u * kk, 16, 8u * RB, kSwR),
                                  BWD ? smem_desc(bb + 2048u * kk, (uint32_t)RP * 128u, 1024, kSw128)
                                      : smem_desc(bb + 32u * kk, 16, 8u * RB, kSwR),
                                  idesc, (!drop || j > 0 || kk > 0) ? 1u : 0u);
                    mma2_commit_mc(empty_bar(stage));
                }
                __syncwarp();
                advance();
            }
            if (lane == 0) mma2_commit_mc(acc_full0 + 8 * b);
            __syncwarp();
            ++it;
        }
#ifdef SMLM_MEASURE
        if (args.dbg && lane == 0 && (cid % 8) == 0)
            printf("[gemm2 %s] cluster %d items %u cycles %lld wait_operands %lld (%.1f%%) wait_acc %lld (%.1f%%)\n",
                   BWD ? "bwd" : "fwd", cid, it, clock64() - t_begin, t_full, 100.0 * t_full / (clock64() - t_begin), t_acc,
                   100.0 * t_acc / (clock64() - t_begin));
#endif
#undef SMLM_WAIT_FULL
#undef SMLM_WAIT_ACC
    } else if (warp >= 4) {
        // ========================= epilogue (both CTAs, own 128 rows) =========================
        const int q = warp - 4;
        const int m = q * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const uint32_t acc_empty_l = map_to_rank(acc_empty0, 0);
        uint32_t it = 0;
        for (int w = cid; w < total; w += n_clusters) {
            int pi, gnt;
            decode_pair(w, args.n_pairs, args.n_nt, args.group_m, pi, gnt);
            const int p = proj_of(args, gnt);
            const Gemm2Proj &P = args.proj[p];
            const DevHalf mine = args.pairs[pi].h[rank];
            const bool dl = drop && n_expand(args.pairs[pi]) > 0;   // a LoRA accumulator to combine
            const int n0 = (gnt - P.nt0) * kBN;
            const bool row_ok = m < mine.rows;
            const int row = mine.row0 + m;
            __nv_bfloat16 *Y = reinterpret_cast<__nv_bfloat16 *>(P.Y);
            const uint32_t b = drop ? 0u : (it & 1), u = drop ? it : (it >> 1);
            mbar_wait(acc_full0 + 8 * b, u & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < kBN / 16; ++c) {
                uint32_t r[16];
                tmem_ld16(acc_col(b) + lane_base + 16u * c, r);
                tmem_wait_ld();
                const int col = n0 + 16 * c;
                if (dl) {
                    uint32_t l[16];
                    tmem_ld16(acc_col(1) + lane_base + 16u * c, l);
                    tmem_wait_ld();
                    if (row_ok) {
#pragma unroll
                        for (int e = 0; e < 16; e += 2) {
                            const uint32_t kp = drop_keep2(args.drop, (uint32_t)row, (uint32_t)(col + e));
                            r[e] = __float_as_uint(__uint_as_float(r[e]) +
                                                   ((kp & 1u) ? args.drop.scale * __uint_as_float(l[e]) : 0.f));
                            r[e + 1] = __float_as_uint(__uint_as_float(r[e + 1]) +
                                                       ((kp & 2u) ? args.drop.scale * __uint_as_float(l[e + 1]) : 0.f));
                        }
                    }
                }
                if (row_ok && col < P.N) {
                    uint4 *dst = reinterpret_cast<uint4 *>(Y + (size_t)row * P.N + col);
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
            tc_fence_before();
            mbar_arrive_cluster(acc_empty_l + 8 * b);
            if (drop) mbar_arrive_cluster(acc_empty_l + 8);
            ++it;
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
    }
}

// ======================= forward, 512-column items (both TMEM halves) =======================
// The 256 x 256 item above moves 64 KB of operands into the pair per 8.4 MFLOP and waits for
// them ~19 % of the time at ~11 TB/s of L2 -> SM traffic (the measured MMA-issuer operand waits);
// a 256 x 512 item reuses each staged X tile for two W halves: 96 KB per 16.8 MFLOP (25 % fewer
// bytes per flop).  Both 256-column accumulators belong to one item, so the epilogue drains
// half 0, then half 1, and the next item's half-1 MMAs are deferred (their stages held in the
// ring) until half 1 is drained: the tensor pipe keeps working on half 0 meanwhile.
constexpr uint32_t kStageW = kA2 + 2 * kB2;   // X 128 rows + W half 0 + W half 1 (128 rows each), 48 KB
constexpr uint32_t kYChunkW = 128 * 64 * 2;   // 128 rows x 64 bf16 columns, SW128 (one TMA store)

__device__ __forceinline__ void tma_store_2d_w(const void *map, uint32_t ssrc, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(ssrc), "r"(c0), "r"(c1)
                 : "memory");
}

// global n-tile pair -> (projection, first column); n-tiles pair up inside each projection (an
// odd last one is a half-empty pair: its W box is out of bounds, zero-filled, and not stored)
__device__ __forceinline__ int proj_of_w(const Gemm2Args &a, int gq, int &n0) {
    int q0 = 0, pp = 0;
    n0 = gq * 512;
#pragma unroll
    for (int p = 0; p < kGemm2MaxProj; ++p) {
        if (p < a.n_proj) {
            const int nq = ((a.proj[p].N + 255) / 256 + 1) / 2;
            if (gq >= q0) {
                pp = p;
                n0 = (gq - q0) * 512;
            }
            q0 += nq;
        }
    }
    return pp;
}

template <int RP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    smlm_gemm2w_kernel(const __grid_constant__ Gemm2Args args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    constexpr uint32_t RB = RP * 2;
    constexpr uint32_t kSwR = RB >= 128 ? kSw128 : (RB == 64 ? kSw64 : kSw32);
    const int stages = args.stages;
    const uint32_t stg = base + stages * kStageW;   // 2 x 16 KB: bf16 64-column chunks for the TMA stores
    const uint32_t bar = stg + 2u * kYChunkW;
    auto full_bar = [&](int s) { return bar + 8u * s; };
    auto empty_bar = [&](int s) { return bar + 8u * (stages + s); };
    const uint32_t acc_full = bar + 16u * stages;
    const uint32_t acc_empty0 = acc_full + 8;   // half h: acc_empty0 + 8 h
    const uint32_t tmem_slot = acc_full + 24;
    auto a_addr = [&](int s) { return base + s * kStageW; };
    auto b_addr = [&](int s, int h) { return base + s * kStageW + kA2 + (uint32_t)h * kB2; };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty0, 256);       // both CTAs' epilogue threads (leader's copy is used)
        mbar_init(acc_empty0 + 8, 256);
        fence_mbar_init();
        for (int p = 0; p < args.n_proj; ++p) {
            tma_prefetch_desc(&args.proj[p].tmA);
            tma_prefetch_desc(&args.proj[p].tmW);
            if (args.proj[p].has_u) tma_prefetch_desc(&args.proj[p].tmU);
            if (args.proj[p].has_v) tma_prefetch_desc(&args.proj[p].tmV);
        }
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t *>(base_ptr + (tmem_slot - base));
    auto acc_col = [&](int h) { return tmem_base + 256u * (uint32_t)h; };
    pdl_wait();
    pdl_trigger();

    const int n_clusters = gridDim.x / 2;
    const int cid = blockIdx.x / 2;
    int n_nt2 = 0;
#pragma unroll
    for (int p = 0; p < kGemm2MaxProj; ++p)
        if (p < args.n_proj) n_nt2 += ((args.proj[p].N + 255) / 256 + 1) / 2;
    const int total = args.n_pairs * n_nt2;

    if (warp == 0) {
        // ========================= TMA producer (both CTAs) =========================
        int stage = 0;
        uint32_t phase = 0;
        auto advance = [&]() {
            if (++stage == stages) { stage = 0; phase ^= 1; }
        };
        uint64_t pol_keep;   // X tiles are re-read for every n-tile pair of their raster group
        asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
        for (int w = cid; w < total; w += n_clusters) {
            int pi, gq, n0;
            decode_pair(w, args.n_pairs, n_nt2, args.group_m, pi, gq);
            const int p = proj_of_w(args, gq, n0);
            const Gemm2Proj &P = args.proj[p];
            const DevPair pr = args.pairs[pi];
            const DevHalf &mine = pr.h[rank];
            const int nkb = P.K / kBK;
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(empty_bar(stage), phase ^ 1);
                if (lane == 0) {
                    const uint32_t fb = map_to_rank(full_bar(stage), 0);   // the leader's barrier
                    if (leader) mbar_expect_tx(full_bar(stage), 2u * kStageW);
                    tma_load_2d_pair_hint(a_addr(stage), &P.tmA, fb, kb * kBK, mine.row0, pol_keep);
                    tma_load_2d_pair(b_addr(stage, 0), &P.tmW, fb, kb * kBK, n0 + 128 * (int)rank);
                    tma_load_2d_pair(b_addr(stage, 1), &P.tmW, fb, kb * kBK, n0 + 256 + 128 * (int)rank);
                }
                __syncwarp();
                advance();
            }
            // expand blocks: A = this CTA's s*V rows of the block (zeros if the block belongs to the
            // other half), B = the block adapter's B_a rows of both column halves
            const int nb0 = merged(pr) ? 1 : half_blocks(pr.h[0]);
            const int nexp = n_expand(pr);
            for (int j = 0; j < nexp; ++j) {
                const int owner = merged(pr) ? (int)rank : (j < nb0 ? 0 : 1);
                const DevHalf &h = pr.h[owner];
                const int jj = (merged(pr) || owner == 0) ? j : j - nb0;
                const bool is_short = (h.flags & kPairShort) != 0;
                const int slot = is_short ? args.blocks[h.blk0 + jj].slot : h.slot;
                const SlotDev *sd = P.slots + slot;
                const CUtensorMap *amap = is_short ? &P.tmU : &P.tmV;
                const int arow = owner == (int)rank ? (is_short ? (h.blk0 + jj) * 128 : h.tile * 128)
                                                    : (is_short ? P.u_rows : P.v_rows);   // OOB: zeros
                mbar_wait(empty_bar(stage), phase ^ 1);
                if (lane == 0) {
                    const uint32_t fb = map_to_rank(full_bar(stage), 0);
                    if (leader) mbar_expect_tx(full_bar(stage), 2u * 384u * RB);
                    tma_load_2d_pair(a_addr(stage), amap, fb, 0, arow);
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const int rb0 = n0 + 256 * hh + 128 * (int)rank;
                        tma_load_2d_pair(b_addr(stage, hh), &sd->tmBk, fb, 0, rb0);
                        tma_load_2d_pair(b_addr(stage, hh) + 64u * RB, &sd->tmBk, fb, 0, rb0 + 64);
                    }
                }
                __syncwarp();
                advance();
            }
        }
    } else if (warp == 1 && leader) {
        // ========================= MMA issuer (leader CTA) =========================
        int stage = 0;
        uint32_t phase = 0;
        constexpr uint32_t idesc = idesc_bf16(256, 256, 0, 0);
        uint32_t it = 0;
        int pst[8], pjj[8];   // stages whose half-1 MMAs wait for half 1 of the accumulator
#ifdef SMLM_MEASURE
        long long t_full = 0, t_acc = 0;
        const long long t_begin = clock64();
#endif
        for (int w = cid; w < total; w += n_clusters) {
            int pi, gq, n0;
            decode_pair(w, args.n_pairs, n_nt2, args.group_m, pi, gq);
            const DevPair pr = args.pairs[pi];
            const int nkb = args.proj[proj_of_w(args, gq, n0)].K / kBK;
            const int nst = nkb + n_expand(pr);
            const uint32_t par = (it & 1) ^ 1;
#ifdef SMLM_MEASURE
            long long t0 = clock64();
#endif
            mbar_wait(acc_empty0, par);   // half 0 drained by the previous item's epilogue
#ifdef SMLM_MEASURE
            t_acc += clock64() - t0;
#endif
            tc_fence_after();
            bool h1 = false;
            int pend = 0;
            // half h of stage st (j-th stage of the item: a K-block, or an expand block past nkb)
            auto issue = [&](int st, int j, int hh) {
                const uint32_t ab = a_addr(st), bb = b_addr(st, hh);
                if (j < nkb) {
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                        mma2_bf16(acc_col(hh), smem_desc(ab + 32u * k, 16, 1024, kSw128), smem_desc(bb + 32u * k, 16, 1024, kSw128),
                                  idesc, (j | k) != 0);
                } else {
#pragma unroll
                    for (int kk = 0; kk < RP / 16; ++kk)
                        mma2_bf16(acc_col(hh), smem_desc(ab + 32u * kk, 16, 8u * RB, kSwR),
                                  smem_desc(bb + 32u * kk, 16, 8u * RB, kSwR), idesc, 1u);
                }
            };
            auto flush = [&]() {   // half-1 MMAs of the held stages, then release them
                if (lane == 0)
                    for (int q = 0; q < pend; ++q) {
                        issue(pst[q], pjj[q], 1);
                        mma2_commit_mc(empty_bar(pst[q]));
                    }
                __syncwarp();
                pend = 0;
            };
            for (int j = 0; j < nst; ++j) {
#ifdef SMLM_MEASURE
                t0 = clock64();
#endif
                mbar_wait(full_bar(stage), phase);
#ifdef SMLM_MEASURE
                t_full += clock64() - t0;
#endif
                tc_fence_after();
                if (lane == 0) issue(stage, j, 0);
                __syncwarp();
                if (h1) {
                    if (lane == 0) {
                        issue(stage, j, 1);
                        mma2_commit_mc(empty_bar(stage));
                    }
                    __syncwarp();
                } else {
                    pst[pend] = stage;
                    pjj[pend] = j;
                    ++pend;
                    // every ring stage held: the next stage cannot arrive before half 1 is free
                    if (pend == stages) {
                        mbar_wait(acc_empty0 + 8, par);
                        h1 = true;
                    } else {
                        h1 = mbar_test(acc_empty0 + 8, par) != 0;
                    }
                    if (h1) {
                        tc_fence_after();
                        flush();
                    }
                }
                if (++stage == stages) { stage = 0; phase ^= 1; }
            }
            if (pend > 0) {
                mbar_wait(acc_empty0 + 8, par);
                tc_fence_after();
                flush();
            }
            if (lane == 0) mma2_commit_mc(acc_full);
            __syncwarp();
            ++it;
        }
#ifdef SMLM_MEASURE
        if (args.dbg && lane == 0 && (cid % 8) == 0)
            printf("[gemm2w fwd] cluster %d items %u cycles %lld wait_operands %lld (%.1f%%) wait_acc0 %lld (%.1f%%)\n", cid, it,
                   clock64() - t_begin, t_full, 100.0 * t_full / (clock64() - t_begin), t_acc, 100.0 * t_acc / (clock64() - t_begin));
#endif
    } else if (warp >= 4) {
        // ========================= epilogue (both CTAs, own 128 rows) =========================
        // a full 128-row tile: 64-column chunks staged in shared memory (128-byte swizzle) and
        // stored by TMA (a warp's direct stores would touch 32 rows = 32 lines per instruction);
        // the last, partial tile of a segment: direct stores of its own rows
        const int q = warp - 4;
        const int m = q * 32 + lane;
        const int tid_e = threadIdx.x - 128;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const uint32_t acc_empty_l = map_to_rank(acc_empty0, 0);
        uint32_t it = 0, chunk = 0;
        for (int w = cid; w < total; w += n_clusters) {
            int pi, gq, n0;
            decode_pair(w, args.n_pairs, n_nt2, args.group_m, pi, gq);
            const int p = proj_of_w(args, gq, n0);
            const Gemm2Proj &P = args.proj[p];
            const DevHalf mine = args.pairs[pi].h[rank];
            const bool full = mine.rows == 128;
            const bool row_ok = m < mine.rows;
            const int row = mine.row0 + m;
            __nv_bfloat16 *Y = reinterpret_cast<__nv_bfloat16 *>(P.Y);
            mbar_wait(acc_full, it & 1);
            tc_fence_after();
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
#pragma unroll 1
                for (int c4 = 0; c4 < 4; ++c4) {
                    const int col = n0 + 256 * hh + 64 * c4;
                    if (col >= P.N) break;   // a half-empty pair (odd n-tile count)
                    const uint32_t buf = stg + (chunk & 1u) * kYChunkW;
                    if (full) {
                        // the TMA store that last read this buffer is done reading it
                        if (tid_e == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                        named_bar_sync(1, 128);
                    }
#pragma unroll 1
                    for (int c = 0; c < 4; ++c) {
                        uint32_t r[16];
                        tmem_ld16(acc_col(hh) + lane_base + 64u * c4 + 16u * c, r);
                        tmem_wait_ld();
                        uint4 pk[2];
#pragma unroll
                        for (int q4 = 0; q4 < 2; ++q4) {
                            pk[q4].x = pack_bf16x2(__uint_as_float(r[8 * q4 + 0]), __uint_as_float(r[8 * q4 + 1]));
                            pk[q4].y = pack_bf16x2(__uint_as_float(r[8 * q4 + 2]), __uint_as_float(r[8 * q4 + 3]));
                            pk[q4].z = pack_bf16x2(__uint_as_float(r[8 * q4 + 4]), __uint_as_float(r[8 * q4 + 5]));
                            pk[q4].w = pack_bf16x2(__uint_as_float(r[8 * q4 + 6]), __uint_as_float(r[8 * q4 + 7]));
                        }
                        if (full) {
#pragma unroll
                            for (int q4 = 0; q4 < 2; ++q4) {
                                const uint32_t u = (uint32_t)(2 * c + q4);   // 16-byte unit of the 128-byte row
                                const uint32_t off = (uint32_t)m * 128u + ((u ^ ((uint32_t)m & 7u)) << 4);
                                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + off), "r"(pk[q4].x),
                                             "r"(pk[q4].y), "r"(pk[q4].z), "r"(pk[q4].w)
                                             : "memory");
                            }
                        } else if (row_ok && col + 16 * c < P.N) {
                            uint4 *dst = reinterpret_cast<uint4 *>(Y + (size_t)row * P.N + col + 16 * c);
                            dst[0] = pk[0];
                            dst[1] = pk[1];
                        }
                    }
                    if (full) {
                        fence_proxy_async_smem();
                        named_bar_sync(1, 128);
                        if (tid_e == 0) {
                            tma_store_2d_w(&P.tmY, buf, col, mine.row0);
                            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                        }
                        ++chunk;
                    }
                }
                tc_fence_before();
                mbar_arrive_cluster(acc_empty_l + 8u * hh);   // half hh may take the next item's MMAs
            }
            ++it;
        }
        if (tid_e == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // staging read before exit
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
    }
}

template <int RP>
int launch2w_impl(const Gemm2Args &a, int num_sms, cudaStream_t st) {
    auto kern = smlm_gemm2w_kernel<RP>;
    const size_t smem = 1024 + (size_t)a.stages * kStageW + 2 * kYChunkW + 256;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        attr_done = true;
    }
    int n_nt2 = 0;
    for (int p = 0; p < a.n_proj; ++p) n_nt2 += ((a.proj[p].N + 255) / 256 + 1) / 2;
    const int total = a.n_pairs * n_nt2;
    int clusters = num_sms / 2;
    if (total < clusters) clusters = total;
    return (int)launch_pdl(kern, dim3(2 * clusters), dim3(kThreads2), smem, st, a);
}

template <bool BWD, int RP>
int launch2_impl(const Gemm2Args &a, int num_sms, cudaStream_t st) {
    auto kern = smlm_gemm2_kernel<BWD, RP>;
    const size_t smem = 1024 + (size_t)a.stages * kStage2 + 256;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        attr_done = true;
    }
    const int total = a.n_pairs * a.n_nt;
    int clusters = num_sms / 2;
    if (total < clusters) clusters = total;
    return (int)launch_pdl(kern, dim3(2 * clusters), dim3(kThreads2), smem, st, a);
}

}  // namespace

int gemm2_stages(int) {
    const size_t fixed = 1024 + 256;
    int s = (int)((232448 - fixed) / kStage2);
    return s > 8 ? 8 : s;
}
// the forward launches take the 512-column kernel (smlm_gemm2w_kernel): 4 stages of 48 KB
int gemm2w_stages() { return (int)((232448 - 1024 - 256 - 2 * kYChunkW) / kStageW); }

int launch_gemm2(const Gemm2Args &a, bool bwd, int num_sms, cudaStream_t st) {
    if (a.n_pairs == 0 || a.n_nt == 0) return 0;
    if (!bwd) {
        Gemm2Args w = a;
        w.stages = gemm2w_stages();
        switch (a.r_pad) {
            case 16: return launch2w_impl<16>(w, num_sms, st);
            case 32: return launch2w_impl<32>(w, num_sms, st);
            case 64: return launch2w_impl<64>(w, num_sms, st);
        }
        return (int)cudaErrorInvalidValue;
    }
    switch (a.r_pad * (bwd ? -1 : 1)) {
        case -16: return launch2_impl<true, 16>(a, num_sms, st);
        case -32: return launch2_impl<true, 32>(a, num_sms, st);
        case -64: return launch2_impl<true, 64>(a, num_sms, st);
    }
    return (int)cudaErrorInvalidValue;
}

}  // namespace smlm
