// kernels_tc2.cu -- forward SMLM GEMM on CTA pairs (tcgen05 cta_group::2, M = 256).
//
// Default forward (PRE = true, DESIGN K1): s*V was computed once per tile by the pre-shrink pass
// (kernels_tc.cu smlm_u_kernel, vf), so the n-tile is the full 256 W rows and the expand is one
// extra K-block whose A operand is the tile-compact s*V loaded by TMA.  PRE = false keeps the
// fused variant (SMLM_FUSED_SHRINK=1): A_a stacked under the W n-tile so the shrink rides in the
// N=256 MMA and V never leaves the SM pair (n-tile 256 - r_pad).  Each work item covers TWO
// 128-row tiles of the same segment (same adapter), one per CTA of a cluster pair.  The pair issues one M=256 MMA per K-step: each CTA stages its own 128 X rows and HALF
// of the 256-row B tile (W rows [n0, n0+128) in CTA 0; W rows [n0+128, n0+BNW) + A_a in CTA 1),
// halving the per-SM operand traffic of the 1-CTA kernel; 6 pipeline stages of 32 KB.
// Only the leader CTA (rank 0) issues MMAs; completions are multicast to both CTAs.
#include <cuda_runtime.h>

#include "device_types.h"
#include "pdl.cuh"
#include "sm100.cuh"

namespace smlm {
using namespace sm100;

namespace {

constexpr int kThreads2 = 256;
constexpr uint32_t kA2 = 128 * 128;   // own 128 X rows x 64 k
constexpr uint32_t kB2 = 128 * 128;   // half of the 256 B rows x 64 k
constexpr uint32_t kStage2 = kA2 + kB2;

__device__ __forceinline__ void decode_pair(int w, int n_pairs, int n_nt, int group_m, int &pi, int &nt) {
    const int gsz = group_m * n_nt;
    const int g = w / gsz;
    const int first = g * group_m;
    const int gm = min(group_m, n_pairs - first);
    const int local = w - g * gsz;
    pi = first + local % gm;
    nt = local / gm;
}

// PRE (forward only): s*V was precomputed once per tile (smlm_u_kernel, vf) -- the n-tile is the
// full 256 W rows (no A_a stacked under W, no per-n-tile re-shrink) and the expand K-block takes
// its A operand from the tile-compact s*V by TMA, like the backward's s*U.
template <bool BWD, int RP, bool PRE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    smlm_gemm2_kernel(const __grid_constant__ Gemm2Args args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    constexpr uint32_t RB = RP * 2;
    // forward: n-tile = 256 - RP output columns (A_a stacked under W in CTA 1's half of B);
    // backward: n-tile = 256 columns of dX, W as the MN-major B operand (two 64-column boxes per CTA)
    constexpr int BNW = (BWD || PRE) ? 256 : 256 - RP;
    constexpr int W1 = (BWD || PRE) ? 128 : BNW - 128;
    constexpr uint32_t kSwR = RB >= 128 ? kSw128 : (RB == 64 ? kSw64 : kSw32);
    const int stages = args.stages;
    const uint32_t sv_addr = base + stages * kStage2;
    const uint32_t bar = sv_addr + 128 * RB;
    auto full_bar = [&](int s) { return bar + 8u * s; };
    auto empty_bar = [&](int s) { return bar + 8u * (stages + s); };
    const uint32_t acc_full0 = bar + 16u * stages;
    const uint32_t acc_empty0 = acc_full0 + 16;
    const uint32_t v_full = acc_full0 + 32;
    const uint32_t sv_ready = acc_full0 + 40;
    const uint32_t tmem_slot = acc_full0 + 48;
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
        mbar_init(v_full, 1);
        mbar_init(sv_ready, 256);
        fence_mbar_init();
        tma_prefetch_desc(&args.tmX);
        tma_prefetch_desc(&args.tmW0);
        if (args.has_u) tma_prefetch_desc(&args.tmU);
        if (!BWD && !PRE) tma_prefetch_desc(&args.tmW1);
        if (PRE) tma_prefetch_desc(&args.tmV);
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
    const int total = args.n_pairs * args.n_ntiles;
    const int nkb = args.K / kBK;

    if (warp == 0) {
        // ========================= TMA producer (both CTAs) =========================
        int stage = 0;
        uint32_t phase = 0;
        auto advance = [&]() {
            if (++stage == stages) { stage = 0; phase ^= 1; }
        };
        for (int w = cid; w < total; w += n_clusters) {
            int pi, nt;
            decode_pair(w, args.n_pairs, args.n_ntiles, args.group_m, pi, nt);
            const DevPair pr = args.pairs[pi];
            const int n0 = nt * BNW;
            const bool lora = pr.slot >= 0;
            const SlotDev *sd = lora ? args.slots + pr.slot : nullptr;
            const int my_row0 = leader ? pr.row0 : pr.row0 + 128;
            // backward: W column boxes past N are skipped (in is a multiple of 64)
            auto nbox = [&](int rk) {
                int nb = 0;
                for (int i = 0; i < 2; ++i) nb += (n0 + 128 * rk + 64 * i < args.N);
                return nb;
            };
            const uint32_t bytes_pair =
                BWD ? 2u * kA2 + 8192u * (nbox(0) + nbox(1))
                    : 2u * kA2 + 128u * 128u + (uint32_t)W1 * 128u + ((lora && !PRE) ? RP * 128u : 0u);
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(empty_bar(stage), phase ^ 1);
                if (lane == 0) {
                    const uint32_t fb = map_to_rank(full_bar(stage), 0);   // the leader's barrier
                    if (leader) mbar_expect_tx(full_bar(stage), bytes_pair);
                    tma_load_2d_pair(a_addr(stage), &args.tmX, fb, kb * kBK, my_row0);
                    if (BWD) {
                        for (int i = 0; i < 2; ++i) {
                            const int c0 = n0 + 128 * (int)rank + 64 * i;
                            if (c0 < args.N) tma_load_2d_pair(b_addr(stage) + 8192u * i, &args.tmW0, fb, c0, kb * kBK);
                        }
                    } else if (leader) {
                        tma_load_2d_pair(b_addr(stage), &args.tmW0, fb, kb * kBK, n0);
                    } else if (PRE) {
                        tma_load_2d_pair(b_addr(stage), &args.tmW0, fb, kb * kBK, n0 + 128);
                    } else {
                        tma_load_2d_pair(b_addr(stage), &args.tmW1, fb, kb * kBK, n0 + 128);
                        if (lora) tma_load_2d_pair(b_addr(stage) + W1 * 128u, &sd->tmA, fb, kb * kBK, 0);
                    }
                }
                __syncwarp();
                advance();
            }
            if (!BWD && (pr.flags & kPairShort)) {
                // short tile (CTA 0; CTA 1 is a masked dummy): one K = r_pad block per adapter,
                // A = block-diagonal s*V rows, B = B_u rows [n0 + 128 rank, +128)
                for (int bi = 0; bi < pr.nblk; ++bi) {
                    const SlotDev *bs = args.slots + args.blocks[pr.blk0 + bi].slot;
                    mbar_wait(empty_bar(stage), phase ^ 1);
                    if (lane == 0) {
                        const uint32_t fb = map_to_rank(full_bar(stage), 0);
                        if (leader) mbar_expect_tx(full_bar(stage), 2u * 256u * RB);
                        tma_load_2d_pair(a_addr(stage), &args.tmU, fb, 0, (pr.blk0 + bi) * 128);
                        const int rb0 = n0 + 128 * (int)rank;
                        tma_load_2d_pair(b_addr(stage), &bs->tmBk, fb, 0, rb0);
                        tma_load_2d_pair(b_addr(stage) + 64u * RB, &bs->tmBk, fb, 0, rb0 + 64);
                    }
                    __syncwarp();
                    advance();
                }
            }
            if (lora) {
                mbar_wait(empty_bar(stage), phase ^ 1);
                if (lane == 0) {
                    const uint32_t fb = map_to_rank(full_bar(stage), 0);
                    if (PRE) {
                        // s*V rows of this CTA's tile (precomputed) + B_a rows [n0 + 128 rank, +128)
                        if (leader) mbar_expect_tx(full_bar(stage), 2u * 256u * RB);
                        tma_load_2d_pair(a_addr(stage), &args.tmV, fb, 0, (pr.tile + (int)rank) * 128);
                        const int rb0 = n0 + 128 * (int)rank;
                        tma_load_2d_pair(b_addr(stage), &sd->tmBk, fb, 0, rb0);
                        tma_load_2d_pair(b_addr(stage) + 64u * RB, &sd->tmBk, fb, 0, rb0 + 64);
                    } else if (BWD) {
                        // s*U rows of this CTA's tile (K-major) + A_a columns [n0 + 128 rank, +128) (MN-major)
                        if (leader) mbar_expect_tx(full_bar(stage), 2u * 256u * RB);
                        tma_load_2d_pair(a_addr(stage), &args.tmU, fb, 0, (pr.tile + (int)rank) * 128);
                        for (int i = 0; i < 2; ++i)
                            tma_load_2d_pair(b_addr(stage) + (uint32_t)i * RP * 128u, &sd->tmA, fb,
                                             n0 + 128 * (int)rank + 64 * i, 0);
                    } else {
                        // B_a rows [n0 + 128 rank, +128) x r_pad (two 64-row boxes)
                        if (leader) mbar_expect_tx(full_bar(stage), 2u * 128u * RB);
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
        // Forward LoRA items: the expand K-block of item i waits for the epilogue's s*V (sv_ready),
        // so it is DEFERRED into the main loop of item i+1 (other TMEM buffer) and issued as soon as
        // sv_ready is observed, at the latest before the ring wraps onto its stage.
        int stage = 0;
        uint32_t phase = 0;
        auto advance = [&]() {
            if (++stage == stages) { stage = 0; phase ^= 1; }
        };
        constexpr uint32_t idesc = idesc_bf16(256, 256, 0, BWD ? 1 : 0);
        uint32_t it = 0, lora_it = 0;
        int pend_stage = -1, since = 0;
        uint32_t pend_phase = 0, pend_b = 0, pend_lit = 0;
        auto issue_expand = [&](int st, uint32_t ph, uint32_t bb_, bool from_sv) {
            mbar_wait(full_bar(st), ph);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t bb = b_addr(st);
                const uint32_t aop = from_sv ? sv_addr : a_addr(st);
#pragma unroll
                for (int kk = 0; kk < RP / 16; ++kk)
                    mma2_bf16(acc_col(bb_), smem_desc(aop + 32u * kk, 16, 8u * RB, kSwR),
                              BWD ? smem_desc(bb + 2048u * kk, (uint32_t)RP * 128u, 1024, kSw128)
                                  : smem_desc(bb + 32u * kk, 16, 8u * RB, kSwR),
                              idesc, 1);
                mma2_commit_mc(empty_bar(st));
            }
            __syncwarp();
        };
        auto flush = [&](bool block) {
            if (pend_stage < 0) return;
            if (!block && since < stages - 2) {
                uint32_t ok = lane == 0 ? mbar_test(sv_ready, pend_lit & 1) : 0;
                ok = __shfl_sync(0xffffffffu, ok, 0);
                if (!ok) return;
            }
            mbar_wait(sv_ready, pend_lit & 1);
            issue_expand(pend_stage, pend_phase, pend_b, true);
            if (lane == 0) mma2_commit_mc(acc_full0 + 8 * pend_b);
            __syncwarp();
            pend_stage = -1;
        };
        for (int w = cid; w < total; w += n_clusters) {
            int pi, nt;
            decode_pair(w, args.n_pairs, args.n_ntiles, args.group_m, pi, nt);
            const DevPair pr = args.pairs[pi];
            const bool lora = pr.slot >= 0;
            const uint32_t b = it & 1, u = it >> 1;
            const uint32_t acc = acc_col(b);
            if (pend_stage >= 0 && pend_b == b) flush(true);
            mbar_wait(acc_empty0 + 8 * b, (u & 1) ^ 1);
            tc_fence_after();
            for (int kb = 0; kb < nkb; ++kb) {
                if (!BWD) flush(false);
                mbar_wait(full_bar(stage), phase);
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
                if (pend_stage >= 0) ++since;
            }
            if (lora) {
                if (BWD || PRE) {  // s*U / s*V arrives by TMA: expand right away
                    issue_expand(stage, phase, b, false);
                    advance();
                    if (lane == 0) mma2_commit_mc(acc_full0 + 8 * b);
                    __syncwarp();
                } else {
                    if (lane == 0) mma2_commit_mc(v_full);
                    __syncwarp();
                    flush(true);   // at most one deferred expand
                    pend_stage = stage;
                    pend_phase = phase;
                    pend_b = b;
                    pend_lit = lora_it;
                    since = 0;
                    advance();
                    if (!args.defer) flush(true);
                }
                ++lora_it;
            } else {
                if (!BWD && (pr.flags & kPairShort)) {
                    for (int bi = 0; bi < pr.nblk; ++bi) {
                        flush(false);
                        mbar_wait(full_bar(stage), phase);
                        tc_fence_after();
                        if (lane == 0) {
                            const uint32_t ab = a_addr(stage), bb = b_addr(stage);
#pragma unroll
                            for (int kk = 0; kk < RP / 16; ++kk)
                                mma2_bf16(acc, smem_desc(ab + 32u * kk, 16, 8u * RB, kSwR),
                                          smem_desc(bb + 32u * kk, 16, 8u * RB, kSwR), idesc, 1);
                            mma2_commit_mc(empty_bar(stage));
                        }
                        __syncwarp();
                        advance();
                        if (pend_stage >= 0) ++since;
                    }
                }
                if (lane == 0) mma2_commit_mc(acc_full0 + 8 * b);
                __syncwarp();
            }
            ++it;
        }
        flush(true);
    } else if (warp >= 4) {
        // ========================= epilogue (both CTAs, own 128 rows) =========================
        const int q = warp - 4;
        const int m = q * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const uint32_t sv_ready_l = map_to_rank(sv_ready, 0);
        const uint32_t acc_empty_l = map_to_rank(acc_empty0, 0);
        uint32_t it = 0, lora_it = 0;
        __nv_bfloat16 *Y = reinterpret_cast<__nv_bfloat16 *>(args.Y);
        for (int w = cid; w < total; w += n_clusters) {
            int pi, nt;
            decode_pair(w, args.n_pairs, args.n_ntiles, args.group_m, pi, nt);
            const DevPair pr = args.pairs[pi];
            const int n0 = nt * BNW;
            const bool lora = pr.slot >= 0;
            const int my_rows = leader ? min(pr.rows, 128) : max(pr.rows - 128, 0);
            const bool row_ok = m < my_rows;
            const int row = pr.row0 + 128 * (int)rank + m;
            const uint32_t b = it & 1, u = it >> 1;
            if (lora && !BWD && !PRE) {
                mbar_wait(v_full, lora_it & 1);
                tc_fence_after();
                uint32_t v[RP];
#pragma unroll
                for (int c = 0; c < RP; c += 16) {
                    uint32_t tmp[16];
                    tmem_ld16(acc_col(b) + BNW + lane_base + c, tmp);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; ++j) v[c + j] = tmp[j];
                }
                if (nt == 0 && row_ok && (pr.flags & kPairFT) && args.Vsave) {
                    __nv_bfloat16 *vs = reinterpret_cast<__nv_bfloat16 *>(args.Vsave) + (size_t)row * args.r;
#pragma unroll
                    for (int j = 0; j < RP; ++j)
                        if (j < args.r) vs[j] = __float2bfloat16_rn(__uint_as_float(v[j]));
                }
                const float s = pr.scale;
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
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                tc_fence_before();
                mbar_arrive_cluster(sv_ready_l);
                ++lora_it;
            }
            mbar_wait(acc_full0 + 8 * b, u & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c = 0; c < BNW / 16; ++c) {
                uint32_t r[16];
                tmem_ld16(acc_col(b) + lane_base + 16u * c, r);
                tmem_wait_ld();
                const int col = n0 + 16 * c;
                if (row_ok && col < args.N) {
                    uint4 *dst = reinterpret_cast<uint4 *>(Y + (size_t)row * args.N + col);
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

template <bool BWD, int RP, bool PRE = false>
int launch2_impl(const Gemm2Args &a, int num_sms, cudaStream_t st) {
    auto kern = smlm_gemm2_kernel<BWD, RP, PRE>;
    const size_t smem = 1024 + (size_t)a.stages * kStage2 + 128 * RP * 2 + 256;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        attr_done = true;
    }
    const int total = a.n_pairs * a.n_ntiles;
    int clusters = num_sms / 2;
    if (total < clusters) clusters = total;
    return (int)launch_pdl(kern, dim3(2 * clusters), dim3(kThreads2), smem, st, a);
}

}  // namespace

int gemm2_stages(int r_pad) {
    const size_t fixed = 1024 + (size_t)128 * r_pad * 2 + 256;
    int s = (int)((232448 - fixed) / kStage2);
    return s > 8 ? 8 : s;
}

int launch_gemm2(const Gemm2Args &a, bool bwd, int num_sms, cudaStream_t st) {
    if (a.n_pairs == 0 || a.n_ntiles == 0) return 0;
    if (!bwd && a.pre) {
        switch (a.r_pad) {
            case 16: return launch2_impl<false, 16, true>(a, num_sms, st);
            case 32: return launch2_impl<false, 32, true>(a, num_sms, st);
            case 64: return launch2_impl<false, 64, true>(a, num_sms, st);
        }
        return (int)cudaErrorInvalidValue;
    }
    switch (a.r_pad * (bwd ? -1 : 1)) {
        case 16: return launch2_impl<false, 16>(a, num_sms, st);
        case 32: return launch2_impl<false, 32>(a, num_sms, st);
        case 64: return launch2_impl<false, 64>(a, num_sms, st);
        case -16: return launch2_impl<true, 16>(a, num_sms, st);
        case -32: return launch2_impl<true, 32>(a, num_sms, st);
        case -64: return launch2_impl<true, 64>(a, num_sms, st);
    }
    return (int)cudaErrorInvalidValue;
}

}  // namespace smlm
