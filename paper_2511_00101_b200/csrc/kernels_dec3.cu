// kernels_dec3.cu -- the decode / short-row forward, HBM-bound, in ONE launch.
//
// PAPER.md P:687 (§4.2): decode throughput plateaus "indicating that the GPU memory access
// bottleneck has been hit".  A pure decode batch (<= 512 rows) is a skinny product: the cost is
// streaming W and the batch's A_u / B_u from HBM once.  One launch per call; several projections
// that share X (q/k/v, gate/up) ride in the same launch.  The grid is one wave of
// CTA pairs (clusters of 2, tcgen05 cta_group::2: M = 256 decode rows, 128 per CTA; N = 256 rows of
// the B operand, 128 staged per CTA; 6-stage TMA ring) working on two kinds of tiles:
//
//   * V tiles (the shrink, first in the grid): B = the stacked A_u of 256/r_pad adapters of the
//     batch (each by its own TMA descriptor, issued lane-parallel) -> X A_u^T for every (row,
//     adapter) pair; split K (ks_v).  After the split-K reduction the owner of each 32-column
//     chunk writes the block-diagonal bf16 slab of its adapters (s*V for the rows of the adapter,
//     zero for every other row) and V_save, then publishes on a counter.
//   * W tiles: B = 256 rows of W_p -> the base product; split K (ks).  After its base K range,
//     split s folds in the expand of every adapter u with slot(u) % ks == s as one more
//     K = r_pad block (A operand: the adapter's slab rows of this CTA; B operand: B_u rows of the
//     tile), after waiting for the slabs -- the LoRA term lands in the base accumulator.
//   * Split-K reduction in-kernel (both kinds): each CTA stores the 32-column chunks it does not
//     own as coalesced float4 rows (L2-resident), counts itself in on the tile's counter, bulk-loads
//     the peers' partials of its own chunks into the idle ring and sums them in split order
//     (deterministic, independent of the row position); W tiles store bf16 Y with TMA.
//
// Counters (pool-owned int[dec3_counter_ints()], zero at pool creation, self-resetting):
//   [0] V-tile CTAs that published their slabs, [1] CTAs departed (the last one resets
//   everything), [2 + tile] split arrivals of a tile (V tiles first, then W tiles),
//   [258] V-tile CTAs that issued their first ring of loads (the W tiles start streaming after).
// All CTAs of a launch are co-resident (grid <= one wave of pairs) -- required by the spin-waits.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "device_types.h"
#include "pdl.cuh"
#include "sm100.cuh"

namespace smlm {
using namespace sm100;

namespace {

constexpr int kT3 = 256;
constexpr uint32_t kA3 = 128 * 128;   // own 128 decode rows x 64 k
constexpr uint32_t kB3 = 128 * 128;   // own 128 W rows x 64 k
constexpr uint32_t kStage3 = kA3 + kB3;
constexpr uint32_t kYStage = 128 * 32 * 2;   // bf16 Y chunk staged for the TMA store
constexpr int kVIssuedCtr = 2 + 256;          // counter: V-tile CTAs that issued their first ring of loads

__device__ __forceinline__ void dbg_stamp(const Dec3Args &a, int k) {
    if (a.dbg) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.dbg[blockIdx.x * 16 + k] = t;
    }
}

__device__ __forceinline__ void tma_store_2d(const void *map, uint32_t ssrc, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(ssrc), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_load(uint32_t sdst, const void *gsrc, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sdst),
                 "l"(gsrc), "r"(bytes), "r"(bar)
                 : "memory");
}
struct Item3 {
    bool vtile;
    int g, s, p, ks, tile, item0;
    int n0;   // W tile: first output column; V tile: first adapter index (uidx)
};
// pair w -> item: V items (row group, projection, V tile, split) first, then W items (row group,
// W tile, split); the splits of a tile are consecutive pairs (item0 = the tile's first)
__device__ __forceinline__ Item3 dec3_item(const Dec3Args &a, int w) {
    Item3 it;
    if (w < a.n_vpairs) {
        it.vtile = true;
        it.ks = a.ks_v;
        it.s = w % a.ks_v;
        it.tile = w / a.ks_v;                      // V tile id
        const int vt = it.tile % a.n_vt, gp = it.tile / a.n_vt;
        it.p = gp % a.n_proj;
        it.g = gp / a.n_proj;
        it.n0 = vt * (256 / a.r_pad);
    } else {
        it.vtile = false;
        it.ks = a.ks;
        const int w2 = w - a.n_vpairs;
        it.s = w2 % a.ks;
        const int tw = w2 / a.ks;
        it.tile = a.n_vpairs / a.ks_v + tw;      // tile ids: V tiles, then W tiles
        it.g = tw / a.n_wt;
        const int t = tw % a.n_wt;
        it.p = 0;
        for (int p = 1; p < a.n_proj; ++p)
            if (t >= a.proj[p].nt0) it.p = p;
        it.n0 = (t - a.proj[it.p].nt0) * 256;
    }
    it.item0 = w - it.s;
    return it;
}

template <int RP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kT3, 1) smlm_dec3_kernel(const __grid_constant__ Dec3Args a,
                                                                                        const __grid_constant__ Dec3Inline inl) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    constexpr uint32_t RB = RP * 2;
    constexpr uint32_t kSwR = RB >= 128 ? kSw128 : (RB == 64 ? kSw64 : kSw32);
    constexpr int APC = 128 / RP;   // stacked adapters per CTA of a V tile
    // expand adapters per ring stage (16 KB A + 16 KB B per CTA)
    constexpr int EPS = 64 / RP;
    const int ST = a.stages;
    const uint32_t ystage = base + ST * kStage3;   // 2 x 8 KB bf16 Y staging (TMA store)
    const uint32_t bar = ystage + 2 * kYStage;
    auto full_bar = [&](int s) { return bar + 8u * s; };
    auto empty_bar = [&](int s) { return bar + 8u * (ST + s); };
    const uint32_t acc_full = bar + 16u * ST;
    const uint32_t xbar = acc_full + 8;
    const uint32_t tmem_slot = acc_full + 16;
    auto a_addr = [&](int s) { return base + s * kStage3; };
    auto b_addr = [&](int s) { return base + s * kStage3 + kA3; };

    if (threadIdx.x == 0) dbg_stamp(a, 10);   // entry (stamp 0: setup done, after the grid-dependency wait)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int cid = blockIdx.x >> 1;
    const bool active = cid < a.n_vpairs + a.n_wpairs;
    const Item3 it = dec3_item(a, active ? cid : 0);
    const Dec3Proj &P = a.proj[it.p];
    if (active && threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(xbar, 1);
        fence_mbar_init();
        tma_prefetch_desc(&a.tmX);
        tma_prefetch_desc(&P.tmW);
        tma_prefetch_desc(&P.tmY);
        if (a.n_uniq) tma_prefetch_desc(&P.tmSV);
    }
    // the batch's adapter slots and (W tiles) this split's expand adapters, staged once in shared
    // memory in parallel (parameter / global reads in serial loops cost ~0.1 us each)
    __shared__ int s_ulist[kDec3InlineSlots];
    __shared__ int s_uslot[kDec3InlineSlots];
    __shared__ int s_wcnt[kT3 / 32];
    __shared__ int s_ucount;
    if (active) {
        const int nu = a.n_uniq, ksp = it.ks, s0 = it.s;
        const bool expand = !it.vtile;
        const int u = threadIdx.x;
        int sl = -1;
        if (u < nu && u < kDec3InlineSlots) sl = inl.uslot[u];
        if (u < kDec3InlineSlots) s_uslot[u] = sl;
        const bool mine = sl >= 0 && expand && sl % ksp == s0;
        const uint32_t bal = __ballot_sync(0xffffffffu, mine);
        if (lane == 0) s_wcnt[warp] = __popc(bal);
        __syncthreads();
        int off = 0, tot = 0;
        for (int w = 0; w < kT3 / 32; ++w) {
            off += w < warp ? s_wcnt[w] : 0;
            tot += s_wcnt[w];
        }
        if (mine) s_ulist[off + __popc(bal & ((1u << lane) - 1u))] = u;
        if (threadIdx.x == 0) s_ucount = tot;
    }
    if (active && warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(256)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = active ? *reinterpret_cast<volatile uint32_t *>(base_ptr + (tmem_slot - base)) : 0u;
    // nothing in global memory is read before this point: the slot table (TMA descriptors of the
    // adapters) may be written by the stream's preceding work
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) dbg_stamp(a, 0);

    const int ks = it.ks;
    const int nkb = a.K / kBK;
    auto kb_range = [&](int s, int &kb0, int &kb1) {
        const int q = nkb / ks, rm = nkb % ks;
        kb0 = s * q + min(s, rm);
        kb1 = kb0 + q + (s < rm ? 1 : 0);
    };
    const int v_target = 2 * a.n_vpairs;   // V-tile CTAs that publish their slabs

    if (!active) {
        // idle pair (the wave is larger than the work)
    } else if (warp == 0) {
        // ========================= TMA producer (both CTAs) =========================
        int stage = 0;
        uint32_t phase = 0;
        const int xrow = it.g * 256 + 128 * (int)rank;
        const int wrow = it.n0 + 128 * (int)rank;
        int kb0, kb1;
        kb_range(it.s, kb0, kb1);
        // V tile: this CTA stacks adapters [u0, u0 + nad) of the batch; the peer holds the next APC
        const int u0 = it.n0 + APC * (int)rank;
        const int nad = it.vtile ? max(0, min(APC, a.n_uniq - u0)) : 0;
        const int nad1 = it.vtile ? max(0, min(APC, a.n_uniq - (it.n0 + APC))) : 0;
        const uint32_t bytes_pair = it.vtile ? 2u * kA3 + (uint32_t)(max(0, min(APC, a.n_uniq - it.n0)) + nad1) * RP * 128u
                                             : 2u * kStage3;
        if (it.vtile && lane < nad) {
            const void *d = &P.slots[s_uslot[u0 + lane]].tmA;
            tma_prefetch_desc(d);
        }
        if (!it.vtile && a.n_vpairs > 0) {
            // the V tiles' first ring of loads goes to the memory system before the W stream: the
            // V chain (shrink -> split-K reduction -> publish) is what the W tiles' expand waits for
            if (lane == 0)
                while (ld_acquire_gpu(a.ctr + kVIssuedCtr) < 2 * a.n_vpairs) __nanosleep(64);
            __syncwarp();
        }
        for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(empty_bar(stage), phase ^ 1);
            const uint32_t fb = map_to_rank(full_bar(stage), 0);
            if (lane == 0 && leader) mbar_expect_tx(full_bar(stage), bytes_pair);
            __syncwarp();
            // one TMA per lane: lane 31 the X rows, lanes 0.. the B operand (W rows, or the stacked
            // A_u of a V tile -- several boxes, issued in parallel)
            if (lane == 31) tma_load_2d_pair(a_addr(stage), &a.tmX, fb, kb * kBK, xrow);
            if (!it.vtile) {
                if (lane == 0) tma_load_2d_pair(b_addr(stage), &P.tmW, fb, kb * kBK, wrow);
            } else if (lane < nad) {
                tma_load_2d_pair(b_addr(stage) + (uint32_t)lane * RP * 128u, &P.slots[s_uslot[u0 + lane]].tmA, fb,
                                 kb * kBK, 0);
            }
            __syncwarp();
            if (it.vtile && lane == 0 && kb - kb0 + 1 == min(ST, kb1 - kb0)) atom_add_release_gpu(a.ctr + kVIssuedCtr, 1);
            if (++stage == ST) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) dbg_stamp(a, 1);
        if (!it.vtile && s_ucount > 0) {
            // the s*V slabs are published by the V tiles
            if (lane == 0) {
                while (ld_acquire_gpu(a.ctr) < v_target) {   // one thread per CTA: a tight spin is cheapest
                }
                fence_proxy_async_global();
                dbg_stamp(a, 2);
            }
            __syncwarp();
            // EPS adapters per ring stage (each: 128 slab rows + 128 B_u rows per CTA), issued
            // lane-parallel: a split's expand is one or two ring rounds instead of one per adapter
            for (int iu0 = 0; iu0 < s_ucount; iu0 += EPS) {
                const int na = min(EPS, s_ucount - iu0);
                mbar_wait(empty_bar(stage), phase ^ 1);
                const uint32_t fb = map_to_rank(full_bar(stage), 0);
                if (lane == 0 && leader) mbar_expect_tx(full_bar(stage), (uint32_t)na * 2u * 256u * RB);
                __syncwarp();
                if (lane < na) {
                    const int u = s_ulist[iu0 + lane];
                    const SlotDev *sd = P.slots + s_uslot[u];
                    const uint32_t off = (uint32_t)lane * 128u * RB;
                    tma_load_2d_pair(a_addr(stage) + off, &P.tmSV, fb, 0, (it.g * a.n_uniq + u) * 256 + 128 * (int)rank);
                    tma_load_2d_pair(b_addr(stage) + off, &sd->tmBk, fb, 0, wrow);
                    tma_load_2d_pair(b_addr(stage) + off + 64u * RB, &sd->tmBk, fb, 0, wrow + 64);
                }
                __syncwarp();
                if (++stage == ST) { stage = 0; phase ^= 1; }
            }
            if (lane == 0) dbg_stamp(a, 8);
        }
    } else if (warp == 1 && leader) {
        // ========================= MMA issuer (leader CTA) =========================
        int stage = 0;
        uint32_t phase = 0;
        constexpr uint32_t idesc = idesc_bf16(256, 256, 0, 0);
        int kb0, kb1;
        kb_range(it.s, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(full_bar(stage), phase);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t ab = a_addr(stage), bb = b_addr(stage);
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k)
                    mma2_bf16(tmem_base, smem_desc(ab + 32u * k, 16, 1024, kSw128),
                              smem_desc(bb + 32u * k, 16, 1024, kSw128), idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                mma2_commit_mc(empty_bar(stage));
            }
            __syncwarp();
            if (++stage == ST) { stage = 0; phase ^= 1; }
        }
        const int n_exp = it.vtile ? 0 : s_ucount;
        for (int iu0 = 0; iu0 < n_exp; iu0 += EPS) {
            const int na = min(EPS, n_exp - iu0);
            mbar_wait(full_bar(stage), phase);
            tc_fence_after();
            if (lane == 0) {
                for (int jj = 0; jj < na; ++jj) {
                    const uint32_t ab = a_addr(stage) + (uint32_t)jj * 128u * RB, bb = b_addr(stage) + (uint32_t)jj * 128u * RB;
#pragma unroll
                    for (int kk = 0; kk < RP / 16; ++kk)
                        mma2_bf16(tmem_base, smem_desc(ab + 32u * kk, 16, 8u * RB, kSwR),
                                  smem_desc(bb + 32u * kk, 16, 8u * RB, kSwR), idesc, 1u);
                }
                mma2_commit_mc(empty_bar(stage));
            }
            __syncwarp();
            if (++stage == ST) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) {
            dbg_stamp(a, 9);
            mma2_commit_mc(acc_full);
        }
        __syncwarp();
    } else if (warp == 3 && !it.vtile && s_ucount > 0) {
        // expand operands of this split: descriptors and B_u rows of the tile -> caches / L2
        for (int iu = lane; iu < s_ucount; iu += 32) {
            const int sl = s_uslot[s_ulist[iu]];
            const SlotDev *sd = P.slots + sl;
            tma_prefetch_desc(&sd->tmBk);
            const int wrow = it.n0 + 128 * (int)rank;
            if (wrow < P.out) {
                const char *bp = reinterpret_cast<const char *>(sd->B) + (size_t)wrow * sd->r * 2;
                const uint32_t bytes = (uint32_t)(min(128, P.out - wrow) * sd->r * 2);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(bp), "r"(bytes) : "memory");
            }
        }
    } else if (warp >= 4) {
        // ========================= epilogue warps (both CTAs) =========================
        const int ew = warp - 4;
        const int tid_e = threadIdx.x - 128;
        const int m = ew * 32 + lane;   // TMEM lane = decode row inside this CTA's 128
        const uint32_t lane_base = (uint32_t)(ew * 32) << 16;
        const int row0 = it.g * 256 + 128 * (int)rank;
        const int row = row0 + m;
        Dec3RowInfo ri{-1, 0.f, 0, 0};
        if (it.vtile && row < a.S) ri = inl.rows[row];
        mbar_wait(acc_full, 0);
        tc_fence_after();
        if (tid_e == 0) dbg_stamp(a, 4);
        // partial of (split s2, chunk c) of this CTA's rows: [8 q][128 m] float4 (coalesced)
        auto part = [&](int s2, int c) {
            return reinterpret_cast<float4 *>(a.kpart) +
                   ((((size_t)(it.item0 + s2) * 2 + rank) * 8 + c) * 8) * 128 + m;
        };
        // W tiles exchange their split partials in bf16 (each split accumulated in fp32 in TMEM; the
        // owner adds its own fp32 chunk to the peers' bf16 ones in split order): [4 q][128 m] uint4
        auto part_w = [&](int s2, int c) {
            return reinterpret_cast<uint4 *>(a.kpart) + ((((size_t)(it.item0 + s2) * 2 + rank) * 8 + c) * 4) * 128 + m;
        };
        constexpr uint32_t kPartW = 128u * 32u * 2u;   // bytes of one bf16 chunk partial
        if (it.vtile) {
            // ---- V tile: only each row's own-adapter columns matter, so the split-K reduction moves
            // r_pad floats per row (not the whole 256-column accumulator) ----
            const int APT = 256 / RP;
            const int ua = ri.uidx;
            const bool in_tile = ua >= it.n0 && ua < it.n0 + APT;
            const int col0 = (ua - it.n0) * RP;   // the row's adapter columns [col0, col0 + RP)
            float vp[RP];
#pragma unroll
            for (int j = 0; j < RP; ++j) vp[j] = 0.f;
            constexpr int W = RP < 32 ? RP : 32;  // columns of one adapter inside a 32-column chunk
#pragma unroll 1
            for (int c = 0; c < 8; ++c) {
                uint32_t rr[32];
                tmem_ld32(tmem_base + lane_base + 32u * c, rr);
                tmem_wait_ld();
                if (!__any_sync(0xffffffffu, in_tile && col0 < 32 * c + 32 && col0 + RP > 32 * c)) continue;
#pragma unroll
                for (int h = 0; h < 32 / W; ++h) {
                    const int col = 32 * c + h * W;
                    if (in_tile && col >= col0 && col < col0 + RP) {
                        const int j0 = col - col0;   // 0, or 32 for r_pad = 64
#pragma unroll
                        for (int e = 0; e < W; ++e) {
                            if (j0 == 0) vp[e] = __uint_as_float(rr[h * W + e]);
                            else vp[(RP > 32 ? 32 : 0) + e] = __uint_as_float(rr[h * W + e]);
                        }
                    }
                }
            }
            // compact partial of this split: [item][rank][128 rows][RP] fp32
            float *vpart = a.kpart + ((size_t)it.item0 * 2 + rank) * 128 * RP;   // split s2 at + s2 * 2 * 128 * RP
            if (ks > 1) {
                if (in_tile) {
                    float4 *dst = reinterpret_cast<float4 *>(vpart + ((size_t)it.s * 2 * 128 + m) * RP);
#pragma unroll
                    for (int q = 0; q < RP / 4; ++q) __stcg(dst + q, make_float4(vp[4 * q], vp[4 * q + 1], vp[4 * q + 2], vp[4 * q + 3]));
                }
                // the CTA barrier orders every thread's partial stores before thread 0's gpu-scope
                // release (cumulative), as in a split-K semaphore: no per-thread fence
                named_bar_sync(1, 128);
                if (tid_e == 0) {
                    dbg_stamp(a, 3);
                    int *arrive = a.ctr + 2 + it.tile;
                    atom_add_release_gpu(arrive, 1);
                    while (ld_acquire_gpu(arrive) < 2 * ks) {
                    }
                    dbg_stamp(a, 5);
                }
                named_bar_sync(1, 128);
            }
            // rows m with m % ks == s: sum the splits in order, write the row's slab entries for every
            // adapter of the tile (s*V for its own adapter, zero otherwise) and V_save
            if (m % ks == it.s && row < a.S) {
                if (in_tile && ks > 1) {
                    // all splits' partials of a 16-column slice in flight at once, summed in split order
#pragma unroll
                    for (int j0 = 0; j0 < RP; j0 += 16)
#pragma unroll 1
                    for (int sb = 0; sb < ks; sb += 8) {   // 8 splits in flight, then the next 8
                        float t[8][16];
#pragma unroll
                        for (int s2 = 0; s2 < 8; ++s2) {
                            if (sb + s2 < ks) {
                                const float4 *src = reinterpret_cast<const float4 *>(vpart + ((size_t)(sb + s2) * 2 * 128 + m) * RP + j0);
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    const float4 f = __ldcg(src + q);
                                    t[s2][4 * q] = f.x;
                                    t[s2][4 * q + 1] = f.y;
                                    t[s2][4 * q + 2] = f.z;
                                    t[s2][4 * q + 3] = f.w;
                                }
                            }
                        }
#pragma unroll
                        for (int s2 = 0; s2 < 8; ++s2)
                            if (sb + s2 < ks)
#pragma unroll
                                for (int j = 0; j < 16; ++j) vp[j0 + j] = sb + s2 == 0 ? t[0][j] : vp[j0 + j] + t[s2][j];
                    }
                }
                __nv_bfloat16 *sv = reinterpret_cast<__nv_bfloat16 *>(P.sv);
                for (int ad = 0; ad < APT; ++ad) {
                    const int uu = it.n0 + ad;
                    if (uu >= a.n_uniq) break;
                    uint4 *dst = reinterpret_cast<uint4 *>(sv + ((size_t)(it.g * a.n_uniq + uu) * 256 + (row & 255)) * RP);
                    const bool own = in_tile && uu == ua;
#pragma unroll
                    for (int q = 0; q < RP / 8; ++q) {
                        uint4 pk = make_uint4(0, 0, 0, 0);
                        if (own) {
                            const float s = ri.scale;
                            pk.x = pack_bf16x2(s * vp[8 * q + 0], s * vp[8 * q + 1]);
                            pk.y = pack_bf16x2(s * vp[8 * q + 2], s * vp[8 * q + 3]);
                            pk.z = pack_bf16x2(s * vp[8 * q + 4], s * vp[8 * q + 5]);
                            pk.w = pack_bf16x2(s * vp[8 * q + 6], s * vp[8 * q + 7]);
                        }
                        dst[q] = pk;
                    }
                }
                __nv_bfloat16 *vsave = reinterpret_cast<__nv_bfloat16 *>(P.Vsave);
                if (in_tile && ri.ft && vsave) {
#pragma unroll
                    for (int j = 0; j < RP; ++j)
                        if (j < a.r) vsave[(size_t)row * a.r + j] = __float2bfloat16_rn(vp[j]);
                }
            }
            // publish: the slabs are read by TMA (async proxy) in other CTAs
            fence_proxy_async_global();
            named_bar_sync(1, 128);
            if (tid_e == 0) {
                atom_add_release_gpu(a.ctr, 1);
                dbg_stamp(a, 6);
                dbg_stamp(a, 15);   // marks a V-tile CTA for the timeline scripts
            }
        } else {
            if (ks > 1) {
    #pragma unroll 1
                for (int c = 0; c < 8; ++c) {
                    if (c % ks == it.s) continue;
                    uint32_t rr[32];
                    tmem_ld32(tmem_base + lane_base + 32u * c, rr);
                    tmem_wait_ld();
                    uint4 *dst = part_w(it.s, c);
    #pragma unroll
                    for (int q = 0; q < 4; ++q)
                        __stcg(dst + q * 128, make_uint4(pack_bf16x2(__uint_as_float(rr[8 * q]), __uint_as_float(rr[8 * q + 1])),
                                                         pack_bf16x2(__uint_as_float(rr[8 * q + 2]), __uint_as_float(rr[8 * q + 3])),
                                                         pack_bf16x2(__uint_as_float(rr[8 * q + 4]), __uint_as_float(rr[8 * q + 5])),
                                                         pack_bf16x2(__uint_as_float(rr[8 * q + 6]), __uint_as_float(rr[8 * q + 7]))));
                }
                named_bar_sync(1, 128);
                if (tid_e == 0) {
                    dbg_stamp(a, 3);
                    int *arrive = a.ctr + 2 + it.tile;
                    atom_add_release_gpu(arrive, 1);
                    while (ld_acquire_gpu(arrive) < 2 * ks) {
                    }
                    dbg_stamp(a, 5);
                }
                named_bar_sync(1, 128);
                // peers' partials of the owned chunks -> the (now idle) ring with one mbarrier
                if (tid_e == 0) {
                    fence_proxy_async_global();
                    const int n_own = (8 - it.s + ks - 1) / ks;
                    mbar_expect_tx(xbar, (uint32_t)(n_own * (ks - 1)) * kPartW);
                    int slot = 0;
                    for (int c = it.s; c < 8; c += ks)
                        for (int s2 = 0; s2 < ks; ++s2) {
                            if (s2 == it.s) continue;
                            bulk_load(base + (uint32_t)slot * kPartW, part_w(s2, c) - m, kPartW, xbar);
                            ++slot;
                        }
                }
                mbar_wait(xbar, 0);
                if (tid_e == 0) dbg_stamp(a, 7);
            }
            // own chunks: sum the splits in order, bf16 into the idle ring above the loaded partials
            // (<= 7 x 16 KB), then one TMA store per chunk (rows >= S / columns >= out clipped)
            const uint32_t ybase = base + 7u * 16384u;
#pragma unroll 1
            for (int c = it.s, oi = 0; c < 8; c += ks, ++oi) {
                float v[32];
                {
                    uint32_t rr[32];
                    tmem_ld32(tmem_base + lane_base + 32u * c, rr);
                    tmem_wait_ld();
#pragma unroll 1
                    for (int s2 = 0, j = 0; s2 < ks; ++s2) {
                        float t[32];
                        if (s2 == it.s) {
#pragma unroll
                            for (int e = 0; e < 32; ++e) t[e] = __uint_as_float(rr[e]);
                        } else {
                            const uint4 *src = reinterpret_cast<const uint4 *>(base_ptr + (size_t)(oi * (ks - 1) + j) * kPartW) + m;
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const uint4 f = src[q * 128];
                                const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&f);
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const float2 x = __bfloat1622float2(h[i]);
                                    t[8 * q + 2 * i] = x.x;
                                    t[8 * q + 2 * i + 1] = x.y;
                                }
                            }
                            ++j;
                        }
#pragma unroll
                        for (int e = 0; e < 32; ++e) v[e] = s2 == 0 ? t[e] : v[e] + t[e];
                    }
                }
                uint4 *ys = reinterpret_cast<uint4 *>(base_ptr + (ybase - base) + (size_t)oi * kYStage);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint4 pk;
                    pk.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
                    pk.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
                    pk.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
                    pk.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
                    ys[m * 4 + q] = pk;
                }
            }
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (tid_e == 0) {
                for (int c = it.s, oi = 0; c < 8; c += ks, ++oi)
                    tma_store_2d(&P.tmY, ybase + (uint32_t)oi * kYStage, it.n0 + 32 * c, row0);
                bulk_commit();
            }
            if (tid_e == 0) {
                bulk_wait_all();
                dbg_stamp(a, 6);
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (active && warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256) : "memory");
    }
    // the last CTA to leave resets the counters for the next launch
    if (threadIdx.x == 0) {
        __threadfence();
        if (atom_add_acq_rel_gpu(a.ctr + 1, 1) == (int)gridDim.x - 1) {
            a.ctr[0] = 0;
            a.ctr[1] = 0;
            a.ctr[kVIssuedCtr] = 0;
            const int tiles = a.n_vpairs / a.ks_v + a.n_groups * a.n_wt;
            for (int t = 0; t < tiles; ++t) a.ctr[2 + t] = 0;
        }
    }
}

static_assert(sizeof(Dec3Args) + sizeof(Dec3Inline) <= 32764, "kernel parameters exceed 32 KB");

constexpr size_t dec3_smem() { return 1024 + (size_t)6 * kStage3 + 2 * kYStage + 256; }

template <int RP>
cudaError_t dec3_attr() {
    static cudaError_t done = cudaErrorNotReady;
    if (done != cudaSuccess)
        done = cudaFuncSetAttribute(smlm_dec3_kernel<RP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dec3_smem());
    return done;
}

// The CTAs of one launch spin-wait on each other (V publish, split-K arrival), so they must all be
// resident at once: the grid is capped by the clusters that fit the device at one CTA per SM (on
// an otherwise idle GPU every CTA is placed; a kernel of another stream only delays the late
// ones).  Two spin-waiting grids that each hold part of the GPU could wait on each other: with
// the pool option SMLM_OPT_DEC_COOPERATIVE the launch is cooperative (the whole grid is
// co-scheduled), for callers that issue decode calls on several streams at once (~2 us per
// launch, measured).
template <int RP>
int dec3_max_clusters_impl() {
    static int cached = -1;
    if (cached >= 0) return cached;
    if (dec3_attr<RP>() != cudaSuccess) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * kDec3MaxPairs);
    cfg.blockDim = dim3(kT3);
    cfg.dynamicSmemBytes = dec3_smem();
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, smlm_dec3_kernel<RP>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cached = n;
    return n;
}

template <int RP>
int launch_dec3_impl(const Dec3Args &a, const Dec3Inline &in, int clusters, cudaStream_t st) {
    cudaError_t e = dec3_attr<RP>();
    if (e != cudaSuccess) return (int)e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(kT3);
    cfg.dynamicSmemBytes = dec3_smem();
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = a.cooperative ? 2 : 1;
    return (int)cudaLaunchKernelEx(&cfg, smlm_dec3_kernel<RP>, a, in);
}

}  // namespace

int dec3_stages() { return 6; }

int dec3_max_clusters(int r_pad) {
    switch (r_pad) {
        case 16: return dec3_max_clusters_impl<16>();
        case 32: return dec3_max_clusters_impl<32>();
        case 64: return dec3_max_clusters_impl<64>();
    }
    return 0;
}

int launch_dec3(const Dec3Args &a, const Dec3Inline &in, int clusters, cudaStream_t st) {
    switch (a.r_pad) {
        case 16: return launch_dec3_impl<16>(a, in, clusters, st);
        case 32: return launch_dec3_impl<32>(a, in, clusters, st);
        case 64: return launch_dec3_impl<64>(a, in, clusters, st);
    }
    return (int)cudaErrorInvalidValue;
}

}  // namespace smlm
