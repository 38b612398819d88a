// kernels_dec3.cu -- the decode / short-row forward, HBM-bound, in ONE launch.
//
// PAPER.md P:687 (§4.2): decode throughput plateaus "indicating that the GPU memory access
// bottleneck has been hit".  A pure decode batch (<= 512 rows) is a skinny product: the cost is
// streaming W and the batch's A_u / B_u from HBM once.  One launch per call; several projections
// that share X (q/k/v, gate/up) ride in the same launch.  The grid is one wave of
// CTA pairs (clusters of 2) with two roles:
//
//   * W pairs (tcgen05 cta_group::2): item = (row group of 256 decode rows, W tile of 256 output
//     columns, K split).  M = 256 decode rows (128 per CTA), N = 256 W rows (128 staged per CTA):
//     per SM 16 KB of X and 16 KB of W per 64-K block, 6-stage TMA ring.  After its base K range,
//     split s folds in the expand of every adapter u with slot(u) % ksplit == s as one more
//     K = r_pad block: A operand = the adapter's block-diagonal s*V slab (rows of other adapters
//     are zero), B operand = B_u rows of the tile -- the LoRA term lands in the same fp32
//     accumulator as the base product.  Split-K reduction in-kernel: each CTA stores the 32-column
//     chunks it does not own (coalesced float4 rows, L2-resident), and once all 2*ksplit CTAs of
//     the tile have arrived, sums its own chunks in split order (deterministic, independent of the
//     row position) and stores bf16 Y with TMA.
//   * Shrink pairs (the rest of the wave, all 8 warps, SIMT): V = A_u x for <= 8 rows of one
//     adapter per item; the two CTAs of the pair take the two halves of K (128-bit granules of
//     A_u and x per lane, lane partials, a 31-shuffle transpose-reduce, warps combined in fixed
//     order, the peer half added through distributed shared memory), then write the adapter's
//     block-diagonal bf16 slab (s*V rows, zeros elsewhere) and V_save.  W pairs wait for the slabs
//     only before their expand blocks, i.e. after their own main loop.
//
// Counters (pool-owned int[dec3_counter_ints()], zero at pool creation, self-resetting):
//   [0] shrink items published, [1] CTAs departed (the last one resets everything),
//   [2 + tile] split arrivals of a W tile.
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
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_load(uint32_t sdst, const void *gsrc, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sdst),
                 "l"(gsrc), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// v[0..31] per lane -> lane l returns the warp sum of v[l] (31 shuffles)
__device__ __forceinline__ float warp_transpose_reduce32(float (&v)[32], int lane) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int q = 0; q < off; ++q) {
            const float send = up ? v[q] : v[q + off];
            const float keep = up ? v[q + off] : v[q];
            v[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return v[0];
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4 &u, float *f) {
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

struct Item3 {
    int g, s, p, tile, n0;
};
// W item w -> (tile = w / ks, split = w % ks); tile -> (row group, projection, n-tile)
__device__ __forceinline__ Item3 dec3_item(const Dec3Args &a, int w) {
    Item3 it;
    it.s = w % a.ks;
    it.tile = w / a.ks;
    it.g = it.tile / a.n_wt;
    const int t = it.tile % a.n_wt;
    it.p = 0;
    for (int p = 1; p < a.n_proj; ++p)
        if (t >= a.proj[p].nt0) it.p = p;
    it.n0 = (t - a.proj[it.p].nt0) * 256;
    return it;
}

// ------------------------------------------------------------------------------------------
// shrink pair: items (projection, adapter, <= 8 rows); CTA `rank` takes every other 128-bit granule
// of K.  The pair's items are staged in shared memory first (no dependent global loads later).
// ------------------------------------------------------------------------------------------
// shared-memory layout of a shrink CTA (inside the pipeline ring, which shrink pairs do not use)
template <int RP, int NW, int MI>
struct ShrinkSmem {
    static constexpr uint32_t red = 0;                                  // [NW warps][8 rows][RP] fp32
    static constexpr uint32_t own = red + NW * 8 * RP * 4;             // [8 rows][RP] this CTA's K half
    static constexpr uint32_t items = own + 8 * RP * 4;                // [MI] Dec3SItem
    static constexpr uint32_t rx = items + MI * sizeof(Dec3SItem);     // [MI][8][RP] peer halves
    static constexpr uint32_t bars = rx + MI * 8 * RP * 4;             // [MI] mbarriers
    static constexpr uint32_t end = (bars + MI * 8 + 1023u) & ~1023u;
};
// a shrink CTA runs two independent 4-warp workers (warps 0-3, 4-7) so that one worker's loads
// overlap the other's FMAs; each worker stages at most kShrMI items
constexpr int kShrMI = 32;

__device__ __forceinline__ void mbar_arrive_remote_release(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}

// ------------------------------------------------------------------------------------------
// shrink pair: items (projection, adapter, <= 8 rows); CTA `rank` takes every other 128-bit
// granule of K.  Items are staged in shared memory first; CTA 1 pushes its K half of every item
// into CTA 0's shared memory (one slot and one mbarrier per item, no cluster-wide barrier).
// ------------------------------------------------------------------------------------------
template <int RP, int NW, int MI>
__device__ __forceinline__ void dec3_shrink_worker(const Dec3Args &a, const Dec3Inline &inl, uint8_t *smem,
                                                   uint32_t smem_s, uint32_t rank, int sp, int n_sp, int tid,
                                                   int bar_id) {
    using L = ShrinkSmem<RP, NW, MI>;
    constexpr int NT = NW * 32;
    constexpr int JG = 8;   // A rows per pass (acc 8x8 + x 8x8 + A 8 granules in registers)
    const int warp = tid >> 5, lane = tid & 31;
    auto bar = [&]() { named_bar_sync(bar_id, NT); };
    const __nv_bfloat16 *X = reinterpret_cast<const __nv_bfloat16 *>(a.X);
    const int K = a.K, r = a.r, n_groups = a.n_groups, n_uniq = a.n_uniq, n_si = a.n_sitems;
    float *red = reinterpret_cast<float *>(smem + L::red);
    float *own = reinterpret_cast<float *>(smem + L::own);
    Dec3SItem *its = reinterpret_cast<Dec3SItem *>(smem + L::items);
    const int n_mine = (a.flags & 8) ? 0 : (sp < n_si ? min((n_si - sp + n_sp - 1) / n_sp, MI) : 0);
    {
        constexpr int W4 = sizeof(Dec3SItem) / 16;
        uint4 *dst = reinterpret_cast<uint4 *>(its);
        for (int e = tid; e < n_mine * W4; e += NT) {
            const int item = sp + (e / W4) * n_sp, w4 = e % W4;
            dst[e] = a.inl ? reinterpret_cast<const uint4 *>(&inl.items[item])[w4]
                           : __ldg(reinterpret_cast<const uint4 *>(a.sitems + item) + w4);
        }
    }
    bar();
    if (tid == 0 && sp == 0) dbg_stamp(a, 10);
    const int ngr = K / 8;                                     // 128-bit granules of a row
    const int gl = (int)rank * NT + tid;              // this lane's first granule
    for (int ii0 = 0; ii0 < n_mine; ++ii0) {
        const Dec3SItem &si = its[ii0];
        const __nv_bfloat16 *A = reinterpret_cast<const __nv_bfloat16 *>(si.A);
        const int n = si.n;
        int rows[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) rows[i] = si.rows[i];
        // one granule per lane per 512-lane sweep of K; A rows in groups of 8, the next group's
        // loads in flight while the current group is multiplied (one HBM round trip for r <= 16)
#pragma unroll 1
        for (int sw = 0; sw < ngr; sw += 2 * NT) {   // every lane takes part (shuffles), idle lanes load zeros
            const int gr = sw + gl;
            const bool gok = gr < ngr;
            float xf[8][8];
            {
                uint4 xa[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    xa[i] = (i < n && gok) ? __ldg(reinterpret_cast<const uint4 *>(X + (size_t)rows[i] * K) + gr)
                                           : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int i = 0; i < 8; ++i) bf16x8_to_f32(xa[i], xf[i]);
            }
            auto load_group = [&](int j0, uint4 (&aa)[JG]) {
#pragma unroll
                for (int j = 0; j < JG; ++j)
                    aa[j] = (j0 + j < r && gok) ? __ldg(reinterpret_cast<const uint4 *>(A + (size_t)(j0 + j) * K) + gr)
                                                : make_uint4(0, 0, 0, 0);
            };
            uint4 aa[JG], an[JG];
            load_group(0, aa);
            if (JG < r) load_group(JG, an);
#pragma unroll 1
            for (int j0 = 0; j0 < RP && j0 < r; j0 += JG) {
                float acc[8][JG];
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < JG; ++j) acc[i][j] = 0.f;
#pragma unroll
                for (int j = 0; j < JG; ++j) {
                    float af[8];
                    bf16x8_to_f32(aa[j], af);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
#pragma unroll
                        for (int e = 0; e < 8; ++e) acc[i][j] = fmaf(af[e], xf[i][e], acc[i][j]);
                }
#pragma unroll
                for (int j = 0; j < JG; ++j) aa[j] = an[j];
                if (j0 + 2 * JG < r) load_group(j0 + 2 * JG, an);
                // lanes -> one value each (transpose-reduce); the sweep's partials accumulate in red
#pragma unroll
                for (int h = 0; h < JG / 4; ++h) {
                    float v[32];
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                        for (int i = 0; i < 8; ++i) v[jj * 8 + i] = acc[i][4 * h + jj];
                    const float s = warp_transpose_reduce32(v, lane);
                    float *dst = &red[(warp * 8 + (lane & 7)) * RP + j0 + 4 * h + (lane >> 3)];
                    *dst = sw == 0 ? s : *dst + s;
                }
            }
        }
        if (tid == 0 && ii0 == 0) dbg_stamp(a, 11);
        bar();
        // warps in fixed order -> this CTA's K half; CTA 1 pushes it into CTA 0's slot of this item
        const uint32_t rx_s = smem_s + L::rx + (uint32_t)ii0 * 8 * RP * 4;
        const uint32_t bar_s = smem_s + L::bars + (uint32_t)ii0 * 8;
        if (rank == 1) {
            const uint32_t rx_peer = map_to_rank(rx_s, 0);
            for (int e = tid; e < 8 * RP; e += NT) {
                const int ii = e / RP, jj = e % RP;
                float t = 0.f;
                if (jj < r)
                    for (int w = 0; w < NW; ++w) t += red[(w * 8 + ii) * RP + jj];
                st_cluster_f32(rx_peer + (uint32_t)e * 4u, t);
            }
            mbar_arrive_remote_release(map_to_rank(bar_s, 0));   // every thread: its stores are released
        } else {
            for (int e = tid; e < 8 * RP; e += NT) {
                const int ii = e / RP, jj = e % RP;
                float t = 0.f;
                if (jj < r)
                    for (int w = 0; w < NW; ++w) t += red[(w * 8 + ii) * RP + jj];
                own[e] = t;
            }
            mbar_wait_acq_cluster(bar_s, 0);
            bar();
            if (tid == 0 && ii0 == 0) dbg_stamp(a, 13);
            const Dec3Proj &P = a.proj[si.p];
            __nv_bfloat16 *sv = reinterpret_cast<__nv_bfloat16 *>(P.sv);
            __nv_bfloat16 *vsave = reinterpret_cast<__nv_bfloat16 *>(P.Vsave);
            const float *rx = reinterpret_cast<const float *>(smem + L::rx + (size_t)ii0 * 8 * RP * 4);
            if (si.zero_fill) {
                // the adapter's slab rows of every other batch row (and past S) are zero
                for (int e = tid; e < n_groups * 256; e += NT) {
                    if ((si.mask[e >> 5] >> (e & 31)) & 1u) continue;
                    uint4 *z = reinterpret_cast<uint4 *>(sv + ((size_t)((e >> 8) * n_uniq + si.uidx) * 256 + (e & 255)) * RP);
#pragma unroll
                    for (int q = 0; q < RP / 8; ++q) z[q] = make_uint4(0, 0, 0, 0);
                }
            }
            for (int e = tid; e < 8 * RP; e += NT) {
                const int ii = e / RP, jj = e % RP;
                if (ii >= n) continue;
                const float v = own[e] + rx[e];   // K half 0 + K half 1 (fixed order)
                const int row = si.rows[ii];
                sv[((size_t)((row >> 8) * n_uniq + si.uidx) * 256 + (row & 255)) * RP + jj] =
                    __float2bfloat16_rn(si.scale[ii] * v);
                if (((si.ft_mask >> ii) & 1) && vsave && jj < r)
                    vsave[(size_t)row * r + jj] = __float2bfloat16_rn(v);
            }
        }
        if (tid == 0 && ii0 == 0) dbg_stamp(a, 14);
        bar();   // red / own reusable
    }
    // publish (slabs are read by TMA in other CTAs: generic -> async proxy)
    const int done = (a.flags & 8) ? (sp < n_si ? (n_si - sp + n_sp - 1) / n_sp : 0) : n_mine;
    if (rank == 0 && done) {
        fence_proxy_async_global();
        __threadfence();
        bar();
        if (tid == 0) atom_add_release_gpu(a.ctr, done);
    }
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

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int cid = blockIdx.x >> 1;
    const int n_clusters = gridDim.x >> 1;
    const bool wpair = cid < a.n_wpairs;
    if (wpair && threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(xbar, 1);
        fence_mbar_init();
        tma_prefetch_desc(&a.tmX);
        for (int p = 0; p < a.n_proj; ++p) {
            tma_prefetch_desc(&a.proj[p].tmW);
            tma_prefetch_desc(&a.proj[p].tmY);
            if (a.n_uniq) tma_prefetch_desc(&a.proj[p].tmSV);
        }
    }
    // this split's expand adapters (uslot index), in ascending order, staged once in shared memory:
    // the producer / MMA loops then never touch parameter or global memory per adapter
    __shared__ int s_ulist[kDec3InlineSlots];
    __shared__ int s_uslot[kDec3InlineSlots];
    __shared__ int s_wcnt[kT3 / 32];
    __shared__ int s_ucount;
    if (wpair) {
        // parallel: every thread one adapter (param / global reads in a serial loop cost ~0.1 us each)
        const int nu = a.n_uniq, ksp = a.ks, s0 = cid % ksp;
        const bool expand = !(a.flags & 4);
        const int u = threadIdx.x;
        int sl = -1;
        if (u < nu && u < kDec3InlineSlots) sl = (a.flags & 64) ? u : (a.inl ? inl.uslot[u] : a.uslot[u]);
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
    using SL = ShrinkSmem<RP, 4, kShrMI>;
    if (!wpair && rank == 0 && threadIdx.x == 0) {
        // per-item hand-off barriers of both workers (CTA 1's 128 worker threads arrive remotely)
        for (int wk = 0; wk < 2; ++wk)
            for (int i = 0; i < kShrMI; ++i) mbar_init(base + wk * SL::end + SL::bars + 8u * i, 128);
        fence_mbar_init();
    }
    if (wpair && warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot), "r"(256)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = wpair ? *reinterpret_cast<volatile uint32_t *>(base_ptr + (tmem_slot - base)) : 0u;
    pdl_wait();
    pdl_trigger();
    if (threadIdx.x == 0) dbg_stamp(a, 0);

    if (!wpair) {
        // ========================= shrink pair =========================
        const int wk = warp >> 2;   // worker 0: warps 0-3, worker 1: warps 4-7
        dec3_shrink_worker<RP, 4, kShrMI>(a, inl, base_ptr + wk * SL::end, base + wk * SL::end, rank,
                                          2 * (cid - a.n_wpairs) + wk, 2 * (n_clusters - a.n_wpairs),
                                          threadIdx.x & 127, 2 + wk);
        if (threadIdx.x == 0) dbg_stamp(a, 1);
    } else {
        const int ks = a.ks;
        const int nkb = a.K / kBK;
        // split s owns k-blocks kb_of(i), i in [0, cnt): a contiguous range, or (flag 16, measurement)
        // interleaved s, s + ks, ... so the splits of a tile read neighbouring 128-byte pieces of W rows
        const bool kil = (a.flags & 16) != 0;
        auto kb_range = [&](int s, int &kb0, int &kb1) {
            if (kil) {
                kb0 = 0;
                kb1 = (nkb - s + ks - 1) / ks;
                return;
            }
            const int q = nkb / ks, rm = nkb % ks;
            kb0 = s * q + min(s, rm);
            kb1 = kb0 + q + (s < rm ? 1 : 0);
        };
        auto kb_of = [&](int s, int i) { return kil ? s + i * ks : i; };
        const Item3 it = dec3_item(a, cid);   // one W item per pair
        const Dec3Proj &P = a.proj[it.p];
        if (warp == 0) {
            // ========================= TMA producer (both CTAs) =========================
            int stage = 0;
            uint32_t phase = 0;
            const int xrow = it.g * 256 + 128 * (int)rank;
            const int wrow = it.n0 + 128 * (int)rank;
            int kb0, kb1;
            kb_range(it.s, kb0, kb1);
            // flag 256 (measurement): the W stream starts once the shrink has published, so the shrink's
            // A_u / x reads do not queue behind ~20 MB of W requests in HBM
            if ((a.flags & 256) && a.n_uniq > 0) {
                if (lane == 0)
                    while (ld_acquire_gpu(a.ctr) < a.n_sitems) __nanosleep(64);
                __syncwarp();
            }
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(empty_bar(stage), phase ^ 1);
                if (lane == 0) {
                    const uint32_t fb = map_to_rank(full_bar(stage), 0);
                    if (leader) mbar_expect_tx(full_bar(stage), 2u * kStage3);
                    const int kc = kb_of(it.s, kb) * kBK;
                    tma_load_2d_pair(a_addr(stage), &a.tmX, fb, kc, xrow);
                    tma_load_2d_pair(b_addr(stage), &P.tmW, fb, kc, wrow);
                }
                __syncwarp();
                if (++stage == ST) { stage = 0; phase ^= 1; }
            }
            if (lane == 0) dbg_stamp(a, 1);
            if (a.n_uniq > 0) {
                // the s*V slabs are published by the shrink pairs
                if (lane == 0) {
                    while (ld_acquire_gpu(a.ctr) < a.n_sitems) __nanosleep(64);
                    fence_proxy_async_global();
                    dbg_stamp(a, 2);
                }
                __syncwarp();
                for (int iu = 0; iu < s_ucount; ++iu) {
                    const int u = s_ulist[iu];
                    const int sl = s_uslot[u];
                    mbar_wait(empty_bar(stage), phase ^ 1);
                    if (lane == 0) {
                        const uint32_t fb = map_to_rank(full_bar(stage), 0);
                        if (leader) mbar_expect_tx(full_bar(stage), (a.flags & 2) ? 256u * RB : 2u * 256u * RB);
                        tma_load_2d_pair(a_addr(stage), &P.tmSV, fb, 0, (it.g * a.n_uniq + u) * 256 + 128 * (int)rank);
                        const SlotDev *sd = P.slots + sl;
                        if (!(a.flags & 2)) {
                            tma_load_2d_pair(b_addr(stage), &sd->tmBk, fb, 0, wrow);
                            tma_load_2d_pair(b_addr(stage) + 64u * RB, &sd->tmBk, fb, 0, wrow + 64);
                        }
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
                if (lane == 0 && ((kb - kb0) & 3) == 0 && (kb - kb0) < 24) dbg_stamp(a, 10 + (kb - kb0) / 4);
                if (lane == 0) {
                    const uint32_t ab = a_addr(stage), bb = b_addr(stage);
                    if (!(a.flags & 32) || kb == kb0) {
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k)
                            mma2_bf16(tmem_base, smem_desc(ab + 32u * k, 16, 1024, kSw128),
                                      smem_desc(bb + 32u * k, 16, 1024, kSw128), idesc, (kb > kb0 || k > 0) ? 1u : 0u);
                    }
                    mma2_commit_mc(empty_bar(stage));
                }
                __syncwarp();
                if (++stage == ST) { stage = 0; phase ^= 1; }
            }
            for (int iu = 0; iu < s_ucount; ++iu) {
                mbar_wait(full_bar(stage), phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t ab = a_addr(stage), bb = b_addr(stage);
#pragma unroll
                    for (int kk = 0; kk < RP / 16; ++kk)
                        mma2_bf16(tmem_base, smem_desc(ab + 32u * kk, 16, 8u * RB, kSwR),
                                  smem_desc(bb + 32u * kk, 16, 8u * RB, kSwR), idesc, 1u);
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
        } else if (warp == 3 && a.n_uniq > 0) {
            // expand operands of this split: descriptors and B_u rows of the tile -> caches / L2
            for (int iu = lane; iu < s_ucount; iu += 32) {
                const int sl = s_uslot[s_ulist[iu]];
                const SlotDev *sd = P.slots + sl;
                tma_prefetch_desc(&sd->tmBk);
                const int wrow = it.n0 + 128 * (int)rank;
                if (wrow < P.out) {
                    const char *bp = reinterpret_cast<const char *>(sd->B) + (size_t)wrow * a.r * 2;
                    const uint32_t bytes = (uint32_t)(min(128, P.out - wrow) * a.r * 2);
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
            mbar_wait(acc_full, 0);
            tc_fence_after();
            if (tid_e == 0) dbg_stamp(a, 4);
            // partial of (split s2, chunk c) of this CTA's rows: [8 q][128 m] float4 (coalesced)
            auto part = [&](int s2, int c) {
                return reinterpret_cast<float4 *>(a.kpart) +
                       ((((size_t)(it.tile * ks + s2) * 2 + rank) * 8 + c) * 8) * 128 + m;
            };
            if (ks > 1) {
#pragma unroll 1
                for (int c = 0; c < 8; ++c) {
                    if (c % ks == it.s) continue;
                    uint32_t rr[32];
                    tmem_ld32(tmem_base + lane_base + 32u * c, rr);
                    tmem_wait_ld();
                    float4 *dst = part(it.s, c);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        __stcg(dst + q * 128, make_float4(__uint_as_float(rr[4 * q]), __uint_as_float(rr[4 * q + 1]),
                                                          __uint_as_float(rr[4 * q + 2]), __uint_as_float(rr[4 * q + 3])));
                }
                __threadfence();
                named_bar_sync(1, 128);
                if (tid_e == 0) {
                    dbg_stamp(a, 3);
                    int *arrive = a.ctr + 2 + it.tile;
                    atom_add_release_gpu(arrive, 1);
                    while (ld_acquire_gpu(arrive) < 2 * ks) __nanosleep(32);
                    dbg_stamp(a, 5);
                }
                named_bar_sync(1, 128);
            }
            // peers' partials of the owned chunks -> the (now idle) ring with one mbarrier
            const int n_own = (8 - it.s + ks - 1) / ks;
            if (ks > 1) {
                if (tid_e == 0) {
                    fence_proxy_async_global();
                    mbar_expect_tx(xbar, (uint32_t)(n_own * (ks - 1)) * 16384u);
                    int slot = 0;
                    for (int c = it.s; c < 8; c += ks)
                        for (int s2 = 0; s2 < ks; ++s2) {
                            if (s2 == it.s) continue;
                            bulk_load(base + (uint32_t)slot * 16384u, part(s2, c) - m, 16384u, xbar);
                            ++slot;
                        }
                }
                mbar_wait(xbar, 0);
                if (tid_e == 0) dbg_stamp(a, 7);
            }
            int ybuf = 0;
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
                            const float4 *src = reinterpret_cast<const float4 *>(base_ptr + (size_t)(oi * (ks - 1) + j) * 16384u) + m;
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const float4 f = src[q * 128];
                                t[4 * q] = f.x;
                                t[4 * q + 1] = f.y;
                                t[4 * q + 2] = f.z;
                                t[4 * q + 3] = f.w;
                            }
                            ++j;
                        }
#pragma unroll
                        for (int e = 0; e < 32; ++e) v[e] = s2 == 0 ? t[e] : v[e] + t[e];
                    }
                }
                // bf16 chunk -> staging -> TMA store (rows >= S and columns >= out are clipped)
                if (tid_e == 0) bulk_wait_read1();   // the store issued from this buffer two chunks ago has read it
                named_bar_sync(1, 128);
                uint4 *ys = reinterpret_cast<uint4 *>(base_ptr + (ystage - base) + ybuf * kYStage);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint4 pk;
                    pk.x = pack_bf16x2(v[8 * q + 0], v[8 * q + 1]);
                    pk.y = pack_bf16x2(v[8 * q + 2], v[8 * q + 3]);
                    pk.z = pack_bf16x2(v[8 * q + 4], v[8 * q + 5]);
                    pk.w = pack_bf16x2(v[8 * q + 6], v[8 * q + 7]);
                    ys[m * 4 + q] = pk;
                }
                fence_proxy_async_smem();
                named_bar_sync(1, 128);
                if (tid_e == 0) {
                    tma_store_2d(&P.tmY, ystage + ybuf * kYStage, it.n0 + 32 * c, row0);
                    bulk_commit();
                }
                ybuf ^= 1;
            }
            if (tid_e == 0) {
                bulk_wait_all();
                dbg_stamp(a, 6);
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (wpair && warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(256) : "memory");
    }
    // the last CTA to leave resets the counters for the next launch
    if (threadIdx.x == 0) {
        __threadfence();
        if (atom_add_acq_rel_gpu(a.ctr + 1, 1) == (int)gridDim.x - 1) {
            a.ctr[0] = 0;
            a.ctr[1] = 0;
            for (int t = 0; t < a.n_groups * a.n_wt; ++t) a.ctr[2 + t] = 0;
        }
    }
}

static_assert(sizeof(Dec3Args) + sizeof(Dec3Inline) <= 32764, "kernel parameters exceed 32 KB");
static_assert(2 * ShrinkSmem<64, 4, kShrMI>::end <= 6 * kStage3, "shrink workers exceed the ring");

template <int RP>
int launch_dec3_impl(const Dec3Args &a, const Dec3Inline &in, int clusters, cudaStream_t st) {
    auto kern = smlm_dec3_kernel<RP>;
    const size_t smem = 1024 + (size_t)a.stages * kStage3 + 2 * kYStage + 256;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        attr_done = true;
    }
    return (int)launch_pdl(kern, dim3(2 * clusters), dim3(kT3), smem, st, a, in);
}

}  // namespace

int dec3_stages() { return 6; }

int launch_dec3(const Dec3Args &a, const Dec3Inline &in, int clusters, cudaStream_t st) {
    switch (a.r_pad) {
        case 16: return launch_dec3_impl<16>(a, in, clusters, st);
        case 32: return launch_dec3_impl<32>(a, in, clusters, st);
        case 64: return launch_dec3_impl<64>(a, in, clusters, st);
    }
    return (int)cudaErrorInvalidValue;
}

}  // namespace smlm
