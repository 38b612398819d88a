// kernels_attn.cu -- the Alg. 1 attention branch: segment-wise
// causal attention for FINETUNE / EVAL / PREFILL rows, KV-cache initialisation for prefills and
// append + attention over the cache for decodes (reading R14, oracle/attention.py).
//
//   attn_kv_write_kernel   : prefill rows -> cache[slot][0..L) (decode rows are appended by the
//                            decode kernel: cache[slot][past + i])
//   attn_prefill_kernel    : one CTA per (segment, 128-query block, query head), tcgen05 with the
//                            accumulators in TMEM: S = Q K_j^T (M=128, N=128 keys, K=d=128) ->
//                            online softmax by 4 warps (thread = query row; running max / sum in
//                            registers, O rescaled in TMEM when the max moves) -> P (bf16, smem) ->
//                            O += P V_j (N=d, K=128 keys, V as the MN-major operand); K/V tiles by
//                            TMA in a 2-deep ring; S_{j+1} is issued while the softmax of j runs.
//   attn_decode_split_kernel + attn_decode_combine_kernel : split-KV decode, HBM-bound: CTA per
//                            (decode row, KV head, 256-key chunk) -- each K and V row read once for
//                            all G query heads of the group, 64 KB of loads in flight per CTA --
//                            then the splits merged in order (max, sum, o rescaled in fp32).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <cstdio>


#include <algorithm>

#include "device_types.h"
#include "pdl.cuh"
#include "sm100.cuh"

namespace smlm {
using namespace sm100;

namespace {

constexpr int kAT = 384;                 // prefill: 12 warps (0 TMA, 1 MMA, 2 TMEM alloc, 4-11 softmax)
constexpr uint32_t kQBytes = 32768;      // 128 rows x 128 d bf16 (two 64-wide SW128 boxes)
constexpr uint32_t kKVBytes = 65536;     // K tile (32 KB) + V tile (32 KB)
constexpr uint32_t kPBytes = 32768;      // P: 128 rows x 128 keys bf16 (two buffers)

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__global__ void __launch_bounds__(kAT, 1) attn_prefill_kernel(const __grid_constant__ AttnArgs a, int n_units) {
    // persistent: CTA c takes work units c, c + grid, ... (unit = (128-query block, query head),
    // the items sorted by key-block count, longest first); block counters run across units so
    // the TMA ring, the S buffer and the P buffers stream from one unit into the next
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    const uint32_t q_s = base;
    auto kv_s = [&](int b) { return base + kQBytes + (uint32_t)b * kKVBytes; };
    const uint32_t p_s = base + kQBytes + 2 * kKVBytes;
    const uint32_t bar = p_s + 2 * kPBytes;
    const uint32_t q_full = bar, q_empty = bar + 8, s_full = bar + 16, s_free = bar + 24, p_full = bar + 32;
    auto o_done = [&](int b) { return bar + 40u + 8u * b; };   // PV_G committed, G % 2 == b (P buffer b free)
    // K and V of a key block have their own barriers: K_b is free once S has read it, V_b once PV has
    auto k_full = [&](int b) { return bar + 56u + 8u * b; };
    auto k_empty = [&](int b) { return bar + 72u + 8u * b; };
    auto v_full = [&](int b) { return bar + 88u + 8u * b; };
    auto v_empty = [&](int b) { return bar + 104u + 8u * b; };
    const uint32_t tmem_slot = bar + 120;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int group = a.n_heads / a.n_kv_heads;
    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        mbar_init(s_full, 1);
        mbar_init(s_free, 256);
        mbar_init(p_full, 256);
        for (int b = 0; b < 2; ++b) {
            mbar_init(o_done(b), 1);
            mbar_init(k_full(b), 1);
            mbar_init(k_empty(b), 1);
            mbar_init(v_full(b), 1);
            mbar_init(v_empty(b), 1);
        }
        fence_mbar_init();
        tma_prefetch_desc(&a.tmQ);
        tma_prefetch_desc(&a.tmK);
        tma_prefetch_desc(&a.tmV);
    }
    if (warp == 2) tmem_alloc(tmem_slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(base_ptr + (tmem_slot - base));
    const uint32_t S_t = tmem, O_t = tmem + 128;
    pdl_wait();   // the item table is written by the stream's plan upload
    pdl_trigger();

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            int G = 0, u = 0;
            for (int w = blockIdx.x; w < n_units; w += gridDim.x, ++u) {
                const AttnItem it = a.items[w / a.n_heads];
                const int head = w % a.n_heads, kvh = head / group, nkb = it.qb + 1;
                if (u > 0) mbar_wait(q_empty, (u - 1) & 1);   // the previous unit's S MMAs read Q
                mbar_expect_tx(q_full, kQBytes);
                for (int db = 0; db < 2; ++db)
                    tma_load_2d(q_s + 16384u * db, &a.tmQ, q_full, head * 128 + 64 * db, it.row0 + it.qb * 128);
                for (int j = 0; j < nkb; ++j, ++G) {
                    const int b = G & 1;
                    const int k0 = it.row0 + j * 128;
                    // K_j: B operand of S = Q K^T, K-major (rows = keys, 128 B of d per row)
                    mbar_wait(k_empty(b), ((G >> 1) & 1) ^ 1);
                    mbar_expect_tx(k_full(b), kKVBytes / 2);
                    for (int db = 0; db < 2; ++db)
                        tma_load_2d(kv_s(b) + 16384u * db, &a.tmK, k_full(b), kvh * 128 + 64 * db, k0);
                    // V_j: B operand of O += P V, MN-major (rows = keys, 64-wide d boxes)
                    mbar_wait(v_empty(b), ((G >> 1) & 1) ^ 1);
                    mbar_expect_tx(v_full(b), kKVBytes / 2);
                    for (int kb = 0; kb < 2; ++kb)
                        for (int db = 0; db < 2; ++db)
                            tma_load_2d(kv_s(b) + 32768u + 16384u * kb + 8192u * db, &a.tmV, v_full(b),
                                        kvh * 128 + 64 * db, k0 + 64 * kb);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        // order per block G: S_G (after the softmax has read S_{G-1}), then PV_{G-1} -- so S_G
        // overlaps the softmax of G-1 and PV_{G-1} overlaps the softmax of G
        constexpr uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);
        constexpr uint32_t idesc_o = idesc_bf16(128, 128, 0, 1);
        auto issue_pv = [&](int Gp, bool first) {
            const int b = Gp & 1;
            mbar_wait(v_full(b), (Gp >> 1) & 1);
            mbar_wait(p_full, Gp & 1);       // P_Gp in smem, O rescaled
            tc_fence_after();
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t pa = p_s + (uint32_t)b * kPBytes + 16384u * (k >> 2) + 32u * (k & 3);
                    const uint32_t vb = kv_s(b) + 32768u + 16384u * (k >> 2) + 2048u * (k & 3);
                    mma_bf16(O_t, smem_desc(pa, 16, 1024, kSw128), smem_desc(vb, 8192, 1024, kSw128), idesc_o,
                             (!first || k > 0) ? 1u : 0u);
                }
                mma_commit(v_empty(b));
                mma_commit(o_done(b));
            }
            __syncwarp();
        };
        int G = 0, u = 0;
        for (int w = blockIdx.x; w < n_units; w += gridDim.x, ++u) {
            const AttnItem it = a.items[w / a.n_heads];
            const int nkb = it.qb + 1;
            mbar_wait(q_full, u & 1);
            for (int j = 0; j < nkb; ++j, ++G) {
                if (G > 0) mbar_wait(s_free, (G - 1) & 1);   // the softmax has read S_{G-1}
                const int b = G & 1;
                mbar_wait(k_full(b), (G >> 1) & 1);
                tc_fence_after();
                if (lane == 0) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t off = 16384u * (k >> 2) + 32u * (k & 3);
                        mma_bf16(S_t, smem_desc(q_s + off, 16, 1024, kSw128),
                                 smem_desc(kv_s(b) + off, 16, 1024, kSw128), idesc_s, k > 0);
                    }
                    mma_commit(s_full);
                    mma_commit(k_empty(b));
                    if (j == nkb - 1) mma_commit(q_empty);
                }
                __syncwarp();
                if (j > 0) issue_pv(G - 1, j == 1);
            }
            issue_pv(G - 1, nkb == 1);   // the unit's last block
        }
    } else if (warp >= 4) {
        // ---------------- online softmax + epilogue ----------------
        // two warpgroups: warpgroup wg takes key columns [64 wg, 64 wg + 64) of every S block and
        // output columns [64 wg, 64 wg + 64) of O; thread = query row (TMEM lane).  The row's max
        // is combined through shared memory each block; each warpgroup keeps the sum of its own
        // columns (both use the same reference max), added at the unit's end.
        const int wg = (warp - 4) >> 2;
        const int m = (threadIdx.x - 128) & 127;
        const int tid_s = threadIdx.x - 128;   // 0..255
        const uint32_t lane_base = (uint32_t)(((warp - 4) & 3) * 32) << 16;
        const uint32_t col0 = 64u * (uint32_t)wg;
        const float sl2 = a.scale * 1.4426950408889634f;
        uint8_t *pp = base_ptr + (p_s - base);
        __shared__ float s_x[128];   // per row: warpgroup 1's max -> the new reference max; at the end l
        int G = 0;
#ifdef SMLM_MEASURE
        long long c_ws = 0, c_ld = 0, c_exp = 0, c_wo = 0, c_rs = 0, c_ep = 0, c0, c_begin = clock64();
#define TSTAMP() (c0 = clock64())
#define TACC(x) (x += clock64() - c0)
#else
#define TSTAMP()
#define TACC(x)
#endif
        for (int w = blockIdx.x; w < n_units; w += gridDim.x) {
            const AttnItem it = a.items[w / a.n_heads];
            const int head = w % a.n_heads, nkb = it.qb + 1;
            const int qi = it.qb * 128 + m;           // query position inside the segment
            float mi = -INFINITY, li = 0.f;           // reference max (log2 units), this half's sum
            for (int j = 0; j < nkb; ++j, ++G) {
                TSTAMP();
                mbar_wait(s_full, G & 1);
                TACC(c_ws);
                TSTAMP();
                tc_fence_after();
                const int kbase = j * 128 + (int)col0;
                // this half of the S row into registers, then S is free for S_{G+1}
                uint32_t sr[64];
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t r[32];
                    tmem_ld32(S_t + lane_base + col0 + 32u * c, r);
#pragma unroll
                    for (int e = 0; e < 32; ++e) sr[32 * c + e] = r[e];
                }
                tmem_wait_ld();
                tc_fence_before();
                mbar_arrive(s_free);
                TACC(c_ld);
                TSTAMP();
                // keys visible to this row: kj <= qi and kj < len  <=>  kj - kbase < lim
                const int lim = min(qi + 1, it.len) - kbase;
                // every key of this half visible to every row of the warp (all but the diagonal and
                // segment-end blocks): no per-key predicates
                // masked keys become -inf in the registers (only in the diagonal / segment-end
                // blocks: a warp-uniform branch), so the max and exp loops below carry no per-key
                // predicate (exp2(-inf) = 0)
                if (!__all_sync(0xffffffffu, lim >= 64)) {
#pragma unroll
                    for (int e = 0; e < 64; ++e)
                        if (e >= lim) sr[e] = 0xff800000u;   // -inf
                }
                float mx = -INFINITY;
#pragma unroll
                for (int e = 0; e < 64; ++e) mx = fmaxf(mx, __uint_as_float(sr[e]));
                // the row's max: warpgroup 1 publishes its half, warpgroup 0 combines and publishes the
                // new reference.  Lazy rescaling: the reference max moves only when the block's max
                // exceeds it by more than 2^8 (probabilities stay <= 256), so O is rarely rescaled
                if (wg == 1) s_x[m] = mx;
                named_bar_sync(1, 256);
                float m_new;
                if (wg == 0) {
                    mx = fmaxf(mx, s_x[m]);
                    m_new = (mx * sl2 > mi + 8.f) ? mx * sl2 : mi;
                    s_x[m] = m_new;
                }
                named_bar_sync(1, 256);
                if (wg == 1) m_new = s_x[m];
                const float alpha = fast_exp2(mi - m_new);   // 0 on the first block (mi = -inf), else 1 unless moved
                const uint32_t pb = G & 1;
                TACC(c_exp);
                TSTAMP();
                if (G >= 2) mbar_wait(o_done(pb), ((G >> 1) - 1) & 1);   // PV_{G-2} has read P buffer pb
                TACC(c_wo);
                TSTAMP();
                float sum = 0.f;   // of the fp32 probabilities (P itself is rounded to bf16 for the MMA)
                uint8_t *pbuf = pp + pb * kPBytes + wg * 16384;   // key half wg of P (64 keys, SW128)
                const float nm = -m_new;
#pragma unroll
                for (int ch = 0; ch < 8; ++ch) {   // 16-byte chunks of 8 keys
                    uint32_t pk[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int e = 8 * ch + 2 * q;
                        const float p0 = fast_exp2(fmaf(__uint_as_float(sr[e]), sl2, nm));
                        const float p1 = fast_exp2(fmaf(__uint_as_float(sr[e + 1]), sl2, nm));
                        sum += p0 + p1;
                        const __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
                        pk[q] = *reinterpret_cast<const uint32_t *>(&b2);
                    }
                    *reinterpret_cast<uint4 *>(pbuf + m * 128 + ((ch ^ (m & 7)) << 4)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
                li = li * alpha + sum;
                TACC(c_exp);
                TSTAMP();
                if (j > 0) {
                    // P_{G-1} V_{G-1} has landed in O: rescale this warpgroup's 64 columns of it
                    // (warp-collective tcgen05.ld / st: the warp rescales when any of its rows needs it)
                    mbar_wait(o_done((G - 1) & 1), ((G - 1) >> 1) & 1);
                    tc_fence_after();
                    if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
                        for (int c = 0; c < 2; ++c) {
                            uint32_t r[32];
                            tmem_ld32(O_t + lane_base + col0 + 32u * c, r);
                            tmem_wait_ld();
#pragma unroll
                            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
                            tmem_st32(O_t + lane_base + col0 + 32u * c, r);
                        }
                        tmem_wait_st();
                    }
                }
                mi = m_new;
                fence_proxy_async_smem();   // P (generic stores) -> the MMA (async proxy)
                tc_fence_before();
                mbar_arrive(p_full);
                TACC(c_rs);
            }
            TSTAMP();
            // epilogue of the unit: O / l -> bf16 rows of O [S, Hq, d], l = the two halves' sums
            // (added in the same order by both warpgroups)
            named_bar_sync(1, 256);   // warpgroup 1 has read the last block's reference max
            if (wg == 1) s_x[m] = li;
            mbar_wait(o_done((G - 1) & 1), ((G - 1) >> 1) & 1);
            tc_fence_after();
            named_bar_sync(1, 256);
            if (wg == 0) s_x[m] = li + s_x[m];
            named_bar_sync(1, 256);
            const float invl = 1.f / s_x[m];
            // stage the O rows in P buffer 0 (free: the unit's last PV has completed, the next
            // unit's softmax has not started) so the global stores are whole 256-byte rows
            uint8_t *ostage = pp;   // 128 rows x 256 B, 16-byte units XOR-swizzled by row
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
                uint32_t r[32];
                tmem_ld32(O_t + lane_base + col0 + 32u * c, r);
                tmem_wait_ld();
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint4 v;
                    v.x = pack_bf16x2(__uint_as_float(r[8 * q + 0]) * invl, __uint_as_float(r[8 * q + 1]) * invl);
                    v.y = pack_bf16x2(__uint_as_float(r[8 * q + 2]) * invl, __uint_as_float(r[8 * q + 3]) * invl);
                    v.z = pack_bf16x2(__uint_as_float(r[8 * q + 4]) * invl, __uint_as_float(r[8 * q + 5]) * invl);
                    v.w = pack_bf16x2(__uint_as_float(r[8 * q + 6]) * invl, __uint_as_float(r[8 * q + 7]) * invl);
                    const int u = 8 * wg + 4 * c + q;   // 16-byte unit of the row (16 per row)
                    *reinterpret_cast<uint4 *>(ostage + m * 256 + ((u ^ (m & 15)) << 4)) = v;
                }
            }
            named_bar_sync(1, 256);
            {
                const int rsub = tid_s >> 4, u = tid_s & 15;   // 16 rows per pass, 16 threads per row
                __nv_bfloat16 *Ob = reinterpret_cast<__nv_bfloat16 *>(a.O);
#pragma unroll 2
                for (int r0 = 0; r0 < 128; r0 += 16) {
                    const int rr = r0 + rsub;
                    const int qr = it.qb * 128 + rr;
                    if (qr < it.len)
                        *reinterpret_cast<uint4 *>(Ob + ((size_t)(it.row0 + qr) * a.n_heads + head) * 128 + 8 * u) =
                            *reinterpret_cast<const uint4 *>(ostage + rr * 256 + ((u ^ (rr & 15)) << 4));
                }
            }
            tc_fence_before();   // the O reads are ordered before the next unit's p_full
            named_bar_sync(1, 256);   // the staging buffer is P buffer 0 of the next unit; s_x reused
            TACC(c_ep);
        }
#ifdef SMLM_MEASURE
        if (a.dbg && tid_s == 0 && blockIdx.x % 16 == 0) {
            const double T = (double)(clock64() - c_begin);
            printf("[attn prefill] cta %d blocks %d cycles %.0f wait_S %.1f%% ld_S %.1f%% max+exp+P %.1f%% wait_Pfree %.1f%% "
                   "wait_PV+rescale %.1f%% epilogue %.1f%%\n",
                   blockIdx.x, G, T, 100 * c_ws / T, 100 * c_ld / T, 100 * c_exp / T, 100 * c_wo / T, 100 * c_rs / T, 100 * c_ep / T);
        }
#endif
#undef TSTAMP
#undef TACC
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

// ---- prefill, two query heads of one KV group per CTA (GQA group even) ----
// Unit = (128-query block, KV head, head pair): the two heads' 128-row tiles share every K / V
// block, so the tensor pipe always has the other tile's S / PV MMAs while a softmax warpgroup
// works (FA4-style ping-pong of two tiles).  12 warps: 0 TMA (Q, K), 1 MMA issuer, 2 TMEM
// allocator, 3 TMA (V), 4-7 softmax of tile 0, 8-11 softmax of tile 1 (thread = query row).
// Shared memory: Q0 Q1 | K ring 2 | V (one buffer) | P0 P1 (one buffer per tile) = 224 KB.
// TMEM: S0 S1 O0 O1 (128 columns each).
constexpr int kAT2 = 384;
size_t attn_prefill2_smem() { return 1024 + 2 * kQBytes + 2 * (kKVBytes / 2) + kKVBytes / 2 + 2 * kPBytes + 256; }

__global__ void __launch_bounds__(kAT2, 1) attn_prefill2_kernel(const __grid_constant__ AttnArgs a, int n_units) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    auto q_s = [&](int t) { return base + (uint32_t)t * kQBytes; };
    auto k_s = [&](int b) { return base + 2u * kQBytes + (uint32_t)b * 32768u; };
    const uint32_t v_s = base + 2u * kQBytes + 65536u;
    auto p_s = [&](int t) { return base + 2u * kQBytes + 98304u + (uint32_t)t * kPBytes; };
    const uint32_t bar = base + 2u * kQBytes + 98304u + 2u * kPBytes;
    const uint32_t q_full = bar, q_empty = bar + 8, v_full = bar + 16, v_empty = bar + 24;
    auto k_full = [&](int b) { return bar + 32u + 8u * b; };
    auto k_empty = [&](int b) { return bar + 48u + 8u * b; };
    auto s_full = [&](int t) { return bar + 64u + 8u * t; };
    auto s_free = [&](int t) { return bar + 80u + 8u * t; };
    auto p_full = [&](int t) { return bar + 96u + 8u * t; };
    auto o_done = [&](int t) { return bar + 112u + 8u * t; };   // PV of tile t committed (P_t free, O_t updated)
    const uint32_t tmem_slot = bar + 128;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int group = a.n_heads / a.n_kv_heads;
    const int hpairs = a.n_heads / 2;
    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        mbar_init(v_full, 1);
        mbar_init(v_empty, 1);
        for (int b = 0; b < 2; ++b) {
            mbar_init(k_full(b), 1);
            mbar_init(k_empty(b), 1);
            mbar_init(s_full(b), 1);
            mbar_init(s_free(b), 128);
            mbar_init(p_full(b), 128);
            mbar_init(o_done(b), 1);
        }
        fence_mbar_init();
        tma_prefetch_desc(&a.tmQ);
        tma_prefetch_desc(&a.tmK);
        tma_prefetch_desc(&a.tmV);
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t *>(base_ptr + (tmem_slot - base));
    auto S_t = [&](int t) { return tmem + 128u * (uint32_t)t; };
    auto O_t = [&](int t) { return tmem + 256u + 128u * (uint32_t)t; };
    pdl_wait();   // the item table is written by the stream's plan upload
    pdl_trigger();

    if (warp == 0) {
        // ---------------- TMA: Q of both heads, K ring ----------------
        if (lane == 0) {
            int G = 0, u = 0;
            for (int w = blockIdx.x; w < n_units; w += gridDim.x, ++u) {
                const AttnItem it = a.items[w / hpairs];
                const int h0 = 2 * (w % hpairs), kvh = h0 / group, nkb = it.qb + 1;
                if (u > 0) mbar_wait(q_empty, (u - 1) & 1);   // the previous unit's S MMAs read Q
                mbar_expect_tx(q_full, 2 * kQBytes);
                for (int t = 0; t < 2; ++t)
                    for (int db = 0; db < 2; ++db)
                        tma_load_2d(q_s(t) + 16384u * db, &a.tmQ, q_full, (h0 + t) * 128 + 64 * db, it.row0 + it.qb * 128);
                for (int j = 0; j < nkb; ++j, ++G) {
                    const int b = G & 1;
                    mbar_wait(k_empty(b), ((G >> 1) & 1) ^ 1);
                    mbar_expect_tx(k_full(b), 32768u);
                    for (int db = 0; db < 2; ++db)
                        tma_load_2d(k_s(b) + 16384u * db, &a.tmK, k_full(b), kvh * 128 + 64 * db, it.row0 + j * 128);
                }
            }
        }
    } else if (warp == 2) {
        // ---------------- KV-cache writes of the PREFILL rows (no separate launch) ----------------
        // this warp is idle after the TMEM allocation: rows b, b + grid, ... of the cache-write list
        // are copied with 16-byte loads / stores while the tensor pipe and the softmax run
        // (loads of several rows in flight before their stores: one warp must keep ~16 KB moving)
        // the write list is per segment {first row, slot, offset in the list, length}: row rr of the
        // list is found by a scan over the (few) segments
        const int re = a.n_kv_heads * 16;   // uint4 per K (or V) row
        constexpr int kR = 4;               // rows per batch
        int sg = 0;                         // segment of the batch's first row (rows increase)
        for (int r0 = blockIdx.x; a.n_kv_heads <= 8 && r0 < a.n_cache_rows; r0 += kR * gridDim.x) {
            uint4 kv[kR][2][4];
            int src[kR], dst[kR];   // input row, cache row (slot * capacity + position); -1: none
#pragma unroll
            for (int q = 0; q < kR; ++q) {
                const int rr = r0 + q * gridDim.x;
                src[q] = -1;
                dst[q] = 0;
                if (rr < a.n_cache_rows) {
                    int g2 = sg;
                    while (g2 + 1 < a.n_rows && a.rows[g2 + 1].pos <= rr) ++g2;
                    if (q == 0) sg = g2;
                    const AttnRow seg = a.rows[g2];
                    src[q] = seg.row + (rr - seg.pos);
                    dst[q] = seg.slot * a.cache_capacity + (rr - seg.pos);
                }
            }
#pragma unroll
            for (int q = 0; q < kR; ++q)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = lane + 32 * u;
                    if (src[q] >= 0 && i < re) {
                        kv[q][0][u] = reinterpret_cast<const uint4 *>(a.K)[(size_t)src[q] * re + i];
                        kv[q][1][u] = reinterpret_cast<const uint4 *>(a.V)[(size_t)src[q] * re + i];
                    }
                }
#pragma unroll
            for (int q = 0; q < kR; ++q)
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = lane + 32 * u;
                    if (src[q] >= 0 && i < re) {
                        reinterpret_cast<uint4 *>(a.K_cache)[(size_t)dst[q] * re + i] = kv[q][0][u];
                        reinterpret_cast<uint4 *>(a.V_cache)[(size_t)dst[q] * re + i] = kv[q][1][u];
                    }
                }
        }
        // (n_kv_heads <= 8: a K row is at most 128 uint4 = 4 per lane)
    } else if (warp == 3) {
        // ---------------- TMA: V (one buffer; free once both tiles' PV have read it) ----------------
        if (lane == 0) {
            int G = 0;
            for (int w = blockIdx.x; w < n_units; w += gridDim.x) {
                const AttnItem it = a.items[w / hpairs];
                const int kvh = 2 * (w % hpairs) / group, nkb = it.qb + 1;
                for (int j = 0; j < nkb; ++j, ++G) {
                    mbar_wait(v_empty, (G & 1) ^ 1);
                    mbar_expect_tx(v_full, 32768u);
                    for (int kb = 0; kb < 2; ++kb)
                        for (int db = 0; db < 2; ++db)
                            tma_load_2d(v_s + 16384u * kb + 8192u * db, &a.tmV, v_full, kvh * 128 + 64 * db,
                                        it.row0 + j * 128 + 64 * kb);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        // per key block G: S_0(G), S_1(G) (each after its softmax has read S_t(G-1)), then
        // PV_0(G-1), PV_1(G-1) -- a tile's MMAs run while the other tile's softmax works
        constexpr uint32_t idesc_s = idesc_bf16(128, 128, 0, 0);
        constexpr uint32_t idesc_o = idesc_bf16(128, 128, 0, 1);
        auto issue_pv = [&](int Gp, bool first) {
            mbar_wait(v_full, Gp & 1);
            for (int t = 0; t < 2; ++t) {
                mbar_wait(p_full(t), Gp & 1);   // P_t in smem, O_t rescaled
                tc_fence_after();
                if (lane == 0) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t pa = p_s(t) + 16384u * (k >> 2) + 32u * (k & 3);
                        const uint32_t vb = v_s + 16384u * (k >> 2) + 2048u * (k & 3);
                        mma_bf16(O_t(t), smem_desc(pa, 16, 1024, kSw128), smem_desc(vb, 8192, 1024, kSw128), idesc_o,
                                 (!first || k > 0) ? 1u : 0u);
                    }
                    mma_commit(o_done(t));
                }
                __syncwarp();
            }
            if (lane == 0) mma_commit(v_empty);
            __syncwarp();
        };
        int G = 0, u = 0;
        for (int w = blockIdx.x; w < n_units; w += gridDim.x, ++u) {
            const AttnItem it = a.items[w / hpairs];
            const int nkb = it.qb + 1;
            mbar_wait(q_full, u & 1);
            for (int j = 0; j < nkb; ++j, ++G) {
                const int b = G & 1;
                mbar_wait(k_full(b), (G >> 1) & 1);
                for (int t = 0; t < 2; ++t) {
                    if (G > 0) mbar_wait(s_free(t), (G - 1) & 1);   // softmax t has read S_t(G-1)
                    tc_fence_after();
                    if (lane == 0) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const uint32_t off = 16384u * (k >> 2) + 32u * (k & 3);
                            mma_bf16(S_t(t), smem_desc(q_s(t) + off, 16, 1024, kSw128), smem_desc(k_s(b) + off, 16, 1024, kSw128),
                                     idesc_s, k > 0);
                        }
                        mma_commit(s_full(t));
                    }
                    __syncwarp();
                }
                if (lane == 0) {
                    mma_commit(k_empty(b));
                    if (j == nkb - 1) mma_commit(q_empty);
                }
                __syncwarp();
                if (j > 0) issue_pv(G - 1, j == 1);
            }
            issue_pv(G - 1, nkb == 1);   // the unit's last block
        }
    } else if (warp >= 4) {
        // ---------------- online softmax + epilogue of tile t (thread = query row) ----------------
        const int t = (warp - 4) >> 2;
        const int m = (threadIdx.x - 128) & 127;
        const uint32_t lane_base = (uint32_t)(((warp - 4) & 3) * 32) << 16;
        const float sl2 = a.scale * 1.4426950408889634f;
        uint8_t *pbuf = base_ptr + (p_s(t) - base);   // P_t: two 64-key halves, SW128
        int G = 0;
#ifdef SMLM_MEASURE
        long long c_ws = 0, c_ld = 0, c_mx = 0, c_wo = 0, c_exp = 0, c_rs = 0, c_ep = 0, c0, c_begin = clock64();
#define TSTAMP() (c0 = clock64())
#define TACC(x) (x += clock64() - c0)
#else
#define TSTAMP()
#define TACC(x)
#endif
        for (int w = blockIdx.x; w < n_units; w += gridDim.x) {
            const AttnItem it = a.items[w / hpairs];
            const int head = 2 * (w % hpairs) + t, nkb = it.qb + 1;
            const int qi = it.qb * 128 + m;   // query position inside the segment
            float mi = -INFINITY, li = 0.f;   // reference max (log2 units), row sum
            for (int j = 0; j < nkb; ++j, ++G) {
                TSTAMP();
                mbar_wait(s_full(t), G & 1);
                TACC(c_ws);
                TSTAMP();
                tc_fence_after();
                uint32_t sr[128];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t r[32];
                    tmem_ld32(S_t(t) + lane_base + 32u * c, r);
#pragma unroll
                    for (int e = 0; e < 32; ++e) sr[32 * c + e] = r[e];
                }
                tmem_wait_ld();
                tc_fence_before();
                mbar_arrive(s_free(t));
                TACC(c_ld);
                TSTAMP();
                // keys visible to this row: kj <= qi and kj < len; masked keys -> -inf (warp-uniform
                // branch: only the diagonal and segment-end blocks)
                const int lim = min(qi + 1, it.len) - j * 128;
                if (!__all_sync(0xffffffffu, lim >= 128)) {
#pragma unroll
                    for (int e = 0; e < 128; ++e)
                        if (e >= lim) sr[e] = 0xff800000u;
                }
                float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};   // independent chains
#pragma unroll
                for (int e = 0; e < 128; ++e) mx4[e & 3] = fmaxf(mx4[e & 3], __uint_as_float(sr[e]));
                const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
                // lazy rescaling: the reference max moves only past 2^8 (probabilities <= 256)
                const float m_new = (mx * sl2 > mi + 8.f) ? mx * sl2 : mi;
                const float alpha = fast_exp2(mi - m_new);   // 0 on the first block, else 1 unless moved
                // PV_t(G-1) has read P_t and updated O_t (also the previous unit's last block)
                TACC(c_mx);
                TSTAMP();
                if (G > 0) mbar_wait(o_done(t), (G - 1) & 1);
                TACC(c_wo);
                TSTAMP();
                tc_fence_after();
                // packed fp32 pairs (FFMA2 / FADD2): the scale-and-shift and the row sum take one
                // instruction per two keys
                float2 sum2[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};   // independent chains
                const float2 sl2v = make_float2(sl2, sl2), nmv = make_float2(-m_new, -m_new);
#pragma unroll
                for (int ch = 0; ch < 16; ++ch) {   // 16-byte chunks of 8 keys: chunk ch of key half ch / 8
                    uint32_t pk[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int e = 8 * ch + 2 * q;
                        const float2 x = __ffma2_rn(make_float2(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])), sl2v, nmv);
                        const float2 p = make_float2(fast_exp2(x.x), fast_exp2(x.y));
                        sum2[q] = __fadd2_rn(sum2[q], p);
                        const __nv_bfloat162 b2 = __floats2bfloat162_rn(p.x, p.y);
                        pk[q] = *reinterpret_cast<const uint32_t *>(&b2);
                    }
                    const int kh = ch >> 3, cc = ch & 7;
                    *reinterpret_cast<uint4 *>(pbuf + kh * 16384 + m * 128 + ((cc ^ (m & 7)) << 4)) =
                        make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
                const float2 s01 = __fadd2_rn(sum2[0], sum2[1]), s23 = __fadd2_rn(sum2[2], sum2[3]);
                li = li * alpha + ((s01.x + s23.x) + (s01.y + s23.y));
                TACC(c_exp);
                TSTAMP();
                if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
                    for (int c = 0; c < 4; ++c) {
                        uint32_t r[32];
                        tmem_ld32(O_t(t) + lane_base + 32u * c, r);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
                        tmem_st32(O_t(t) + lane_base + 32u * c, r);
                    }
                    tmem_wait_st();
                }
                mi = m_new;
                fence_proxy_async_smem();   // P (generic stores) -> the MMA (async proxy)
                tc_fence_before();
                mbar_arrive(p_full(t));
                TACC(c_rs);
            }
            TSTAMP();
            // epilogue: O_t / l -> bf16 rows of O [S, Hq, d], staged in P_t (its last PV is done)
            mbar_wait(o_done(t), (G - 1) & 1);
            tc_fence_after();
            const float inv = 1.f / li;
            const bool full = it.qb * 128 + 128 <= it.len;   // every row of the tile is stored
            {
                uint32_t r[4][32];   // the whole O row behind one wait
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld32(O_t(t) + lane_base + 32u * c, r[c]);
                tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t vv[4];
#pragma unroll
                        for (int h = 0; h < 4; ++h) {   // FMUL2: two columns per instruction
                            const float2 o2 = __fmul2_rn(make_float2(__uint_as_float(r[c][8 * q + 2 * h]),
                                                                     __uint_as_float(r[c][8 * q + 2 * h + 1])),
                                                         make_float2(inv, inv));
                            vv[h] = pack_bf16x2(o2.x, o2.y);
                        }
                        const uint4 v = make_uint4(vv[0], vv[1], vv[2], vv[3]);
                        const int uu = 4 * c + q;   // 16-byte unit of the 256-byte row
                        if (full)   // two 64-column SW128 halves (the TMA store's layout, = P's)
                            *reinterpret_cast<uint4 *>(pbuf + (uu >> 3) * 16384 + m * 128 + (((uu & 7) ^ (m & 7)) << 4)) = v;
                        else
                            *reinterpret_cast<uint4 *>(pbuf + m * 256 + ((uu ^ (m & 15)) << 4)) = v;
                    }
            }
            if (full) {
                fence_proxy_async_smem();
                named_bar_sync(1 + t, 128);
                if (m == 0) {
                    for (int h = 0; h < 2; ++h)
                        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                                         reinterpret_cast<uint64_t>(&a.tmO)),
                                     "r"(p_s(t) + 16384u * h), "r"(head * 128 + 64 * h), "r"(it.row0 + it.qb * 128)
                                     : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // P_t reusable
                }
            } else {
                named_bar_sync(1 + t, 128);
                const int rsub = m >> 4, uu = m & 15;   // 8 rows per pass, 16 threads per row
                __nv_bfloat16 *Ob = reinterpret_cast<__nv_bfloat16 *>(a.O);
#pragma unroll 2
                for (int r0 = 0; r0 < 128; r0 += 8) {
                    const int rr = r0 + rsub;
                    const int qr = it.qb * 128 + rr;
                    if (qr < it.len)
                        *reinterpret_cast<uint4 *>(Ob + ((size_t)(it.row0 + qr) * a.n_heads + head) * 128 + 8 * uu) =
                            *reinterpret_cast<const uint4 *>(pbuf + rr * 256 + ((uu ^ (rr & 15)) << 4));
                }
            }
            tc_fence_before();          // the O reads are ordered before the next unit's PV
            named_bar_sync(1 + t, 128);   // the staging buffer is P_t of the next unit's first block
            TACC(c_ep);
        }
#ifdef SMLM_MEASURE
        if (a.dbg && m == 0 && blockIdx.x % 16 == 0) {
            const double T = (double)(clock64() - c_begin);
            printf("[attn prefill2] cta %d tile %d blocks %d cycles %.0f wait_S %.1f%% ld_S %.1f%% mask+max %.1f%% wait_PVdone %.1f%% "
                   "exp+P %.1f%% rescale+arrive %.1f%% epilogue %.1f%%\n",
                   blockIdx.x, t, G, T, 100 * c_ws / T, 100 * c_ld / T, 100 * c_mx / T, 100 * c_wo / T, 100 * c_exp / T,
                   100 * c_rs / T, 100 * c_ep / T);
        }
#endif
#undef TSTAMP
#undef TACC
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---- KV-cache writes: row t of K/V [S, Hkv, d] -> cache slot / position (plan: AttnRow) ----
__global__ void __launch_bounds__(256) attn_kv_write_kernel(const AttnArgs a) {
    pdl_wait();
    pdl_trigger();
    // row blockIdx.x of the write list: its segment record by binary search over the offsets
    const int rr = blockIdx.x;
    int lo = 0, hi = a.n_rows - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.rows[mid].pos <= rr) lo = mid;
        else hi = mid - 1;
    }
    const AttnRow sg = a.rows[lo];
    const AttnRow rw{sg.row + (rr - sg.pos), sg.slot, rr - sg.pos, 0};
    if (rw.slot < 0) return;
    const size_t row_elems = (size_t)a.n_kv_heads * 128;
    const uint4 *ks = reinterpret_cast<const uint4 *>(reinterpret_cast<const __nv_bfloat16 *>(a.K) + (size_t)rw.row * row_elems);
    const uint4 *vs = reinterpret_cast<const uint4 *>(reinterpret_cast<const __nv_bfloat16 *>(a.V) + (size_t)rw.row * row_elems);
    const size_t dst = ((size_t)rw.slot * a.cache_capacity + rw.pos) * row_elems;
    uint4 *kd = reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(a.K_cache) + dst);
    uint4 *vd = reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(a.V_cache) + dst);
    for (int i = threadIdx.x; i < (int)(row_elems / 8); i += blockDim.x) {
        kd[i] = ks[i];
        vd[i] = vs[i];
    }
}

// ---- decode (split-KV): CTA (decode row group, KV head, split) takes kAttnDecChunk = 128 cached
// keys of the group's cache slot.  HBM-bound: the slot's K / V bytes are read once for all rows of
// the group (the rows of one DECODE segment, up to kAttnDecCols / G of them) and the CTA's work
// beside its 64 KB of loads is kept small so that three CTAs per SM keep ~190 KB in flight.  The
// chunk's K and V arrive by TMA (SW128 boxes: ldmatrix conflict-free); the scores
// S^T = K_chunk Q^T and O^T = V_chunk^T P run on mma.sync m16n8k16 (keys x query columns, column =
// row * G + head, up to 32 columns; the tensor work is negligible, it only replaces CUDA-core dot
// products); K and V share one 32 KB buffer -- V is loaded into it once every warp is past S, so
// its load overlaps the softmax and four CTAs fit an SM (42 KB each); the chunk's max / sum /
// o (fp32) per (row, head) go to the workspace and
// attn_decode_combine_kernel merges the splits in split order.  P is rounded to bf16 for the PV
// product (as in the prefill kernel); the row sum is taken over the fp32 p ----
constexpr int kDecChunk = kAttnDecChunk;
// one 32 KB chunk buffer (K, then V once every warp is past S: the V load overlaps the softmax)
// and P [32 columns][136] beside it: 42 KB, four CTAs per SM
constexpr size_t kDecSmem = 1024 + 32768 + 32 * 136 * 2;
// byte offset of 16-byte unit c (0..15, 8 bf16 of d) of key row r in a SW128 chunk
__device__ __forceinline__ uint32_t dec_sw(int r, int c) {
    return (uint32_t)((c >> 3) * 16384 + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t &r0, uint32_t &r1, uint32_t &r2, uint32_t &r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
                 "{%0, %1, %2, %3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int G>
__global__ void __launch_bounds__(128, 4) attn_decode_split_kernel(const __grid_constant__ AttnArgs a,
                                                                    const __grid_constant__ AttnDecInline dinl) {
    const AttnRow *drows = a.dec_inline ? dinl.drows : a.drows;
    const AttnDGroup *dgroups = a.dec_inline ? dinl.dgroups : a.dgroups;
    pdl_wait();
    pdl_trigger();
    constexpr int NT = kAttnDecCols / 8;   // n8 tiles of query columns (column = row * G + head)
    const int s = blockIdx.x % a.max_splits;
    const int kvh = (blockIdx.x / a.max_splits) % a.n_kv_heads;
    const AttnDGroup grp = dgroups[blockIdx.x / (a.max_splits * a.n_kv_heads)];
    const int Lmax = grp.pos0 + grp.n;   // keys of the group's last row (the cache holds the rows themselves)
    const int j0 = s * kDecChunk;
    if (j0 >= Lmax) return;
    const int nk = min(kDecChunk, Lmax - j0);
    const int ncol = grp.n * G, ntiles = (ncol + 7) >> 3;
    extern __shared__ __align__(16) uint8_t dsm_raw0[];
    uint8_t *dsm_raw = dsm_raw0 + ((1024u - (smem_u32(dsm_raw0) & 1023u)) & 1023u);   // SW128: 1 KB aligned
    uint8_t *ksm = dsm_raw;              // K chunk [128 keys][128 d], two SW128 halves of 64 d
    uint8_t *vsm = dsm_raw;              // V chunk, same layout, in K's buffer after S
    __nv_bfloat16(*pb)[136] = reinterpret_cast<__nv_bfloat16(*)[136]>(dsm_raw + 32768);   // P [32 columns][136]
    __shared__ __align__(8) uint64_t bars[2];
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    // the chunk's K and V rows by TMA (one 2-D box per 64 d; rows past the chunk are the slot's later
    // positions or the next slot's: masked in S, zeroed in V before P V)
    const int crow = grp.slot * a.cache_capacity + j0;
    // a chunk that starts at or after the segment's first new position holds no cached row: all its
    // visible rows are this call's, appended below from K / V -- no cache load at all
    const int seg_past = drows[grp.d0].pad;
    const bool cached = j0 < seg_past;
    if (t == 0) {
        mbar_init(smem_u32(&bars[0]), 1);
        mbar_init(smem_u32(&bars[1]), 1);
        fence_mbar_init();
        if (cached) {
            mbar_expect_tx(smem_u32(&bars[0]), 32768u);
            for (int h = 0; h < 2; ++h)
                tma_load_2d(smem_u32(ksm) + 16384u * h, &a.tmKc, smem_u32(&bars[0]), kvh * 128 + 64 * h, crow);
        }
    }
    // Q^T as the B operand (k = d, n = column): n = 8 nt + lane / 4, k pairs 2 (lane % 4) (+ 8)
    const int gq = lane >> 2, tq = lane & 3;
    uint32_t qb[NT][8][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        const int n = 8 * nt + gq;
        const bool in = n < ncol;
        const int drow = grp.d0 + (in ? n / G : 0);
        const uint32_t *Qh = reinterpret_cast<const uint32_t *>(
            reinterpret_cast<const __nv_bfloat16 *>(a.Q) + ((size_t)drows[drow].row * a.n_heads + kvh * G + n % G) * 128);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            qb[nt][ks][0] = (in && nt < ntiles) ? Qh[8 * ks + tq] : 0u;
            qb[nt][ks][1] = (in && nt < ntiles) ? Qh[8 * ks + 4 + tq] : 0u;
        }
    }
    __syncthreads();   // barrier init visible
    // this call's rows of the segment up to the group's last one (cache positions seg_past ..
    // pos0 + n - 1, the earlier groups' rows included) are not in the cache yet: they are appended
    // by this kernel, not by a separate cache-write launch -- the CTAs of the chunk(s) holding
    // those positions patch the fresh K / V rows of their KV head into the staged chunk and store
    // them into the cache (rows of earlier groups are stored by several groups: the same bytes)
    const int q0 = max(seg_past, j0), q1 = min(grp.pos0 + grp.n, j0 + kDecChunk);
    auto append_rows = [&](const void *src, void *cache, uint8_t *buf) {
        for (int i = t; i < (q1 - q0) * 16; i += blockDim.x) {
            const int pos = q0 + (i >> 4), u = i & 15;
            const int row = drows[grp.d0 + pos - grp.pos0].row;
            const uint4 v = *(reinterpret_cast<const uint4 *>(reinterpret_cast<const __nv_bfloat16 *>(src) +
                                                             ((size_t)row * a.n_kv_heads + kvh) * 128) + u);
            *reinterpret_cast<uint4 *>(buf + dec_sw(pos - j0, u)) = v;
            *(reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(cache) +
                                        (((size_t)grp.slot * a.cache_capacity + pos) * a.n_kv_heads + kvh) * 128) + u) = v;
        }
    };
    if (cached) mbar_wait(smem_u32(&bars[0]), 0);   // K
    if (q0 < q1) {
        append_rows(a.K, a.K_cache, ksm);
        __syncthreads();
    }
    // S^T (keys x columns): warp w takes keys 32 w .. 32 w + 31 (two m16 tiles), 8 k16 steps over d
    float c[2][NT][4] = {};
    {
        const uint32_t kb = smem_u32(ksm);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                uint32_t a0, a1, a2, a3;
                ldsm_x4(kb + dec_sw(32 * warp + 16 * mt + (lane & 15), 2 * ks + (lane >> 4)), a0, a1, a2, a3);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
                    if (nt < ntiles) mma16816(c[mt][nt], a0, a1, a2, a3, qb[nt][ks][0], qb[nt][ks][1]);
            }
    }
    // the chunk's softmax per query column n (row r = n / G sees cache positions <= pos0 + r), in
    // registers: column max and sum over the warp's 32 keys by shuffles (lanes of equal lane % 4),
    // across the 4 warps through shared memory
    __shared__ float red_m[4][kAttnDecCols], red_l[4][kAttnDecCols];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
        if (nt < ntiles)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int n = 8 * nt + 2 * tq + e;
                const int last = min(nk - 1, grp.pos0 + n / G - j0);   // last visible key of the chunk
                float m = -INFINITY;
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int key = 32 * warp + 16 * mt + gq + 8 * h;
                        const float v = key <= last ? c[mt][nt][2 * h + e] * a.scale : -INFINITY;
                        c[mt][nt][2 * h + e] = v;
                        m = fmaxf(m, v);
                    }
                m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
                m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
                m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
                if (gq == 0) red_m[warp][n] = m;
            }
    __syncthreads();   // every warp is past S: K's buffer takes V
    if (t == 0 && cached) {
        fence_proxy_async_smem();   // the K reads (generic) before the async-proxy V writes
        mbar_expect_tx(smem_u32(&bars[1]), 32768u);
        for (int h = 0; h < 2; ++h) tma_load_2d(smem_u32(vsm) + 16384u * h, &a.tmVc, smem_u32(&bars[1]), kvh * 128 + 64 * h, crow);
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
        if (nt < ntiles)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int n = 8 * nt + 2 * tq + e;
                const float M = fmaxf(fmaxf(red_m[0][n], red_m[1][n]), fmaxf(red_m[2][n], red_m[3][n]));
                float l = 0.f;
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const float v = c[mt][nt][2 * h + e];
                        const float p = v > -INFINITY ? __expf(v - M) : 0.f;
                        l += p;
                        pb[n][32 * warp + 16 * mt + gq + 8 * h] = __float2bfloat16_rn(p);
                    }
                l += __shfl_xor_sync(0xffffffffu, l, 4);
                l += __shfl_xor_sync(0xffffffffu, l, 8);
                l += __shfl_xor_sync(0xffffffffu, l, 16);
                if (gq == 0) red_l[warp][n] = l;
            }
    if (cached) mbar_wait(smem_u32(&bars[1]), 0);   // V
    for (int i = nk * 16 + t; i < kDecChunk * 16; i += blockDim.x)   // V rows past the chunk: zero (p = 0 there)
        *reinterpret_cast<uint4 *>(vsm + dec_sw(i >> 4, i & 15)) = make_uint4(0, 0, 0, 0);
    if (q0 < q1) append_rows(a.V, a.V_cache, vsm);
    __syncthreads();
    // the partial records of the columns whose row sees keys of this chunk: {max, sum, o[128]}
    auto rec = [&](int n) -> float * {
        const int r = n / G;
        return (n < ncol && j0 <= grp.pos0 + r)
                   ? a.dpart + ((((size_t)(grp.d0 + r) * a.n_kv_heads + kvh) * a.max_splits + s) * G + n % G) * 130
                   : nullptr;
    };
    if (t < ncol) {
        float *pr = rec(t);
        if (pr) {
            pr[0] = fmaxf(fmaxf(red_m[0][t], red_m[1][t]), fmaxf(red_m[2][t], red_m[3][t]));
            pr[1] = (red_l[0][t] + red_l[1][t]) + (red_l[2][t] + red_l[3][t]);
        }
    }
    // O^T (d x columns) = V^T P: warp w takes d = 32 w .. 32 w + 31 (two m16 tiles), 8 k16 steps over keys
    float o[2][NT][4] = {};
    {
        const uint32_t vb = smem_u32(vsm);
        const int vr = (lane & 7) + ((lane >> 4) & 1) * 8, vc = 4 * warp + ((lane >> 3) & 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            uint32_t b[NT][2];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const uint32_t *pw = reinterpret_cast<const uint32_t *>(&pb[8 * nt + gq][0]);
                b[nt][0] = nt < ntiles ? pw[8 * kk + tq] : 0u;
                b[nt][1] = nt < ntiles ? pw[8 * kk + 4 + tq] : 0u;
            }
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                uint32_t a0, a1, a2, a3;
                ldsm_x4_t(vb + dec_sw(16 * kk + vr, vc + 2 * mt), a0, a1, a2, a3);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
                    if (nt < ntiles) mma16816(o[mt][nt], a0, a1, a2, a3, b[nt][0], b[nt][1]);
            }
        }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
        if (nt < ntiles)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                float *pr = rec(8 * nt + 2 * tq + e);
                if (pr) {
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                        for (int h = 0; h < 2; ++h) pr[2 + 32 * warp + 16 * mt + gq + 8 * h] = o[mt][nt][2 * h + e];
                }
            }
}

// thread (head g, dims 4 q .. 4 q + 3) of decode row rk / n_kv_heads: the splits merged in split
// order.  32 threads per head: every CTA of the launch is resident in one wave
__global__ void __launch_bounds__(256) attn_decode_combine_kernel(const __grid_constant__ AttnArgs a,
                                                                  const __grid_constant__ AttnDecInline dinl) {
    pdl_wait();
    pdl_trigger();
    const int G = a.n_heads / a.n_kv_heads;
    const int rk = blockIdx.x;
    const AttnRow rw = (a.dec_inline ? dinl.drows : a.drows)[rk / a.n_kv_heads];
    const int kvh = rk % a.n_kv_heads;
    const int ns = (rw.pos + 1 + kDecChunk - 1) / kDecChunk;
    const int g = threadIdx.x >> 5, q = threadIdx.x & 31;
    const float *p0 = a.dpart + ((size_t)rk * a.max_splits * G + g) * 130;
    float M = -INFINITY;
#pragma unroll 4
    for (int s = 0; s < ns; ++s) M = fmaxf(M, p0[(size_t)s * G * 130]);
    float l = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (int s = 0; s < ns; ++s) {   // split order
        const float *p = p0 + (size_t)s * G * 130;
        const float w = __expf(p[0] - M);
        l = fmaf(w, p[1], l);
        const float2 o01 = *reinterpret_cast<const float2 *>(p + 2 + 4 * q);   // 8-byte aligned (130 floats per record)
        const float2 o23 = *reinterpret_cast<const float2 *>(p + 4 + 4 * q);
        o[0] = fmaf(w, o01.x, o[0]);
        o[1] = fmaf(w, o01.y, o[1]);
        o[2] = fmaf(w, o23.x, o[2]);
        o[3] = fmaf(w, o23.y, o[3]);
    }
    __nv_bfloat16 *O = reinterpret_cast<__nv_bfloat16 *>(a.O) + ((size_t)rw.row * a.n_heads + kvh * G + g) * 128 + 4 * q;
    const float inv = 1.f / l;
    *reinterpret_cast<uint2 *>(O) = make_uint2(pack_bf16x2(o[0] * inv, o[1] * inv), pack_bf16x2(o[2] * inv, o[3] * inv));
}

}  // namespace

size_t attn_prefill_smem() { return 1024 + kQBytes + 2 * kKVBytes + 2 * kPBytes + 128; }
static_assert(120 + 4 <= 128, "prefill barriers exceed their area");

int launch_attn(const AttnArgs &a, const AttnDecInline &dinl, int n_items, int n_rows, int n_drows, int n_dgroups,
                cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    // the two-tile prefill kernel (even GQA groups) writes the cache rows itself (warp 2)
    const bool fused_rows = n_items && (a.n_heads / a.n_kv_heads) % 2 == 0 && a.n_kv_heads <= 8;
    if (n_rows && !fused_rows) {
        e = launch_pdl(attn_kv_write_kernel, dim3(a.n_cache_rows), dim3(256), 0, st, a);
        if (e != cudaSuccess) return (int)e;
    }
    if (n_items) {
        static bool attr = false;
        if (!attr) {
            e = cudaFuncSetAttribute(attn_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)attn_prefill_smem());
            if (e != cudaSuccess) return (int)e;
            attr = true;
        }
        int sms = 0, dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int group = a.n_heads / a.n_kv_heads;
        if (group % 2 == 0) {   // two query heads of one KV group per CTA
            static bool attr2 = false;
            if (!attr2) {
                e = cudaFuncSetAttribute(attn_prefill2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)attn_prefill2_smem());
                if (e != cudaSuccess) return (int)e;
                attr2 = true;
            }
            const int units = n_items * (a.n_heads / 2);
            e = launch_pdl(attn_prefill2_kernel, dim3(units < sms ? units : sms), dim3(kAT2), attn_prefill2_smem(), st,
                           a, units);
        } else {
            const int units = n_items * a.n_heads;
            e = launch_pdl(attn_prefill_kernel, dim3(units < sms ? units : sms), dim3(kAT), attn_prefill_smem(), st, a,
                           units);
        }
        if (e != cudaSuccess) return (int)e;
    }
    if (n_drows) {
        const dim3 grid(n_dgroups * a.n_kv_heads * a.max_splits);
        static bool dattr = false;
        if (!dattr) {
            cudaFuncSetAttribute(attn_decode_split_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDecSmem);
            cudaFuncSetAttribute(attn_decode_split_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDecSmem);
            cudaFuncSetAttribute(attn_decode_split_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDecSmem);
            cudaFuncSetAttribute(attn_decode_split_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDecSmem);
            dattr = true;
        }
        switch (a.n_heads / a.n_kv_heads) {
            case 1: e = launch_pdl(attn_decode_split_kernel<1>, grid, dim3(128), kDecSmem, st, a, dinl); break;
            case 2: e = launch_pdl(attn_decode_split_kernel<2>, grid, dim3(128), kDecSmem, st, a, dinl); break;
            case 4: e = launch_pdl(attn_decode_split_kernel<4>, grid, dim3(128), kDecSmem, st, a, dinl); break;
            case 8: e = launch_pdl(attn_decode_split_kernel<8>, grid, dim3(128), kDecSmem, st, a, dinl); break;
            default: return (int)cudaErrorInvalidValue;
        }
        if (e != cudaSuccess) return (int)e;
        e = launch_pdl(attn_decode_combine_kernel, dim3(n_drows * a.n_kv_heads), dim3(32 * (a.n_heads / a.n_kv_heads)), 0,
                       st, a, dinl);
    }
    return (int)e;
}

}  // namespace smlm
