// kernels_attn.cu -- the Alg. 1 attention branch: segment-wise
// causal attention for FINETUNE / EVAL / PREFILL rows, KV-cache initialisation for prefills and
// append + attention over the cache for decodes (reading R14, oracle/attention.py).
//
//   attn_kv_write_kernel   : prefill rows -> cache[slot][0..L), decode rows -> cache[slot][past + i]
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

#include <algorithm>

#include "device_types.h"
#include "pdl.cuh"
#include "sm100.cuh"

namespace smlm {
using namespace sm100;

namespace {

constexpr int kAT = 256;                 // prefill: 8 warps (0 TMA, 1 MMA, 2 TMEM alloc, 4-7 softmax)
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
    auto kv_full = [&](int b) { return bar + 56u + 8u * b; };
    auto kv_empty = [&](int b) { return bar + 72u + 8u * b; };
    const uint32_t tmem_slot = bar + 88;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int group = a.n_heads / a.n_kv_heads;
    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        mbar_init(s_full, 1);
        mbar_init(s_free, 128);
        mbar_init(p_full, 128);
        for (int b = 0; b < 2; ++b) {
            mbar_init(o_done(b), 1);
            mbar_init(kv_full(b), 1);
            mbar_init(kv_empty(b), 1);
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
                    mbar_wait(kv_empty(b), ((G >> 1) & 1) ^ 1);
                    mbar_expect_tx(kv_full(b), kKVBytes);
                    const int k0 = it.row0 + j * 128;
                    // K_j: B operand of S = Q K^T, K-major (rows = keys, 128 B of d per row)
                    for (int db = 0; db < 2; ++db)
                        tma_load_2d(kv_s(b) + 16384u * db, &a.tmK, kv_full(b), kvh * 128 + 64 * db, k0);
                    // V_j: B operand of O += P V, MN-major (rows = keys, 64-wide d boxes)
                    for (int kb = 0; kb < 2; ++kb)
                        for (int db = 0; db < 2; ++db)
                            tma_load_2d(kv_s(b) + 32768u + 16384u * kb + 8192u * db, &a.tmV, kv_full(b),
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
            mbar_wait(p_full, Gp & 1);       // P_Gp in smem, O rescaled
            tc_fence_after();
            const int b = Gp & 1;
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t pa = p_s + (uint32_t)b * kPBytes + 16384u * (k >> 2) + 32u * (k & 3);
                    const uint32_t vb = kv_s(b) + 32768u + 16384u * (k >> 2) + 2048u * (k & 3);
                    mma_bf16(O_t, smem_desc(pa, 16, 1024, kSw128), smem_desc(vb, 8192, 1024, kSw128), idesc_o,
                             (!first || k > 0) ? 1u : 0u);
                }
                mma_commit(kv_empty(b));
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
                mbar_wait(kv_full(b), (G >> 1) & 1);
                tc_fence_after();
                if (lane == 0) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const uint32_t off = 16384u * (k >> 2) + 32u * (k & 3);
                        mma_bf16(S_t, smem_desc(q_s + off, 16, 1024, kSw128),
                                 smem_desc(kv_s(b) + off, 16, 1024, kSw128), idesc_s, k > 0);
                    }
                    mma_commit(s_full);
                    if (j == nkb - 1) mma_commit(q_empty);
                }
                __syncwarp();
                if (j > 0) issue_pv(G - 1, j == 1);
            }
            issue_pv(G - 1, nkb == 1);   // the unit's last block
        }
    } else if (warp >= 4) {
        // ---------------- online softmax + epilogue (thread = query row) ----------------
        const int m = threadIdx.x - 128;
        const uint32_t lane_base = (uint32_t)((warp - 4) * 32) << 16;
        const float sl2 = a.scale * 1.4426950408889634f;
        uint8_t *pp = base_ptr + (p_s - base);
        int G = 0;
        for (int w = blockIdx.x; w < n_units; w += gridDim.x) {
            const AttnItem it = a.items[w / a.n_heads];
            const int head = w % a.n_heads, nkb = it.qb + 1;
            const int qi = it.qb * 128 + m;           // query position inside the segment
            float mi = -INFINITY, li = 0.f;           // running max (log2 units) and sum
            for (int j = 0; j < nkb; ++j, ++G) {
                mbar_wait(s_full, G & 1);
                tc_fence_after();
                const int kbase = j * 128;
                // the whole S row into registers, then S is free for S_{G+1} (it overlaps the exps)
                uint32_t sr[128];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t r[32];
                    tmem_ld32(S_t + lane_base + 32u * c, r);
#pragma unroll
                    for (int e = 0; e < 32; ++e) sr[32 * c + e] = r[e];
                }
                tmem_wait_ld();
                tc_fence_before();
                mbar_arrive(s_free);
                // keys visible to this row: kj <= qi and kj < len  <=>  kj - kbase < lim
                const int lim = min(qi + 1, it.len) - kbase;
                float mx = -INFINITY;
#pragma unroll
                for (int e = 0; e < 128; ++e)
                    if (e < lim) mx = fmaxf(mx, __uint_as_float(sr[e]));
                // lazy rescaling: the reference max moves only when the block's max exceeds it by
                // more than 2^8 (probabilities stay <= 256, exact in fp32 sums and bf16-rounded like
                // any other P), so O is rarely rescaled in TMEM
                const float m_new = (mx * sl2 > mi + 8.f) ? mx * sl2 : mi;
                const float alpha = fast_exp2(mi - m_new);   // 0 on the first block (mi = -inf), else 1 unless moved
                const uint32_t pb = G & 1;
                if (G >= 2) mbar_wait(o_done(pb), ((G >> 1) - 1) & 1);   // PV_{G-2} has read P buffer pb
                float sum = 0.f;
                uint8_t *pbuf = pp + pb * kPBytes;
#pragma unroll
                for (int ch = 0; ch < 16; ++ch) {   // 16-byte chunks of 8 keys: chunk ch of key block ch / 8
                    uint32_t pk[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int e = 8 * ch + 2 * q;
                        const float p0 = e < lim ? fast_exp2(__uint_as_float(sr[e]) * sl2 - m_new) : 0.f;
                        const float p1 = e + 1 < lim ? fast_exp2(__uint_as_float(sr[e + 1]) * sl2 - m_new) : 0.f;
                        const __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
                        // the sum uses the rounded probabilities the MMA multiplies V with
                        const float2 pr = __bfloat1622float2(b2);
                        sum += pr.x + pr.y;
                        pk[q] = *reinterpret_cast<const uint32_t *>(&b2);
                    }
                    const int kb = ch >> 3, cc = ch & 7;
                    *reinterpret_cast<uint4 *>(pbuf + kb * 16384 + m * 128 + ((cc ^ (m & 7)) << 4)) =
                        make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
                li = li * alpha + sum;
                if (j > 0) {
                    // P_{G-1} V_{G-1} has landed in O: rescale it (warp-collective tcgen05.ld / st,
                    // so the warp rescales when any of its rows needs it)
                    mbar_wait(o_done((G - 1) & 1), ((G - 1) >> 1) & 1);
                    tc_fence_after();
                    if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
                        for (int c = 0; c < 4; ++c) {
                            uint32_t r[32];
                            tmem_ld32(O_t + lane_base + 32u * c, r);
                            tmem_wait_ld();
#pragma unroll
                            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
                            tmem_st32(O_t + lane_base + 32u * c, r);
                        }
                        tmem_wait_st();
                    }
                }
                mi = m_new;
                fence_proxy_async_smem();   // P (generic stores) -> the MMA (async proxy)
                tc_fence_before();
                mbar_arrive(p_full);
            }
            // epilogue of the unit: O / l -> bf16 rows of O [S, Hq, d]
            mbar_wait(o_done((G - 1) & 1), ((G - 1) >> 1) & 1);
            tc_fence_after();
            const float inv = 1.f / li;
            const bool ok = qi < it.len;
            __nv_bfloat16 *O = reinterpret_cast<__nv_bfloat16 *>(a.O) +
                               ((size_t)(it.row0 + qi) * a.n_heads + head) * 128;
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t r[32];
                tmem_ld32(O_t + lane_base + 32u * c, r);
                tmem_wait_ld();
                if (ok) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 v;
                        v.x = pack_bf16x2(__uint_as_float(r[8 * q + 0]) * inv, __uint_as_float(r[8 * q + 1]) * inv);
                        v.y = pack_bf16x2(__uint_as_float(r[8 * q + 2]) * inv, __uint_as_float(r[8 * q + 3]) * inv);
                        v.z = pack_bf16x2(__uint_as_float(r[8 * q + 4]) * inv, __uint_as_float(r[8 * q + 5]) * inv);
                        v.w = pack_bf16x2(__uint_as_float(r[8 * q + 6]) * inv, __uint_as_float(r[8 * q + 7]) * inv);
                        *reinterpret_cast<uint4 *>(O + 32 * c + 8 * q) = v;
                    }
                }
            }
            tc_fence_before();   // the O reads are ordered before the next unit's p_full
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

// ---- KV-cache writes: row t of K/V [S, Hkv, d] -> cache slot / position (plan: AttnRow) ----
__global__ void __launch_bounds__(256) attn_kv_write_kernel(const AttnArgs a) {
    pdl_wait();
    pdl_trigger();
    const AttnRow rw = a.rows[blockIdx.x];
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

// ---- decode (split-KV): CTA (decode row, KV head, split) scores its 256 cached keys for the G query
// heads of the group (thread per key: the whole 256-byte K row requested at once, so each CTA has
// 64 KB of loads in flight), takes the chunk's softmax statistics, and accumulates P V with 16
// threads per V row (16-byte loads); partial (max, sum, o) per head go to the workspace and
// attn_decode_combine_kernel merges the splits in split order ----
constexpr int kDecChunk = 256;

template <int G>
__global__ void __launch_bounds__(256) attn_decode_split_kernel(const AttnArgs a) {
    pdl_wait();
    pdl_trigger();
    const int s = blockIdx.x % a.max_splits;
    const int rk = blockIdx.x / a.max_splits;
    const AttnRow rw = a.drows[rk / a.n_kv_heads];
    const int kvh = rk % a.n_kv_heads;
    const int L = rw.pos + 1;   // the cache holds the row itself (appended by attn_kv_write_kernel)
    const int j0 = s * kDecChunk;
    if (j0 >= L) return;
    const int nk = min(kDecChunk, L - j0);
    __shared__ float qs[G][128];
    __shared__ float sc[G][kDecChunk];
    __shared__ float red[8][G][128];   // [warp][head][128] partial outputs
    __shared__ float mloc[G];
    const __nv_bfloat16 *Q = reinterpret_cast<const __nv_bfloat16 *>(a.Q) + ((size_t)rw.row * a.n_heads + kvh * G) * 128;
    for (int e = threadIdx.x; e < G * 128; e += blockDim.x) qs[e / 128][e % 128] = __bfloat162float(Q[e]) * a.scale;
    __syncthreads();
    const size_t row_elems = (size_t)a.n_kv_heads * 128;
    const __nv_bfloat16 *Kc = reinterpret_cast<const __nv_bfloat16 *>(a.K_cache) +
                              ((size_t)rw.slot * a.cache_capacity + j0) * row_elems + kvh * 128;
    const __nv_bfloat16 *Vc = reinterpret_cast<const __nv_bfloat16 *>(a.V_cache) +
                              ((size_t)rw.slot * a.cache_capacity + j0) * row_elems + kvh * 128;
    const int t = threadIdx.x;
    if (t < nk) {
        const uint4 *kr = reinterpret_cast<const uint4 *>(Kc + (size_t)t * row_elems);
        uint4 u[16];
#pragma unroll
        for (int v = 0; v < 16; ++v) u[v] = kr[v];
        float acc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = 0.f;
#pragma unroll
        for (int v = 0; v < 16; ++v) {
            const __nv_bfloat162 *h2 = reinterpret_cast<const __nv_bfloat162 *>(&u[v]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 kf = __bfloat1622float2(h2[i]);
                const int d = 8 * v + 2 * i;
#pragma unroll
                for (int g = 0; g < G; ++g) acc[g] = fmaf(kf.x, qs[g][d], fmaf(kf.y, qs[g][d + 1], acc[g]));
            }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) sc[g][t] = acc[g];
    }
    __syncthreads();
    const int warp = t >> 5, lane = t & 31;
    if (warp < G) {   // the chunk's max per head, then p = exp(s - max) in place
        float mx = -INFINITY;
        for (int j = lane; j < nk; j += 32) mx = fmaxf(mx, sc[warp][j]);
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        for (int j = lane; j < nk; j += 32) sc[warp][j] = __expf(sc[warp][j] - mx);
        if (lane == 0) mloc[warp] = mx;
    }
    __syncthreads();
    // P V: thread (key group kq, dims 8 dq .. 8 dq + 7); 16 keys per round, all 16 rounds' loads first
    const int kq = t >> 4, dq = t & 15;
    float o[G][8];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int e = 0; e < 8; ++e) o[g][e] = 0.f;
#pragma unroll 1
    for (int r0 = 0; r0 < 16; r0 += 8) {
        uint4 u[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int j = kq + 16 * (r0 + r);
            u[r] = j < nk ? *reinterpret_cast<const uint4 *>(Vc + (size_t)j * row_elems + 8 * dq) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int j = kq + 16 * (r0 + r);
            if (j < nk) {
                const __nv_bfloat162 *h2 = reinterpret_cast<const __nv_bfloat162 *>(&u[r]);
                float vf[8];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 f2 = __bfloat1622float2(h2[i]);
                    vf[2 * i] = f2.x;
                    vf[2 * i + 1] = f2.y;
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float p = sc[g][j];
#pragma unroll
                    for (int e = 0; e < 8; ++e) o[g][e] = fmaf(p, vf[e], o[g][e]);
                }
            }
        }
    }
    // the two key groups of a warp (lanes l and l + 16 share dims) by a shuffle, then per warp in smem
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int e = 0; e < 8; ++e) o[g][e] += __shfl_xor_sync(0xffffffffu, o[g][e], 16);
    if (lane < 16) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float4 *dst = reinterpret_cast<float4 *>(&red[warp][g][8 * dq]);
            dst[0] = make_float4(o[g][0], o[g][1], o[g][2], o[g][3]);
            dst[1] = make_float4(o[g][4], o[g][5], o[g][6], o[g][7]);
        }
    }
    __syncthreads();
    // partial of this split: [g] {max, sum, o[128]} in fp32, key groups summed in order
    float *part = a.dpart + (((size_t)rk * a.max_splits + s) * G) * 130;
    for (int e = t; e < G * 128; e += blockDim.x) {
        const int g = e / 128, d = e % 128;
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += red[q][g][d];
        part[g * 130 + 2 + d] = acc;
    }
    if (warp < G) {
        float l = 0.f;
        for (int j = lane; j < nk; j += 32) l += sc[warp][j];
#pragma unroll
        for (int off = 16; off; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
        if (lane == 0) {
            part[warp * 130 + 0] = mloc[warp];
            part[warp * 130 + 1] = l;
        }
    }
}

__global__ void __launch_bounds__(128) attn_decode_combine_kernel(const AttnArgs a) {
    pdl_wait();
    pdl_trigger();
    const int G = a.n_heads / a.n_kv_heads;
    const int rk = blockIdx.x;
    const AttnRow rw = a.drows[rk / a.n_kv_heads];
    const int kvh = rk % a.n_kv_heads;
    const int ns = (rw.pos + 1 + kDecChunk - 1) / kDecChunk;
    const int d = threadIdx.x;
    for (int g = 0; g < G; ++g) {
        const float *p0 = a.dpart + ((size_t)rk * a.max_splits * G + g) * 130;
        float M = -INFINITY;
        for (int s = 0; s < ns; ++s) M = fmaxf(M, p0[(size_t)s * G * 130]);
        float l = 0.f, o = 0.f;
        for (int s = 0; s < ns; ++s) {   // split order
            const float *p = p0 + (size_t)s * G * 130;
            const float w = __expf(p[0] - M);
            l = fmaf(w, p[1], l);
            o = fmaf(w, p[2 + d], o);
        }
        __nv_bfloat16 *O = reinterpret_cast<__nv_bfloat16 *>(a.O) + ((size_t)rw.row * a.n_heads + kvh * G + g) * 128;
        O[d] = __float2bfloat16_rn(o / l);
    }
}

}  // namespace

size_t attn_prefill_smem() { return 1024 + kQBytes + 2 * kKVBytes + 2 * kPBytes + 128; }

int launch_attn(const AttnArgs &a, int n_items, int n_rows, int n_drows, int max_dec_len, cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    if (n_rows) {
        e = launch_pdl(attn_kv_write_kernel, dim3(n_rows), dim3(256), 0, st, a);
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
        const int units = n_items * a.n_heads;
        e = launch_pdl(attn_prefill_kernel, dim3(units < sms ? units : sms), dim3(kAT), attn_prefill_smem(), st, a,
                       units);
        if (e != cudaSuccess) return (int)e;
    }
    if (n_drows) {
        const dim3 grid(n_drows * a.n_kv_heads * a.max_splits);
        switch (a.n_heads / a.n_kv_heads) {
            case 1: e = launch_pdl(attn_decode_split_kernel<1>, grid, dim3(256), 0, st, a); break;
            case 2: e = launch_pdl(attn_decode_split_kernel<2>, grid, dim3(256), 0, st, a); break;
            case 4: e = launch_pdl(attn_decode_split_kernel<4>, grid, dim3(256), 0, st, a); break;
            case 8: e = launch_pdl(attn_decode_split_kernel<8>, grid, dim3(256), 0, st, a); break;
            default: return (int)cudaErrorInvalidValue;
        }
        if (e != cudaSuccess) return (int)e;
        e = launch_pdl(attn_decode_combine_kernel, dim3(n_drows * a.n_kv_heads), dim3(128), 0, st, a);
    }
    return (int)e;
}

}  // namespace smlm
