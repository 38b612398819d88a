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

template <int RP>
__global__ void __launch_bounds__(256) shrink_partial_kernel(const __nv_bfloat16 *__restrict__ X,
                                                             const SlotDev *__restrict__ slots,
                                                             const DevBlock *__restrict__ blocks,
                                                             const DevShortRow *__restrict__ srows, int in_f,
                                                             int r, float *__restrict__ part) {
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
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k0 = c * kChunk;
    for (int e = threadIdx.x; e < r * (kChunk / 8); e += 256) {
        const int j = e / (kChunk / 8), v = e % (kChunk / 8);
        cp_async16(reinterpret_cast<uint4 *>(As) + e, reinterpret_cast<const uint4 *>(A + (size_t)j * in_f + k0) + v);
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
}

// combine partials in chunk order -> block-diagonal s*V (bf16 [128, RP]) and V_save
template <int RP>
__global__ void __launch_bounds__(256) shrink_combine_kernel(const DevBlock *__restrict__ blocks,
                                                             const DevShortRow *__restrict__ srows, int nch,
                                                             int r, const float *__restrict__ part,
                                                             __nv_bfloat16 *__restrict__ Vbd,
                                                             __nv_bfloat16 *__restrict__ Vsave) {
    pdl_wait();
    pdl_trigger();
    const DevBlock blk = blocks[blockIdx.x];
    __shared__ int idx_of[128];
    __shared__ float vals[128][RP];
    for (int i = threadIdx.x; i < 128; i += blockDim.x) idx_of[i] = -1;
    __syncthreads();
    for (int i = threadIdx.x; i < blk.nrows; i += blockDim.x) idx_of[srows[blk.row_begin + i].pos] = i;
    const float *src = part + (size_t)blockIdx.x * nch * 128 * RP;
    for (int e = threadIdx.x; e < blk.nrows * RP; e += blockDim.x) {
        const int i = e / RP, j = e % RP;
        float v = 0.f;
        if (j < r) {
            float t[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) t[c] = c < nch ? __ldcg(src + (size_t)c * 128 * RP + i * RP + j) : 0.f;
            for (int c = 0; c < nch && c < 16; ++c) v += t[c];   // chunk order
            for (int c = 16; c < nch; ++c) v += __ldcg(src + (size_t)c * 128 * RP + i * RP + j);
        }
        vals[i][j] = v;
    }
    __syncthreads();
    __nv_bfloat16 *dst = Vbd + (size_t)blockIdx.x * 128 * RP;
    for (int e = threadIdx.x; e < 128 * RP; e += blockDim.x) {
        const int p = e / RP, j = e % RP;
        const int i = idx_of[p];
        dst[e] = __float2bfloat16_rn(i < 0 ? 0.f : srows[blk.row_begin + i].scale * vals[i][j]);
    }
    if (Vsave) {
        for (int e = threadIdx.x; e < blk.nrows * r; e += blockDim.x) {
            const int i = e / r, j = e % r;
            const DevShortRow sr = srows[blk.row_begin + i];
            if (sr.ft) Vsave[(size_t)sr.row * r + j] = __float2bfloat16_rn(vals[i][j]);
        }
    }
}

// ------------------------------------------------------------------------------------------
// transposed decode GEMM with split K over the stacked rows [W ; A_stack]
//   item = (row tile of 128 rows of W or of the stacked A_u of the batch's adapters,
//           group of <= 256 decode rows, K split)
//   D[n, m] = sum_{k in split} Rows[n0 + n, k] x_m[k]  -> fp32 partial tile [256 m][128 n]
// ------------------------------------------------------------------------------------------
constexpr int kDThreads = 256;
constexpr uint32_t kDA = 128 * 128;   // 128 rows x 64 k
constexpr uint32_t kDB = 256 * 128;   // up to 256 decode rows x 64 k
constexpr uint32_t kDStage = kDA + kDB;

// item w -> (row tile, decode-row group, K split).  With clusters of C CTAs the C consecutive
// items of a cluster share (split, group) and take C consecutive row tiles, so they can share the
// decode rows' X tile through TMA multicast.  Stacked-adapter tiles come first; tiles past
// n_vt + n_nt (cluster padding) are dummies (nt = -1).
__device__ __forceinline__ void dec_item(const DecArgs &a, int w, int &nt, int &grp, int &split) {
    const int C = a.cmc;
    const int n_all = a.n_vt + a.n_nt;
    const int n_tg = (n_all + C - 1) / C;
    const int rank = w % C;
    int rest = w / C;
    const int tg = rest % n_tg;
    rest /= n_tg;
    grp = rest % a.n_groups;
    split = rest / a.n_groups;
    const int o = tg * C + rank;
    nt = o >= n_all ? -1 : (o < a.n_vt ? a.n_nt + o : o - a.n_vt);   // >= n_nt: stacked adapter rows
}

__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const void *map, uint32_t bar, int c0, int c1,
                                               uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "h"(mask)
        : "memory");
}
__device__ __forceinline__ void mma_commit_mc1(uint32_t bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(bar), "h"(mask)
                 : "memory");
}

template <int RP>
__global__ void __launch_bounds__(kDThreads, 1) smlm_dec_kernel(const __grid_constant__ DecArgs args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
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
            mbar_init(empty_bar(s), args.cmc);   // released by the MMAs of every CTA of the cluster
        }
        mbar_init(accf0 + 0, 1);
        mbar_init(accf0 + 8, 1);
        mbar_init(accf0 + 16, 128);
        mbar_init(accf0 + 24, 128);
        fence_mbar_init();
        tma_prefetch_desc(&args.tmW);
        tma_prefetch_desc(&args.tmX);
        if (args.cmc > 1) tma_prefetch_desc(&args.tmX64);
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    tc_fence_before();
    if (args.cmc > 1)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t *>(base_ptr + (tmem_slot - base));
    pdl_wait();
    // programmatic dependent launch: the reduce grid may start (and park) while this one streams
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int C = args.cmc;
    const int n_tg = (args.n_vt + args.n_nt + C - 1) / C;
    const int total = n_tg * C * args.n_groups * args.ksplit;
    uint32_t crank = 0;
    if (C > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    const uint16_t mc_mask = (uint16_t)((1u << C) - 1u);
    const int nkb = args.K / kBK;
    constexpr int kAdPerTile = 128 / RP;   // adapters per stacked row tile

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
            const int t0 = 2 * grp, nt_in = min(2, args.n_tiles - t0);
            const bool dummy = nt < 0;
            const bool vt = nt >= args.n_nt;
            const int a0 = (nt - args.n_nt) * kAdPerTile;
            const int na = vt ? min(kAdPerTile, args.n_uniq - a0) : 0;
            int kb0, kb1;
            kb_range(split, kb0, kb1);
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(empty_bar(stage), phase ^ 1);
                if (lane == 0) {
                    const uint32_t abytes = dummy ? 0u : (vt ? (uint32_t)na * RP * 128u : kDA);
                    mbar_expect_tx(full_bar(stage), abytes + 16384u * nt_in);
                    if (dummy) {
                    } else if (!vt) {
                        tma_load_2d(a_addr(stage), &args.tmW, full_bar(stage), kb * kBK, nt * 128);
                    } else {
                        for (int i = 0; i < na; ++i)
                            tma_load_2d(a_addr(stage) + (uint32_t)i * RP * 128u, &args.slots[args.vt_slots[a0 + i]].tmA,
                                        full_bar(stage), kb * kBK, 0);
                    }
                    if (C == 1) {
                        for (int t = 0; t < nt_in; ++t)
                            tma_load_2d(b_addr(stage) + 16384u * t, &args.tmX, full_bar(stage), kb * kBK,
                                        args.tiles[t0 + t].row0);
                    } else {
                        // quarter crank of the (<= 256)-row X tile, multicast to the whole cluster
                        for (int qq = (int)crank; qq < 2 * nt_in; qq += C)
                            tma_load_2d_mc(b_addr(stage) + 8192u * qq, &args.tmX64, full_bar(stage), kb * kBK,
                                           args.tiles[t0 + qq / 2].row0 + 64 * (qq & 1), mc_mask);
                    }
                }
                __syncwarp();
                if (++stage == ST) { stage = 0; phase ^= 1; }
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
            const int nt_in = min(2, args.n_tiles - 2 * grp);
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
                    if (C == 1)
                        mma_commit(empty_bar(stage));
                    else
                        mma_commit_mc1(empty_bar(stage), mc_mask);
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
        const int n = q * 32 + lane;               // row inside the row tile (TMEM lane)
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        uint32_t it = 0;
        for (int w = blockIdx.x; w < total; w += gridDim.x) {
            int nt, grp, split;
            dec_item(args, w, nt, grp, split);
            const int nt_in = min(2, args.n_tiles - 2 * grp);
            const int pair = nt * args.n_groups + grp;
            const uint32_t b = it & 1, u = it >> 1;
            mbar_wait(accf0 + 8 * b, u & 1);
            tc_fence_after();
            float *mypart = args.part + ((size_t)pair * args.ksplit + split) * 256 * 128;
            for (int c = 0; c < (nt < 0 ? 0 : 128 * nt_in); c += 32) {
                uint32_t rr[32];
                tmem_ld32(tmem_base + 256u * b + lane_base + c, rr);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; ++j) mypart[(size_t)(c + j) * 128 + n] = __uint_as_float(rr[j]);
            }
            tc_fence_before();
            mbar_arrive(accf0 + 16 + 8 * b);
            ++it;
        }
    }
    if (C > 1)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else
        __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

// ------------------------------------------------------------------------------------------
// reduce + expand: CTA (W row tile nt, decode-row group, 32-row chunk)
//   V[m][j]      = sum_s part[stacked tile of (u(m), j)][s][m][.]       (fixed split order)
//   Y[m][n0+n]   = sum_s part[nt][s][m][n] + s_m * sum_j B_u(m)[n0+n][j] V[m][j]
// ------------------------------------------------------------------------------------------
// CTA (W row tile nt, decode-row group, chunk of 8 decode rows); thread = (row, 4 columns)
template <int RP>
__global__ void __launch_bounds__(256) dec_reduce_kernel(const __grid_constant__ DecArgs args) {
    const int nt = blockIdx.x;
    const int grp = blockIdx.y >> 5, mc = blockIdx.y & 31;
    __shared__ float Vs[8][RP + 1];
    __shared__ DecRow rs[8];
    __shared__ const __nv_bfloat16 *bptr[8];
    const int ks = args.ksplit;
    const size_t tile_elems = 256 * 128;
    if (threadIdx.x < 8) {
        const DecRow dr = args.rows[grp * 256 + mc * 8 + threadIdx.x];
        rs[threadIdx.x] = dr;
        bptr[threadIdx.x] = dr.uidx >= 0 ? reinterpret_cast<const __nv_bfloat16 *>(args.slots[args.vt_slots[dr.uidx]].B)
                                         : nullptr;
    }
    __syncthreads();
    if (rs[0].row < 0 && rs[7].row < 0 && rs[3].row < 0) {
        // fully padded chunk (rows are packed from the start of each tile)
        bool any = false;
        for (int i = 0; i < 8; ++i) any |= rs[i].row >= 0;
        if (!any) return;
    }
    // wait for the GEMM grid (programmatic dependent launch) before touching its partials
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int e = threadIdx.x; e < 8 * RP; e += 256) {
        const int ml = e / RP, j = e % RP;
        const DecRow dr = rs[ml];
        float v = 0.f;
        if (dr.row >= 0 && dr.uidx >= 0 && j < args.r) {
            const int vrow = dr.uidx * RP + j;
            const int pair = (args.n_nt + vrow / 128) * args.n_groups + grp;
            const float *pp = args.part + (size_t)pair * ks * tile_elems + (size_t)(mc * 8 + ml) * 128 + (vrow & 127);
            for (int s0 = 0; s0 < ks; s0 += 8) {
                float t[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) t[u] = s0 + u < ks ? __ldcg(pp + (size_t)(s0 + u) * tile_elems) : 0.f;
#pragma unroll
                for (int u = 0; u < 8; ++u) v += t[u];
            }
            if (nt == 0 && dr.ft && args.Vsave)
                reinterpret_cast<__nv_bfloat16 *>(args.Vsave)[(size_t)dr.row * args.r + j] = __float2bfloat16_rn(v);
        }
        Vs[ml][j] = v;
    }
    __syncthreads();
    // phase 2: warp = decode row, lane = columns n0 + lane + 32 q (q = 0..3): coalesced partial
    // loads, B_u rows read as consecutive 2*r-byte rows across the warp, coalesced bf16 stores
    const int ml = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = nt * 128;
    const DecRow dr = rs[ml];
    if (dr.row < 0) return;
    const int pair = nt * args.n_groups + grp;
    const float *pbase = args.part + (size_t)pair * ks * tile_elems + (size_t)(mc * 8 + ml) * 128 + lane;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int s0 = 0; s0 < ks; s0 += 4) {
        float t[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q)
                t[u][q] = s0 + u < ks ? __ldcg(pbase + (size_t)(s0 + u) * tile_elems + 32 * q) : 0.f;
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] += t[u][q];
    }
    const __nv_bfloat16 *B = bptr[ml];
    if (B) {
        float l[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int jg = 0; jg < RP; jg += 8) {
            if (jg < args.r) {
                uint4 bu[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int n = n0 + lane + 32 * q;
                    bu[q] = n < args.N ? __ldg(reinterpret_cast<const uint4 *>(B + (size_t)n * args.r + jg))
                                       : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    float bf[8];
                    bf16x8_f32(bu[q], bf);
#pragma unroll
                    for (int e = 0; e < 8; ++e) l[q] = fmaf(bf[e], Vs[ml][jg + e], l[q]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] += dr.scale * l[q];
    }
    __nv_bfloat16 *Y = reinterpret_cast<__nv_bfloat16 *>(args.Y) + (size_t)dr.row * args.N;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int n = n0 + lane + 32 * q;
        if (n < args.N) Y[n] = __float2bfloat16_rn(acc[q]);
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
    const int n_tg = (a.n_nt + a.n_vt + a.cmc - 1) / a.cmc;
    const int total = n_tg * a.cmc * a.n_groups * a.ksplit;
    int grid = total < num_sms ? total : num_sms;
    grid -= grid % a.cmc;
    cudaLaunchConfig_t c1 = {};
    c1.gridDim = dim3(grid);
    c1.blockDim = dim3(kDThreads);
    c1.dynamicSmemBytes = smem;
    c1.stream = st;
    cudaLaunchAttribute at1[2];
    at1[0].id = cudaLaunchAttributeClusterDimension;
    at1[0].val.clusterDim.x = a.cmc;
    at1[0].val.clusterDim.y = 1;
    at1[0].val.clusterDim.z = 1;
    at1[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at1[1].val.programmaticStreamSerializationAllowed = 1;
    c1.attrs = at1;
    c1.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&c1, kern, a);
    if (e != cudaSuccess) return (int)e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.n_nt, a.n_groups * 32);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, dec_reduce_kernel<RP>, a);
    return (int)e;
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
    cudaError_t e = cudaSuccess;
    switch (r_pad) {
        case 16:
            e = launch_pdl(shrink_partial_kernel<16>, g1, dim3(256), (16 + kRowsPerPass) * kChunk * 2, st, X, slots, blocks, srows, in_f, r, part);
            if (e != cudaSuccess) return (int)e;
            e = launch_pdl(shrink_combine_kernel<16>, dim3(n_blocks), dim3(256), 0, st, blocks, srows, nch, r, part, Vbd, Vsave);
            break;
        case 32:
            cudaFuncSetAttribute(shrink_partial_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (32 + kRowsPerPass) * kChunk * 2);
            e = launch_pdl(shrink_partial_kernel<32>, g1, dim3(256), (32 + kRowsPerPass) * kChunk * 2, st, X, slots, blocks, srows, in_f, r, part);
            if (e != cudaSuccess) return (int)e;
            e = launch_pdl(shrink_combine_kernel<32>, dim3(n_blocks), dim3(256), 0, st, blocks, srows, nch, r, part, Vbd, Vsave);
            break;
        case 64:
            cudaFuncSetAttribute(shrink_partial_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (64 + kRowsPerPass) * kChunk * 2);
            e = launch_pdl(shrink_partial_kernel<64>, g1, dim3(256), (64 + kRowsPerPass) * kChunk * 2, st, X, slots, blocks, srows, in_f, r, part);
            if (e != cudaSuccess) return (int)e;
            e = launch_pdl(shrink_combine_kernel<64>, dim3(n_blocks), dim3(256), 0, st, blocks, srows, nch, r, part, Vbd, Vsave);
            break;
        default: return (int)cudaErrorInvalidValue;
    }
    return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
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
