// kernels_decf.cu -- fused decode kernel: one launch per pure-decode call.
//
// Same transposed split-K product as smlm_dec_kernel (M = stacked rows [A_u of the batch's
// adapters ; W], N = <= 256 decode rows, K = in split over the CTAs of a cluster), but the split
// partials never leave the chip and the expand happens in the same launch:
//   1. main loop: TMA W (or stacked A_u) rows + the decode rows' X tile -> tcgen05, fp32 in TMEM
//   2. every CTA copies its partial tile [256 m][128 n] into its own shared memory; cluster barrier
//   3. CTA `split` of a cluster reduces decode rows [split*M/ks, (split+1)*M/ks) of the tile by
//      reading the ks partials through DSMEM in split order (deterministic)
//   4. stacked-adapter tiles publish V (per decode row, its own adapter) to global memory and
//      release a counter; W tiles acquire it, then add s * B_u(m) V(m) and store bf16 Y once.
// All CTAs are co-resident (grid <= #SMs, one CTA per SM), and only W tiles wait (on adapter
// tiles, which never wait), so the cross-cluster dependency cannot deadlock.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "device_types.h"
#include "sm100.cuh"

namespace smlm {
using namespace sm100;

namespace {

constexpr int kFThreads = 256;
constexpr uint32_t kFA = 128 * 128;   // 128 rows x 64 k
constexpr uint32_t kFB = 256 * 128;   // <= 256 decode rows x 64 k
constexpr uint32_t kFStage = kFA + kFB;

__device__ __forceinline__ uint32_t f_cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t f_mapa(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}
__device__ __forceinline__ void f_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void f_bf16x8(const uint4 &u, float (&f)[8]) {
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 t = __bfloat1622float2(h[i]);
        f[2 * i] = t.x;
        f[2 * i + 1] = t.y;
    }
}

template <int RP>
__global__ void __launch_bounds__(kFThreads, 1) smlm_decf_kernel(const __grid_constant__ DecFArgs args) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - raw);
    const int ST = args.stages;
    const uint32_t bar = base + ST * kFStage;
    auto full_bar = [&](int s) { return bar + 8u * s; };
    auto empty_bar = [&](int s) { return bar + 8u * (ST + s); };
    const uint32_t acc_full = bar + 16u * ST;
    const uint32_t tmem_slot = acc_full + 8;
    auto a_addr = [&](int s) { return base + s * kFStage; };
    auto b_addr = [&](int s) { return base + s * kFStage + kFA; };
    // the partial tile [256 m][128 n] fp32 (128 KB) reuses the stage buffers after the main loop
    float *part = reinterpret_cast<float *>(base_ptr);
    const uint32_t part_addr = base;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ks = args.ksplit;
    const int split = (int)f_cluster_rank();
    const int tile = blockIdx.x / ks;                 // stacked-adapter tiles first, then W tiles
    const bool vt = tile < args.n_vt;
    const int nt = vt ? 0 : tile - args.n_vt;
    const int a0 = tile * (128 / RP);                 // first adapter of a stacked tile
    const int na = vt ? min(128 / RP, args.n_uniq - a0) : 0;
    const int M = args.m_rows;                        // decode rows (<= 256), padded to 128-multiples
    const int ncol = M > 128 ? 256 : 128;
    const int nkb = args.K / kBK;
    const int q_ = nkb / ks, rm = nkb % ks;
    const int kb0 = split * q_ + min(split, rm), kb1 = kb0 + q_ + (split < rm ? 1 : 0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        mbar_init(acc_full, 1);
        fence_mbar_init();
        tma_prefetch_desc(&args.tmW);
        tma_prefetch_desc(&args.tmX);
    }
    if (warp == 2) tmem_alloc(tmem_slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t *>(base_ptr + (tmem_slot - base));

    if (warp == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(empty_bar(stage), phase ^ 1);
            if (lane == 0) {
                mbar_expect_tx(full_bar(stage), (vt ? (uint32_t)na * RP * 128u : kFA) + (uint32_t)ncol * 128u);
                if (!vt) {
                    tma_load_2d(a_addr(stage), &args.tmW, full_bar(stage), kb * kBK, nt * 128);
                } else {
                    for (int i = 0; i < na; ++i)
                        tma_load_2d(a_addr(stage) + (uint32_t)i * RP * 128u,
                                    &args.slots[args.vt_slots[a0 + i]].tmA, full_bar(stage), kb * kBK, 0);
                }
                for (int t = 0; t * 128 < ncol; ++t)
                    tma_load_2d(b_addr(stage) + 16384u * t, &args.tmX, full_bar(stage), kb * kBK,
                                args.tile_row0[t]);
            }
            __syncwarp();
            if (++stage == ST) { stage = 0; phase ^= 1; }
        }
    } else if (warp == 1) {
        int stage = 0;
        uint32_t phase = 0;
        const uint32_t idesc = ncol == 256 ? idesc_bf16(128, 256, 0, 0) : idesc_bf16(128, 128, 0, 0);
        uint32_t acc_on = 0;
        for (int kb = kb0; kb < kb1; ++kb) {
            mbar_wait(full_bar(stage), phase);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t ab = a_addr(stage), bb = b_addr(stage);
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k) {
                    mma_bf16(tmem_base, smem_desc(ab + 32u * k, 16, 1024, kSw128),
                             smem_desc(bb + 32u * k, 16, 1024, kSw128), idesc, acc_on);
                    acc_on = 1;
                }
                mma_commit(empty_bar(stage));
            }
            __syncwarp();
            if (++stage == ST) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) mma_commit(acc_full);
        __syncwarp();
    }
    // every thread: wait for the accumulator, then warps 4..7 spill it into shared memory
    mbar_wait(acc_full, 0);
    tc_fence_after();
    if (warp >= 4) {
        const int q = warp - 4;
        const int n = q * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        for (int c = 0; c < ncol; c += 32) {
            uint32_t rr[32];
            tmem_ld32(tmem_base + lane_base + c, rr);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) part[(c + j) * 128 + n] = __uint_as_float(rr[j]);
        }
    }
    tc_fence_before();
    f_cluster_sync();   // all partials of the cluster are in shared memory

    // ---- reduction of this CTA's slice of decode rows over the ks partials (DSMEM) ----
    const int m_lo = split * M / ks, m_hi = (split + 1) * M / ks;
    // thread -> (decode rows m_lo + (tid>>5) + 8 i, 4 consecutive tile rows nq)
    const int nq = 4 * (threadIdx.x & 31);
    const int r8 = threadIdx.x >> 5;
    float4 accv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) accv[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < ks; ++s) {
        const uint32_t pb = f_mapa(part_addr, s);
        float4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int m = m_lo + r8 + 8 * i;
            v[i] = m < m_hi ? ld_dsmem_f4(pb + (uint32_t)(m * 128 + nq) * 4u) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            accv[i].x += v[i].x; accv[i].y += v[i].y; accv[i].z += v[i].z; accv[i].w += v[i].w;
        }
    }
    f_cluster_sync();   // peers may now reuse / exit (no more DSMEM reads of their partials)

    if (vt) {
        // publish V for the decode rows whose adapter lives in this stacked tile
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int m = m_lo + r8 + 8 * i;
            if (m >= m_hi) continue;
            const DecRow dr = args.rows[m];
            if (dr.row < 0 || dr.uidx < a0 || dr.uidx >= a0 + na) continue;
            const int jbase = (dr.uidx - a0) * RP;   // this adapter's rows inside the tile
            const float vals[4] = {accv[i].x, accv[i].y, accv[i].z, accv[i].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = nq + e - jbase;
                if (j >= 0 && j < args.r) {
                    args.Vg[(size_t)m * RP + j] = vals[e];
                    if (dr.ft && args.Vsave)
                        reinterpret_cast<__nv_bfloat16 *>(args.Vsave)[(size_t)dr.row * args.r + j] =
                            __float2bfloat16_rn(vals[e]);
                }
            }
        }
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(args.v_done, 1ull);
    } else {
        // stage the slice's row records and V while waiting for the stacked-adapter CTAs
        float *Vs = part;   // [64][RP] fp32, own shared memory (partials no longer needed)
        DecRow *rs = reinterpret_cast<DecRow *>(part + 64 * RP);
        const __nv_bfloat16 **bp = reinterpret_cast<const __nv_bfloat16 **>(rs + 64);
        if (threadIdx.x < m_hi - m_lo) {
            const DecRow dr = args.rows[m_lo + threadIdx.x];
            rs[threadIdx.x] = dr;
            bp[threadIdx.x] = dr.uidx >= 0 ? reinterpret_cast<const __nv_bfloat16 *>(args.slots[args.vt_slots[dr.uidx]].B)
                                           : nullptr;
        }
        if (args.n_vt > 0) {
            if (threadIdx.x == 0) {
                unsigned long long v;
                do {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(args.v_done) : "memory");
                    if (v < args.v_target) __nanosleep(64);
                } while (v < args.v_target);
            }
            __syncthreads();
            for (int e = threadIdx.x; e < (m_hi - m_lo) * RP; e += kFThreads)
                Vs[e] = __ldcg(args.Vg + (size_t)m_lo * RP + e);
        }
        __syncthreads();
        const int n0 = nt * 128;
        __nv_bfloat16 *Y = reinterpret_cast<__nv_bfloat16 *>(args.Y);
#pragma unroll 2
        for (int i = 0; i < 8; ++i) {
            const int ml = r8 + 8 * i;
            if (m_lo + ml >= m_hi) continue;
            const DecRow dr = rs[ml];
            if (dr.row < 0 || n0 + nq >= args.N) continue;
            float4 y = accv[i];
            const __nv_bfloat16 *Bp = bp[ml];
            if (Bp) {
                const __nv_bfloat16 *B = Bp + (size_t)(n0 + nq) * args.r;
                float l[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int jg = 0; jg < RP; jg += 8) {
                    if (jg < args.r) {
                        uint4 bu[4];
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) bu[q4] = __ldg(reinterpret_cast<const uint4 *>(B + (size_t)q4 * args.r + jg));
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            float bf[8];
                            f_bf16x8(bu[q4], bf);
#pragma unroll
                            for (int e = 0; e < 8; ++e) l[q4] = fmaf(bf[e], Vs[ml * RP + jg + e], l[q4]);
                        }
                    }
                }
                y.x += dr.scale * l[0]; y.y += dr.scale * l[1]; y.z += dr.scale * l[2]; y.w += dr.scale * l[3];
            }
            uint2 pk;
            pk.x = pack_bf16x2(y.x, y.y);
            pk.y = pack_bf16x2(y.z, y.w);
            *reinterpret_cast<uint2 *>(Y + (size_t)dr.row * args.N + n0 + nq) = pk;
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 256);
    }
}

template <int RP>
int launch_decf_impl(const DecFArgs &a, cudaStream_t st) {
    auto kern = smlm_decf_kernel<RP>;
    const size_t smem = 1024 + (size_t)a.stages * kFStage + 256;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return (int)e;
        attr_done = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((a.n_vt + a.n_nt) * a.ksplit);
    cfg.blockDim = dim3(kFThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = a.ksplit;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return (int)cudaLaunchKernelEx(&cfg, kern, a);
}

}  // namespace

int launch_decf(const DecFArgs &a, cudaStream_t st) {
    switch (a.r_pad) {
        case 16: return launch_decf_impl<16>(a, st);
        case 32: return launch_decf_impl<32>(a, st);
        case 64: return launch_decf_impl<64>(a, st);
    }
    return (int)cudaErrorInvalidValue;
}

}  // namespace smlm
