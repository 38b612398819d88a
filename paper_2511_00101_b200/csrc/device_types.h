// device_types.h -- records shared by the host API and the kernels.
#pragma once
#include <cuda.h>
#include <stdint.h>

#include "plan.h"

namespace smlm {

constexpr int kBN = 256;   // n-tile width (one tcgen05 M=128 x N=256 fp32 accumulator)
constexpr int kBK = 64;    // k-block: 64 bf16 = one 128-byte swizzle row

// One adapter slot (device copy of the pool's slot table; adapters are
// loaded/unloaded at runtime per linear layer).  The TMA descriptors point at the caller's
// (borrowed) A/B tensors.
struct alignas(64) SlotDev {
    CUtensorMap tmA;   // A [r,in]  box {64, r_pad} SWIZZLE_128B: fwd shrink (K-major), bwd expand (MN-major)
    CUtensorMap tmBn;  // B [out,r] box {r_pad, 256} swizzle(r_pad*2 B): fwd expand operand (K-major)
    CUtensorMap tmBk;  // B [out,r] box {r_pad, 64}  swizzle(r_pad*2 B): bwd U operand (MN-major)
    const void *A;
    const void *B;
    float *dA;
    float *dB;
    float scale;
    int used;
    int pad[6];
};
static_assert(sizeof(SlotDev) % 64 == 0, "SlotDev must keep 64-byte alignment of tensor maps");

struct GemmArgs {
    CUtensorMap tmA;   // X [S,in] (fwd) or dY [S,out] (bwd): box {64,128} SW128
    CUtensorMap tmB;   // W [out,in]: fwd box {64,256} (K-major); bwd box {64,64} (MN-major)
    CUtensorMap tmV;   // fwd short tiles: block-diagonal s*V [nblk*128, r_pad], box {r_pad,128}
    const SlotDev *slots;
    const DevTile *tiles;
    const DevBlock *blocks;
    int n_tiles;
    int K;          // reduction length: in (fwd) / out (bwd)
    int N;          // output width: out (fwd) / in (bwd)
    int n_ntiles;   // ceil(N / 256)
    int r;
    int r_pad;
    int stages;
    int group_m;    // m-tiles per raster group (L2 reuse)
    int has_w;      // fwd: 0 => Y holds the base output, only the LoRA term is added (RMW)
    void *Y;        // fwd: Y [S,out]; bwd: dX [S,in]
    void *Vsave;    // fwd: bf16 [S,r] (FT rows of long tiles, written by n-tile 0)
    void *sUt;      // bwd: bf16 s*U, tile-compact [n_tiles*128, r_pad] (written by n-tile 0)
    int S;
};

// backward: one adapter with fine-tune rows and bound gradient buffers (PAPER.md P:422 masking)
struct GradGroup {
    int slot;
    int tile_begin;  // into the backward tile list (canonical reduction order)
    int n_tiles;
    int pad;
    float *dA;       // [r,in] fp32 or NULL
    float *dB;       // [out,r] fp32 or NULL
};

// token-contraction GEMM (a5): dA_a^T = X^T (sU) and dB_a = dY^T (sV) over a's fine-tune tiles
struct TokArgs {
    CUtensorMap tmX;    // X  [S,in]  box {64,64} SW128 (MN-major A operand)
    CUtensorMap tmDY;   // dY [S,out] box {64,64} SW128
    CUtensorMap tmSU;   // s*U tile-compact [n_tiles*128, r_pad] box {r_pad,64}
    CUtensorMap tmSV;   // s*V tile-compact [n_tiles*128, r_pad] box {r_pad,64}
    const DevTile *tiles;
    const GradGroup *groups;
    int n_groups;
    int in_f;
    int out_f;
    int r;
    int r_pad;
    int mt_a;           // ceil(in/128)
    int mt_b;           // ceil(out/128)
    int accumulate;
    int stages;
};

// decode / short-row GEMM (transposed, split K)
struct DecArgs {
    CUtensorMap tmW;    // W  [out,in] box {64,128} SW128  (A operand: 128 W rows)
    CUtensorMap tmX;    // X  [S,in]   box {64,128} SW128  (B operand: decode rows)
    CUtensorMap tmV;    // block-diagonal s*V [n_blocks*128, r_pad] box {r_pad,128}
    const SlotDev *slots;
    const DevTile *tiles;    // the short tiles (<= 4)
    const DevBlock *blocks;
    int n_tiles;
    int n_groups;       // ceil(n_tiles / 2): <= 256 decode rows per MMA
    int n_nt;           // ceil(out / 128)
    int ksplit;
    int K;
    int N;
    int r_pad;
    int stages;
    void *Y;
    float *part;        // [n_nt*n_groups][ksplit][256][128] fp32 partials
    int *counters;      // [n_nt*n_groups], zeroed before the launch
};

}  // namespace smlm
