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
    CUtensorMap tmV;   // fwd short tiles: block-diagonal s*V [nblk*128, r_pad]; bwd: tile-compact s*U; box {r_pad,128}
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

// a pair of 128-row tiles of one segment processed by a CTA pair (cta_group::2)
struct alignas(16) DevPair {
    int row0;     // first row of the pair (CTA 0: [row0, row0+128), CTA 1: [row0+128, row0+256))
    int rows;     // valid rows of the pair (<= 256; past a segment end rows are masked)
    int slot;     // adapter or -1
    int flags;    // bit 0: FINETUNE segment (V_save); bit 1: short tile (CTA 0 only, per-adapter blocks)
    float scale;
    int tile;     // backward: index of the pair's first tile in the backward tile list (s*U rows)
    int blk0;     // short pair: first adapter block of the tile
    int nblk;     // short pair: number of adapter blocks
};
constexpr int kPairFT = 1, kPairShort = 2;

struct Gemm2Args {
    CUtensorMap tmX;    // fwd: X [S,in] / bwd: dY [S,out]; box {64,128} SW128
    CUtensorMap tmW0;   // fwd: W box {64,128} (CTA 0's half of B); bwd: W box {64,64} (MN-major)
    CUtensorMap tmW1;   // fwd: W box {64,256-r_pad-128} (CTA 1's W rows; A_a stacked below)
    CUtensorMap tmU;    // bwd: tile-compact s*U; fwd: block-diagonal s*V of short tiles; box {r_pad,128}
    const SlotDev *slots;
    const DevPair *pairs;
    const DevBlock *blocks;   // fwd short pairs
    int has_u;                // tmU is valid
    int defer;                // forward: defer each item's expand into the next item's main loop
    int n_pairs;
    int n_ntiles;
    int group_m;
    int K;
    int N;
    int r;
    int r_pad;
    int stages;
    void *Y;
    void *Vsave;
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

// U = dY B_a over the fine-tune tiles (backward), split K over out
struct UArgs {
    CUtensorMap tmDY;      // dY [S,out] box {64,128} SW128
    const SlotDev *slots;
    const DevTile *tiles;  // backward tile list
    const int *items;      // indices of tiles with an adapter
    int n_items;
    int ksplit;
    int K;                 // out
    int r_pad;
    float *part;           // [n_items][ksplit][128][r_pad] fp32
    void *sUt;             // bf16 [n_tiles*128][r_pad]
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

// decode / short-row GEMM (transposed, split K over the stacked rows [W ; A_u of the batch])
struct DecRow {        // one decode row, indexed by group*256 + m (m = position in the group)
    int row;           // batch row, -1 for padding
    int uidx;          // index of its adapter in vt_slots, -1 = base only
    float scale;       // effective s
    int ft;            // FINETUNE row (V_save)
};
struct DecArgs {
    CUtensorMap tmW;    // W [out,in] box {64,128} SW128 (A operand: 128 W rows)
    CUtensorMap tmX;    // X [S,in]   box {64,128} SW128 (B operand: decode rows)
    CUtensorMap tmX64;  // X [S,in]   box {64,64}  SW128 (multicast quarters of the decode rows)
    const SlotDev *slots;
    const DevTile *tiles;    // the short tiles (<= 4)
    const int *vt_slots;     // distinct adapter slots of the batch, ascending
    const DecRow *rows;      // [n_groups*256]
    int n_tiles;
    int n_groups;       // ceil(n_tiles / 2): <= 256 decode rows per MMA
    int n_nt;           // ceil(out / 128) W row tiles
    int n_vt;           // ceil(n_uniq * r_pad / 128) stacked-adapter row tiles
    int n_uniq;
    int ksplit;
    int cmc;            // cluster size sharing the X tile by TMA multicast (1 or 4)
    int K;
    int N;
    int r;
    int r_pad;
    int stages;
    void *Y;
    void *Vsave;
    float *part;        // [(n_nt+n_vt)*n_groups][ksplit][256][128] fp32 partials
};

// fused decode kernel (<= 256 decode rows): DSMEM split-K reduction + in-kernel expand
struct DecFArgs {
    CUtensorMap tmW;    // W [out,in] box {64,128} SW128
    CUtensorMap tmX;    // X [S,in]   box {64,128} SW128
    const SlotDev *slots;
    const int *vt_slots;     // distinct adapter slots of the batch, ascending
    const DecRow *rows;      // [256] per decode row (m = tile*128 + pos)
    int tile_row0[2];        // first batch row of the (<= 2) short tiles
    int n_vt;                // stacked-adapter row tiles
    int n_nt;                // W row tiles (ceil(out/128))
    int n_uniq;
    int ksplit;              // cluster size along K
    int m_rows;              // 128 * number of short tiles
    int K;
    int N;
    int r;
    int r_pad;
    int stages;
    void *Y;
    void *Vsave;
    float *Vg;               // [256][r_pad] fp32 V of every decode row (workspace)
    unsigned long long *v_done;     // pool-owned release counter
    unsigned long long v_target;    // value of *v_done once this call's adapter tiles are published
};

}  // namespace smlm
