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
    int r;             // this adapter's rank (<= the pool's; heterogeneous ranks)
    int pad[5];
};
static_assert(sizeof(SlotDev) % 64 == 0, "SlotDev must keep 64-byte alignment of tensor maps");
// The slot table's descriptors are written in global memory only by copy-engine transfers
// (register / unregister: cudaMemcpyAsync on the caller's stream, never a kernel that PDL
// successors overlap), and every kernel reads them only after griddepcontrol.wait: the kernel
// launch that follows the transfer in stream order starts with fresh descriptor caches, so a
// descriptor cached for a slot's previous adapter is never used (no tensormap proxy fence needed;
// that fence is required only for descriptors modified by device code).

// LoRA dropout on FINETUNE rows (Table 5; R13): the keep
// mask of element (t, k) of X [S, in] is drawn from a counter-based hash of (seed, t, k) -- the
// definition synth.dropout_keep implements on the host for the oracle (no shared code):
//   c = t * half_in + k / 2 (uint32), h = lowbias32(lowbias32(c ^ s0) ^ s1),
//   u = k odd ? h >> 16 : h & 0xffff, kept <=> u >= thr;  x~ = kept * x * scale, scale = 1/(1 - p)
struct DropArgs {
    uint32_t thr;       // round(p * 65536); 0 = dropout off
    uint32_t s0, s1;    // seed (low / high 32 bits)
    uint32_t half_in;   // ceil(in / 2): hash counters per row
    float scale;        // 65536 / (65536 - thr)
    int on;
};

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

// one 128-row tile of a CTA pair (cta_group::2): CTA `rank` stages rows [row0, row0 + 128)
struct alignas(16) DevHalf {
    int row0;     // first row (rows past `rows` are masked in the epilogue; TMA zero-fills past S)
    int rows;     // valid rows (0: an empty half -- the pair has a single tile)
    int slot;     // long tile: adapter or -1; short tile: -1 (adapters per block)
    int flags;    // kPairFT: FINETUNE segment; kPairShort: short tile (adapter blocks blk0..blk0+nblk)
    float scale;
    int tile;     // long: index in the tile list (row block of the tile-compact s*V / s*U operand)
    int blk0;     // short: first adapter block (row block of the block-diagonal s*V operand)
    int nblk;     // short: number of adapter blocks
};
// two consecutive tiles of the plan (same segment or not) on one CTA pair
struct alignas(16) DevPair {
    DevHalf h[2];
};
constexpr int kPairFT = 1, kPairShort = 2;

// one projection of a CTA-pair GEMM launch (forward: up to kGemm2MaxProj projections sharing X)
constexpr int kGemm2MaxProj = 3;
struct alignas(64) Gemm2Proj {
    CUtensorMap tmA;    // A operand rows: fwd X [S,in] (shared); bwd dY_p [S,out_p]; box {64,128} SW128
    CUtensorMap tmW;    // fwd: W [out,in] box {64,128} (K-major, CTA rank's half of the n-tile);
                        // bwd: W box {64,64} (MN-major)
    CUtensorMap tmU;    // fwd: block-diagonal s*V of short tiles; bwd: tile-compact s*U; box {r_pad,128}
    CUtensorMap tmV;    // fwd: tile-compact s*V of the long tiles (pre-shrink); box {r_pad,128}
    CUtensorMap tmY;    // fwd: Y [S,N] box {64,128} SW128 (TMA store of a 64-column chunk of a full tile)
    const SlotDev *slots;   // this projection's pool slot table
    void *Y;            // fwd: Y [S,N]; bwd: dX [S,N]
    int N;              // output width (fwd out, bwd in)
    int K;              // reduction length (fwd in, bwd out_p)
    int nt0;            // first global n-tile of this projection
    int u_rows, v_rows; // row extents of tmU / tmV (an A box at that row is all zeros)
    int has_u, has_v;
    int pad;
};

struct Gemm2Args {
    Gemm2Proj proj[kGemm2MaxProj];
    int dbg;                  // measure build only (SMLM_GEMM2_DEBUG): the MMA issuer prints its wait cycles
    DropArgs drop;            // backward: dX = W^T dy + keep * scale * (s A_a^T u) (separate LoRA accumulator)
    const DevPair *pairs;
    const DevBlock *blocks;   // fwd short tiles' adapter blocks
    int n_proj;
    int n_pairs;
    int n_nt;                 // n-tiles over all projections
    int group_m;
    int r;
    int r_pad;
    int stages;
};

// backward: one adapter with fine-tune rows and bound gradient buffers (PAPER.md P:422 masking)
struct GradGroup {
    int slot;
    int tile_begin;  // into the backward tile list (canonical reduction order)
    int n_tiles;
    int r;           // the adapter's rank (row count of dA, row stride of dB)
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
    // forward pre-shrink (vf = 1): tmDY holds X [S,in], the adapter operand is A_a (K-major, tmA),
    // the result is s*V tile-compact in sUt; V_save (unscaled, FINETUNE tiles) when non-NULL
    int vf;
    int r;
    void *Vsave;
    int *ctr;   // per-item split arrival counters (pool-owned, self-resetting) or NULL: separate reduce
    // npj > 1: forward pre-shrink of npj projections sharing X in one pass (npj * r_pad <= 128):
    // projection p's adapters from slots_p[p], its s*V / V_save to sUt_p[p] / Vsave_p[p]
    // backward (vf = 0): also write the tile-compact s*V of the same tiles from V_save (the dB
    // operand of the token contraction), folded into the reduction
    const void *Vsave_in;
    void *sVt;
    int npj;
    const SlotDev *slots_p[4];
    void *sUt_p[4];
    void *Vsave_p[4];
    DropArgs drop;   // forward pre-shrink (vf): LoRA dropout of the FINETUNE tiles' X
};
constexpr int kUCtrMax = 4096;   // items per U / pre-shrink launch that use the in-kernel reduce

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
    int mt_a;           // ceil(in / (128 nh)): column items of dA^T
    int mt_b;           // ceil(out / (128 nh)): column items of dB
    int nh;             // 128-column halves per item (1 or 2)
    int accumulate;
    int stages;
    DropArgs drop;      // dA items: LoRA dropout of X (the mask of the forward), dA scaled by drop.scale
    // fused cross-rank reduction: every dA/dB value is also stored at p + fanout_delta[q]
    // (the same slot of peer rank q's staging buffer, mapped over NVLink), tile by tile
    int n_fanout;
    long long fanout_delta[8];
};

// ------------------------------------------------------------------------------------------
// decode path v3 (kernels_dec3.cu): pure short/decode batches (<= 512 rows), one or several
// projections sharing X (q/k/v, gate/up) in ONE launch.  CTA pairs: M = 256 decode rows (128 per
// CTA), N = 256 W rows, split K with an in-kernel reduce-scatter of the fp32 partials; the shrink
// runs on the otherwise idle epilogue warps during the main loop; the expand is one extra
// K = r_pad block per adapter (block-diagonal s*V slab x B_u rows).
// ------------------------------------------------------------------------------------------
constexpr int kDec3MaxProj = 4;
constexpr int kDec3MaxPairs = 74;
constexpr int kDec3MaxShrinkItems = 64;   // per shrink pair (staged in shared memory)    // one wave of CTA pairs (148 SMs); spin-waits need co-residency

struct alignas(64) Dec3Proj {
    CUtensorMap tmW;        // W_p [out_p, in] box {64,128} SW128 (B operand: 128 W rows per CTA)
    CUtensorMap tmY;        // Y_p [S, out_p] box {32,128} (TMA store of a 32-column chunk)
    CUtensorMap tmSV;       // s*V slabs [n_groups*n_uniq*256, r_pad] bf16 box {r_pad,128} (expand A operand)
    const SlotDev *slots;   // pool p's slot table (tmA: stacked-A tiles; tmBk: expand)
    void *sv;               // slab base (generic pointer; written by the V tiles' epilogues)
    void *Vsave;            // [S, r] bf16 or NULL (FINETUNE rows)
    int out;
    int nt0;                // first W tile of this projection (within a row group)
    int n_wt;               // ceil(out_p / 256)
    int pad[7];
};

struct alignas(16) Dec3RowInfo {   // per batch row
    int uidx;               // index of its adapter among the batch's adapters, -1 = none
    float scale;            // effective s = slot_scale * seg_scale
    int ft;                 // FINETUNE row (V_save)
    int pad;
};

struct Dec3Args {
    CUtensorMap tmX;        // X [S, in] box {64,128} SW128 (A operand: 128 decode rows per CTA)
    Dec3Proj proj[kDec3MaxProj];
    float *kpart;           // split-K partials [items][2 ranks][8 chunks][8 q][128 m] float4
    int *ctr;               // pool-owned self-resetting counters (kernels_dec3.cu)
    unsigned long long *dbg;  // optional per-CTA phase timestamps [grid][16] (SMLM_DEC3_DEBUG)
    int n_proj;
    int n_uniq;
    int n_groups;           // ceil(S / 256)
    int n_wt;               // W tiles per row group (all projections)
    int n_vt;               // V tiles per (row group, projection): ceil(n_uniq * r_pad / 256)
    int ks;                 // split-K factor of the W tiles
    int ks_v;               // split-K factor of the V (stacked-A shrink) tiles
    int n_vpairs;           // CTA pairs on V items (= n_groups * n_proj * n_vt * ks_v), first in the grid
    int n_wpairs;           // CTA pairs on W items (= n_groups * n_wt * ks), after the V items
    int S;
    int K;                  // in
    int r;
    int r_pad;
    int stages;
    int cooperative;        // launch attribute (pool option SMLM_OPT_DEC_COOPERATIVE), host side only
};
// small plans ride in the kernel parameters (no H2D copy in the stream)
constexpr int kDec3InlineSlots = 256;
constexpr int kDec3InlineRows = 512;
struct Dec3Inline {
    int uslot[kDec3InlineSlots];
    Dec3RowInfo rows[kDec3InlineRows];
};
// AdamW step over a flat fp32 parameter buffer (kernels_opt.cu)
struct AdamwArgs {
    float *p, *m, *v, *g;
    uint16_t *pb;        // optional bf16 copy of the updated parameters
    size_t n;
    float decay;         // 1 - lr * weight_decay
    float step_size;     // lr / (1 - beta1^t)
    float inv_bc2_sqrt;  // 1 / sqrt(1 - beta2^t)
    float beta1, beta2, eps, gscale, max_norm;
    int zero_grad;
    const float *partial;   // per-CTA sum(g^2) of the clip pass, or nullptr
    int n_partial;
    // fused cross-rank reduction: the gradient is the sum of n_slots slots
    // g[q * slot_stride + i] in rank order q = 0.. (peer ranks wrote theirs over NVLink); the
    // kernels start once *ready >= ready_target (system-scope counter the peers increment)
    int n_slots;            // 1 = a plain gradient buffer
    size_t slot_stride;     // elements between slots (multiple of 4)
    int zero_slot;          // zero_grad clears only this slot (the caller's own)
    const int *ready;
    int ready_target;
};

// ---- the Alg. 1 attention branch (kernels_attn.cu) ----
constexpr int kAttnDecChunk = 128;   // decode attention: cached keys per split CTA
struct alignas(16) AttnItem {   // prefill kernel: one 128-query block of a FINETUNE / EVAL / PREFILL segment
    int row0;    // first row of the segment
    int len;     // segment length (keys and queries are the segment's own rows)
    int qb;      // query block
    int pad;
};
struct alignas(16) AttnRow {    // a row written to the KV cache (kv-write) / a decode row (decode)
    int row;     // row of Q/K/V
    int slot;    // cache slot (-1: no write)
    int pos;     // cache position of this row (decode: it attends to cache[0 .. pos])
    int pad;     // decode rows: the segment's first new cache position (its rows are appended in-kernel)
};
struct alignas(16) AttnDGroup {   // consecutive decode rows of one DECODE segment (one cache slot)
    int d0;      // first decode row (index into drows)
    int n;       // rows (n * G <= kAttnDecCols query columns)
    int pos0;    // cache position of the first row (row i attends to cache[0 .. pos0 + i])
    int slot;
};
constexpr int kAttnDecCols = 32;   // query columns (rows x GQA heads) of one decode CTA
// a decode plan of up to kAttnDecInline rows / groups rides in the decode kernels' parameters (no
// plan upload launch before them)
constexpr int kAttnDecInline = 256;
struct AttnDecInline {
    AttnRow drows[kAttnDecInline];
    AttnDGroup dgroups[kAttnDecInline];
};
struct AttnArgs {
    CUtensorMap tmQ;   // Q [S, Hq*d] box {64, 128}
    CUtensorMap tmK;   // K [S, Hkv*d] box {64, 128}
    CUtensorMap tmV;   // V [S, Hkv*d] box {64, 64}
    CUtensorMap tmO;   // O [S, Hq*d] box {64, 128} SW128 (TMA store of a full 128-row tile)
    CUtensorMap tmKc;  // K cache [slots * capacity, Hkv*d] box {64, 128} SW128 (decode chunks)
    CUtensorMap tmVc;  // V cache, same
    const AttnItem *items;
    const AttnRow *rows;    // cache writes
    const AttnRow *drows;   // decode rows
    const AttnDGroup *dgroups;   // decode row groups (a CTA reads its chunk of the slot's K / V once for them)
    const void *Q, *K, *V;
    void *O;
    void *K_cache, *V_cache;   // [slots, capacity, Hkv, d] bf16
    int n_heads, n_kv_heads;
    int n_rows;        // cache-write records: rows (attn_kv_write_kernel) or, for the two-tile prefill
                       // kernel (its warp 2 copies them), segments {row0, slot, list offset, length}
    int n_cache_rows;  // rows written to the cache
    int cache_capacity;
    float scale;
    float *dpart;      // decode split partials [drows * n_kv_heads * max_splits][G][130] fp32
    int max_splits;    // ceil(longest decode context / kAttnDecChunk)
    int dec_inline;    // drows / dgroups are in the decode kernels' AttnDecInline parameter
    int dbg;           // measure build only (SMLM_ATTN_DEBUG): the softmax warps print their phase cycles
};

// fused cross-rank gradient reduction: every rank's ready counter (peer-mapped)
constexpr int kMaxRanks = 8;
struct FanoutFlags {
    int *flag[kMaxRanks];
    int n;
};

constexpr int kDec3ChunkBytes = 128 * 32 * 4;   // one 32-column fp32 chunk of a CTA accumulator
constexpr int dec3_counter_ints() { return 2 + 2 * 128 + 62; }

}  // namespace smlm
