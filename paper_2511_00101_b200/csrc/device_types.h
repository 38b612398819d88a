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
    int has_w;      // fwd: 0 => Y holds the base output, only the LoRA term is added (RMW)
    void *Y;        // fwd: Y [S,out]; bwd: dX [S,in]
    void *Vsave;    // fwd: bf16 [S,r] (FT rows of long tiles, written by n-tile 0)
    float *Usave;   // bwd: fp32 [S,r] (FT rows, written by n-tile 0)
    int S;
};

}  // namespace smlm
