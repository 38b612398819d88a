// dropout.cuh -- the LoRA dropout keep mask on the device (R13; device_types.h DropArgs).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "device_types.h"

namespace smlm {

__device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// keep bits of elements (t, k) and (t, k + 1) of X, k even: bit 0 -> k, bit 1 -> k + 1
__device__ __forceinline__ uint32_t drop_keep2(const DropArgs &d, uint32_t t, uint32_t k) {
    const uint32_t h = lowbias32(lowbias32((t * d.half_in + (k >> 1)) ^ d.s0) ^ d.s1);
    return ((h & 0xffffu) >= d.thr ? 1u : 0u) | ((h >> 16) >= d.thr ? 2u : 0u);
}
__device__ __forceinline__ bool drop_keep(const DropArgs &d, uint32_t t, uint32_t k) {
    return (drop_keep2(d, t, k & ~1u) >> (k & 1u)) & 1u;
}

// 8 consecutive bf16 of row t starting at column k0 (even): dropped elements zeroed (the 1/(1-p)
// scale is applied in fp32 where the product is reduced)
__device__ __forceinline__ uint4 drop_mask8(const DropArgs &d, uint32_t t, uint32_t k0, uint4 v) {
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t m = drop_keep2(d, t, k0 + 2u * i);
        w[i] &= ((m & 1u) ? 0x0000ffffu : 0u) | ((m & 2u) ? 0xffff0000u : 0u);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// A TMA-staged SW128 box of `rows` rows x 64 bf16 columns at shared address `box` (1024-B aligned):
// the element of logical row r, column c sits at r*128 + ((c/8) ^ (r%8))*16 + (c%8)*2.  Zero the
// dropped elements; row r of the box is X row t0 + r, its column c is X column k0 + c.  Threads
// [tid, nthr) split the box's 16-byte chunks.
__device__ __forceinline__ void drop_mask_box_sw128(const DropArgs &d, uint8_t *box, int rows, uint32_t t0,
                                                    uint32_t k0, int tid, int nthr) {
    for (int e = tid; e < rows * 8; e += nthr) {
        const int r = e >> 3, pc = e & 7;
        const int lc = pc ^ (r & 7);
        uint4 *p = reinterpret_cast<uint4 *>(box + r * 128 + pc * 16);
        *p = drop_mask8(d, t0 + (uint32_t)r, k0 + 8u * (uint32_t)lc, *p);
    }
}

}  // namespace smlm
