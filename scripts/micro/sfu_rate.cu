// Microbenchmark: per-SM issue rate of ex2.approx.ftz.f32, cvt.rn.bf16x2.f32 (F2FP) and a mix,
// to see whether the softmax's bf16 packing shares the MUFU (XU) pipe with the exps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sfu_rate sfu_rate.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

template <int MODE>
__global__ void k(float *out, int iters, long long *cyc) {
    float x[16];
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0 || MODE == 2) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
            if (MODE == 1 || MODE == 2) {
                if (MODE == 1 || (i & 1)) {
                    uint32_t r;
                    asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[i]), "f"(x[(i + 1) & 15]));
                    acc += r;
                }
            }
            if (MODE == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(x[i]));
        }
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 16; ++i) s += x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    float *out;
    long long *cyc, h;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 8);
    const int iters = 4096;
    const char *names[] = {"ex2", "cvt.bf16x2", "ex2 + cvt per 2", "ffma"};
    for (int mode = 0; mode < 4; ++mode)
        for (int th = 128; th <= 1024; th *= 2) {
            if (mode == 0) k<0><<<148, th>>>(out, iters, cyc);
            if (mode == 1) k<1><<<148, th>>>(out, iters, cyc);
            if (mode == 2) k<2><<<148, th>>>(out, iters, cyc);
            if (mode == 3) k<3><<<148, th>>>(out, iters, cyc);
            cudaDeviceSynchronize();
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            const double ops = (double)iters * 16 * th * (mode == 2 ? 1.0 : 1.0);
            printf("%-16s threads %4d : %.2f lane-ops/clk/SM (%s)\n", names[mode], th, ops / h,
                   mode == 2 ? "counting ex2 only" : "");
        }
    return 0;
}
