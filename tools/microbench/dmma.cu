// Does FP64 tensor-core MMA (mma.sync m8n8k4 f64, DMMA) run beside DFMA on
// sm_100a, or share the FP64 pipe?  Three launches of one SM-filling grid:
// DFMA chains only, DMMA only, and half the warps of each kind.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

template <int MODE>   // 0 DFMA, 1 DMMA, 2 half/half by warp
__global__ void k(double* out, int iters) {
    const int warp = threadIdx.x >> 5;
    const bool do_mma = MODE == 1 || (MODE == 2 && (warp & 1));
    double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    double c0[2] = {x0, x1}, c1[2] = {x2, x3}, c2[2] = {x4, x5}, c3[2] = {x6, x7};
    const double a = 0.999999, b = 1e-7;
    if (do_mma) {
        for (int i = 0; i < iters; ++i) {
            dmma(c0, a, b); dmma(c1, a, b); dmma(c2, a, b); dmma(c3, a, b);
        }
    } else {
        for (int i = 0; i < iters; ++i) {
            #pragma unroll
            for (int r = 0; r < 4; ++r) {
                x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
                x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 + c0[0] + c0[1] + c1[0] + c1[1] +
                                                 c2[0] + c2[1] + c3[0] + c3[1];
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 4, threads = 256, iters = 4096;
    double* out;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[3] = {"DFMA only", "DMMA only", "half DFMA / half DMMA warps"};
    for (int rep = 0; rep < 2; ++rep)
        for (int mode = 0; mode < 3; ++mode) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(out, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(out, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            // flops: DFMA warps 32 fma x 2 per iter per thread; DMMA warps 4 mma x 8x8x4x2 per iter per warp
            const double warps = blocks * threads / 32.0;
            double fl;
            if (mode == 0) fl = warps * 32 * iters * 32 * 2.0;
            else if (mode == 1) fl = warps * iters * 4 * 512.0;
            else fl = warps / 2 * 32 * iters * 32 * 2.0 + warps / 2 * iters * 4 * 512.0;
            if (rep) printf("%-30s %8.3f ms  %6.2f TFLOP/s\n", names[mode], ms, fl / ms * 1e-9);
        }
    return 0;
}
