// Pipe-throughput probes on B200 for the lattice-sum inner loop (tools only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double mk(uint32_t lo, uint32_t hi) {
    double x;
    asm("mov.b64 %0, {%1, %2};" : "=d"(x) : "r"(lo), "r"(hi));
    return x;
}

// DFMA throughput with operand b either normal (hi != 0) or denormal (hi == 0)
__global__ void k_dfma(int iters, uint32_t hi, double* out) {
    double b = mk(threadIdx.x * 977 + 12345, hi);
    double a0 = 1.0 + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double c = 0.5;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fma(c, b, a0); a1 = fma(c, b, a1); a2 = fma(c, b, a2); a3 = fma(c, b, a3);
            a4 = fma(c, b, a4); a5 = fma(c, b, a5); a6 = fma(c, b, a6); a7 = fma(c, b, a7);
        }
    }
    double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 1.2345) out[0] = s;
}

// DFMA where the *product* is denormal-input but accumulator normal (acc = fma(big, denorm, acc))
__global__ void k_dfma_big(int iters, uint32_t hi, double* out) {
    double b = mk(threadIdx.x * 977 + 12345, hi);
    double a0 = 1.0 + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double c = 0x1p1000;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fma(c, b, a0); a1 = fma(c, b, a1); a2 = fma(c, b, a2); a3 = fma(c, b, a3);
            a4 = fma(c, b, a4); a5 = fma(c, b, a5); a6 = fma(c, b, a6); a7 = fma(c, b, a7);
        }
    }
    double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 1.2345) out[0] = s;
}

// I2F.F64.U32 throughput
__global__ void k_i2f(int iters, uint32_t seed, double* out) {
    uint32_t r0 = threadIdx.x * 7 + seed, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            s0 += (double)r0; s1 += (double)r1; s2 += (double)r2; s3 += (double)r3;
            r0 += 3; r1 += 5; r2 += 7; r3 += 11;
        }
    }
    double s = s0 + s1 + s2 + s3;
    if (s == 1.2345) out[0] = s;
}

// VIADDMNMX throughput: 8 independent chains
__global__ void k_viadd(int iters, uint32_t z, uint32_t zm, uint32_t* out) {
    uint32_t r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = threadIdx.x * 31 + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int k = 0; k < 8; ++k) r[k] = __viaddmin_u32(r[k], z, r[k] + zm);
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= r[k];
    if (s == 12345) out[0] = s;
}

template <class F>
void timeit(const char* name, F launch, double ops_per_launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %8.3f ms  %.3e ops/s  (%s)\n", name, ms, ops_per_launch / ms * 1e3, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int grid = nsm * 8, T = 256, it = 4000;
    double* d;
    cudaMalloc(&d, 64);
    const double n_dfma = (double)grid * T * it * 16 * 8;
    timeit("DFMA normal operand", [&] { k_dfma<<<grid, T>>>(it, 0x3ff00000u, d); }, n_dfma);
    timeit("DFMA denormal operand (c=0.5)", [&] { k_dfma<<<grid, T>>>(it, 0u, d); }, n_dfma);
    timeit("DFMA denormal operand (c=2^1000)", [&] { k_dfma_big<<<grid, T>>>(it, 0u, d); }, n_dfma);
    timeit("DFMA normal operand (c=2^1000)", [&] { k_dfma_big<<<grid, T>>>(it, 0x00100000u, d); }, n_dfma);
    timeit("I2F.F64.U32 + DADD", [&] { k_i2f<<<grid, T>>>(it, 5u, d); }, (double)grid * T * it * 16 * 4);
    timeit("VIADDMNMX (+IADD)", [&] { k_viadd<<<grid, T>>>(it, 12345u, 12345u - 2147483647u, (uint32_t*)d); },
           (double)grid * T * it * 16 * 8);
    return 0;
}
