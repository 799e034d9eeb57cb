#include <cstdio>
#include <cstdint>
__global__ void chain_viadd(int it, uint32_t z, uint32_t zm, uint32_t* out, long long* cyc) {
    uint32_t r = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < it; ++i) {
#pragma unroll
        for (int u = 0; u < 32; ++u) r = __viaddmin_u32(r, z, r + zm);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = r; cyc[0] = t1 - t0; }
}
__global__ void chain_3op(int it, uint32_t z, uint32_t zm, uint32_t* out, long long* cyc) {
    uint32_t r = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < it; ++i) {
#pragma unroll
        for (int u = 0; u < 32; ++u) { uint32_t a = r + z, b = r + zm; r = min(a, b); }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = r; cyc[0] = t1 - t0; }
}
__global__ void chain_dfma(int it, double c, double* out, long long* cyc) {
    double r = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < it; ++i) {
#pragma unroll
        for (int u = 0; u < 32; ++u) r = fma(r, c, 1.0);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = r; cyc[0] = t1 - t0; }
}
int main() {
    uint32_t* o; long long* c; double* od;
    cudaMalloc(&o, 64); cudaMalloc(&c, 64); cudaMalloc(&od, 64);
    long long h; int it = 1000;
    chain_viadd<<<1, 32>>>(it, 123, 123 - 2147483647u, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    chain_viadd<<<1, 32>>>(it, 123, 123 - 2147483647u, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("viadd+viaddmnmx step latency: %.2f cycles\n", (double)h / (it * 32));
    chain_3op<<<1, 32>>>(it, 123, 123 - 2147483647u, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    chain_3op<<<1, 32>>>(it, 123, 123 - 2147483647u, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("3op step latency: %.2f cycles\n", (double)h / (it * 32));
    chain_dfma<<<1, 32>>>(it, 0.999, od, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    chain_dfma<<<1, 32>>>(it, 0.999, od, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("dfma latency: %.2f cycles\n", (double)h / (it * 32));
    return 0;
}
