#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double mk(uint32_t lo, uint32_t hi) { double x; asm("mov.b64 %0, {%1, %2};" : "=d"(x) : "r"(lo), "r"(hi)); return x; }
template <int K, int MODE>
__global__ void kmix(int it, uint32_t z, uint32_t zm, double c, uint32_t hmask, double* out) {
    uint32_t r[K], H[K]; double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { r[k] = threadIdx.x * 31 + k; H[k] = (threadIdx.x + k) & hmask; acc[k] = 0; }
    for (int i = 0; i < it; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (MODE != 2) r[k] = __viaddmin_u32(r[k], z, r[k] + zm);
                if (MODE != 1) acc[k] = fma(c, mk(MODE == 2 ? (uint32_t)(k + u) : r[k], H[k]), acc[k]);
            }
        }
    }
    double s = 0; uint32_t x = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) { s += acc[k]; x ^= r[k]; }
    if (s == 1.2345 || x == 12345) out[0] = s + x;
}
template <class F> void timeit(const char* name, F f, double units) {
    f(); cudaDeviceSynchronize();
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-36s %8.3f ms %.3e units/s %s\n", name, ms, units / ms * 1e3, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* d; cudaMalloc(&d, 64);
    const int it = 2000;
    for (int occ : {1, 2, 4}) {
        int grid = nsm * occ * 4, T = 256;
        double units = (double)grid * T * it * 4 * 8;
        char nm[64];
        sprintf(nm, "step+dfma K8 blocks/SM=%d", occ * 4);
        timeit(nm, [&] { kmix<8, 0><<<grid, T>>>(it, 123u, 123u - 2147483647u, 0x1p1000, 0u, d); }, units);
        sprintf(nm, "step only K8 blocks/SM=%d", occ * 4);
        timeit(nm, [&] { kmix<8, 1><<<grid, T>>>(it, 123u, 123u - 2147483647u, 0x1p1000, 0u, d); }, units);
        sprintf(nm, "dfma only K8 blocks/SM=%d", occ * 4);
        timeit(nm, [&] { kmix<8, 2><<<grid, T>>>(it, 123u, 123u - 2147483647u, 0x1p1000, 0u, d); }, units);
    }
    return 0;
}
