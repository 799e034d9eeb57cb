#include <cstdio>
#include <cstdint>
// DFMA paired with one integer op per DFMA; 8 independent chains each.
__device__ __forceinline__ double mk(uint32_t lo, uint32_t hi) { double x; asm("mov.b64 %0, {%1, %2};" : "=d"(x) : "r"(lo), "r"(hi)); return x; }
template <int OP>
__global__ void kp(int it, uint32_t a, uint32_t b, double c, double* out) {
    double acc[8], acc2[8]; uint32_t x[8], H[8], xp[8], H2[8]; const uint32_t bv = b + ((threadIdx.x * 7) & (a >> 20));
#pragma unroll
    for (int k = 0; k < 8; ++k) { acc[k] = threadIdx.x + k; x[k] = threadIdx.x * 3 + k; H[k] = (threadIdx.x + k) & (a >> 20); H2[k] = (threadIdx.x + 2*k+1) & (a >> 20); xp[k] = x[k] + 1; acc2[k] = 0; }
    for (int i = 0; i < it; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (OP < 4) acc[k] = fma(acc[k], c, 1.0);
                if (OP == 0) x[k] = __viaddmin_u32(x[k], a, b);    // VIADDMNMX
                if (OP == 1) x[k] = x[k] + a;                      // VIADD
                if (OP == 2) x[k] = x[k] * a + b;                  // IMAD
                if (OP == 3) x[k] = x[k] ^ (a & b) ^ (x[k] >> 3);  // LOP3/SHF (alu)
                if (OP == 9) { x[k] = __viaddmin_u32(x[k], a, x[k] + b); }
                if (OP == 4) { acc[k] = fma(c, mk(k + u, H[k]), acc[k]); x[k] = __viaddmin_u32(x[k], a, x[k] + b); }
                if (OP == 5) { acc[k] = fma(c, mk(x[k], H[k]), acc[k]); x[k] = __viaddmin_u32(x[k], a, x[k] + b); }
                if (OP == 6) { acc[k] = fma(c, mk(x[k], H[k]), acc[k]); x[k] = __viaddmin_u32(x[k], a, x[k] + bv); }
                if (OP == 7) { acc[k] = fma(c, mk(k + u, H[k]), acc[k]); x[k] = __viaddmin_u32(x[k], a, x[k] + bv); }
                if (OP == 8) { x[k] = __viaddmin_u32(x[k], a, x[k] + bv); }
                if (OP == 10) { acc[k] = fma(c, mk(xp[k], H[k]), acc[k]); xp[k] = x[k]; x[k] = __viaddmin_u32(x[k], a, x[k] + b); }
                if (OP == 11) { acc[k] = fma(c, mk(x[k], H[k]), acc[k]); x[k] = __viaddmin_u32(x[k], a, x[k] + b); acc2[k] = fma(c, mk(x[k], H2[k]), acc2[k]); x[k] = __viaddmin_u32(x[k], a, x[k] + b); }
            }
        }
    }
    double s = 0; uint32_t y = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) { s += acc[k] + acc2[k]; y ^= x[k] ^ xp[k]; }
    if (s == 1.2345 || y == 12345) out[0] = s + y;
}
template <class F> void timeit(const char* name, F f, double units) {
    f(); cudaDeviceSynchronize();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-30s %8.3f ms %.3e pairs/s\n", name, ms, units / ms * 1e3);
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* d; cudaMalloc(&d, 64);
    int grid = nsm * 8, T = 256, it = 4000;
    double units = (double)grid * T * it * 32;
    timeit("DFMA + VIADDMNMX", [&] { kp<0><<<grid, T>>>(it, 3u, 7u, 0.999, d); }, units);
    timeit("DFMA + VIADD", [&] { kp<1><<<grid, T>>>(it, 3u, 7u, 0.999, d); }, units);
    timeit("DFMA + IMAD", [&] { kp<2><<<grid, T>>>(it, 3u, 7u, 0.999, d); }, units);
    timeit("DFMA + LOP3/SHF", [&] { kp<3><<<grid, T>>>(it, 3u, 7u, 0.999, d); }, units);
    timeit("modstep (no dfma)", [&] { kp<9><<<grid, T>>>(it, 3u, 7u, 0.999, d); }, units);
    timeit("modstep + DFMA(indep X)", [&] { kp<4><<<grid, T>>>(it, 3u, 7u, 0x1p1000, d); }, units);
    timeit("modstep + DFMA(X=r)", [&] { kp<5><<<grid, T>>>(it, 3u, 7u, 0x1p1000, d); }, units);
    timeit("IMADstep + DFMA(X=r)", [&] { kp<6><<<grid, T>>>(it, 3u, 7u, 0x1p1000, d); }, units);
    timeit("IMADstep + DFMA(indep)", [&] { kp<7><<<grid, T>>>(it, 3u, 7u, 0x1p1000, d); }, units);
    timeit("IMADstep only", [&] { kp<8><<<grid, T>>>(it, 3u, 7u, 0x1p1000, d); }, units);
    timeit("modstep + DFMA(X=r_prev)", [&] { kp<10><<<grid, T>>>(it, 3u, 7u, 0x1p1000, d); }, units);
    timeit("2x(modstep + DFMA) two accs", [&] { kp<11><<<grid, T>>>(it, 3u, 7u, 0x1p1000, d); }, 2 * units);
    return 0;
}
