// Variants of the product k_lin structure (FamArgs in parameter space, one
// tile per CTA) to explore ILP/occupancy trade-offs (tools only).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cmath>
#include "lq_device.cuh"

using namespace lq;

struct Dim2 { double c; uint32_t z, zs, z2, pad; };   // z2 = 2z mod n
struct Args { int d; uint32_t n; uint64_t base, end; Dim2 dims[1024]; };

__device__ __noinline__ double outer(double a) { return exp(-fabs(a * 1e-3)); }

// P points per thread, CH residue chains (stride CH), MINB CTAs/SM
template <int P, int CH, int MINB>
__global__ void __launch_bounds__(256, MINB) kv(const __grid_constant__ Args a, uint32_t hmask, double* out) {
    __shared__ double sh[8];
    uint32_t H[P];
#pragma unroll
    for (int k = 0; k < P; ++k) H[k] = (threadIdx.x + k) & hmask;
    const uint64_t i0_64 = a.base + (uint64_t)blockIdx.x * 256 * P + (uint64_t)threadIdx.x * P;
    const uint32_t i0 = (uint32_t)i0_64, n = a.n;
    double acc[P];
#pragma unroll
    for (int p = 0; p < P; ++p) acc[p] = 0.0;
#pragma unroll 1
    for (int j = 0; j < a.d; ++j) {
        const double c = a.dims[j].c;
        const uint32_t z = a.dims[j].z, zm = z - n;
        uint32_t r[CH];
        r[0] = mulmod_shoup(i0, z, a.dims[j].zs, n);
        uint32_t zc = z, zcm = zm;
        if (CH >= 2) {
            uint32_t zz = 0;
#pragma unroll
            for (int q = 0; q < CH; ++q) zz = __viaddmin_u32(zz, z, zz + zm);
            zc = zz;
            zcm = zc - n;
#pragma unroll
            for (int q = 1; q < CH; ++q) r[q] = step_mod(r[q - 1], z, zm);
        }
#pragma unroll
        for (int p = 0; p < P; p += CH) {
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                acc[p + q] = fma(c, denorm_of(r[q], H[p + q]), acc[p + q]);
                if (p + CH < P) r[q] = step_mod(r[q], zc, zcm);
            }
        }
    }
    double s = 0.0;
#pragma unroll
    for (int p = 0; p < P; ++p) s += (i0_64 + p < a.end) ? outer(acc[p]) : 0.0;
    s = block_sum(s, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

template <class K>
void run(const char* name, K kern, int P, const Args& a, uint64_t npts, double* dout) {
    cudaFuncAttributes at;
    cudaFuncGetAttributes(&at, kern);
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0);
    unsigned grid = (unsigned)(npts / (256 * P));
    kern<<<grid, 256>>>(a, 0u, dout);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        kern<<<grid, 256>>>(a, 0u, dout);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = fminf(best, ms);
    }
    std::vector<double> h(grid);
    cudaMemcpy(h.data(), dout, grid * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    for (double v : h) s += v;
    double pd = (double)npts * a.d;
    printf("%-22s regs=%3d occ=%d  %8.3f ms  %.3e pd/s  %.2f TF(3/pd)  sum=%.17g %s\n", name, at.numRegs, per, best,
           pd / best * 1e3, 3.0 * pd / best * 1e-9, s, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    static Args a;
    a.d = 1000;
    a.n = 2147483647u;
    a.base = 0;
    const uint64_t npts = 1ull << 28;
    a.end = npts;
    uint64_t zz = 1, A = 1440510675ull;
    for (int j = 0; j < a.d; ++j) {
        a.dims[j].z = (uint32_t)zz;
        a.dims[j].zs = (uint32_t)(((uint64_t)zz << 32) / a.n);
        a.dims[j].z2 = (uint32_t)((2 * zz) % a.n);
        a.dims[j].c = std::ldexp(0.01 / a.n, 1074 - 60);
        zz = zz * A % a.n;
    }
    double* dout;
    cudaMalloc(&dout, 8 << 20);
    run("P24 CH2 minb2", kv<24, 2, 2>, 24, a, npts, dout);
    run("P24 CH3 minb2", kv<24, 3, 2>, 24, a, npts, dout);
    run("P24 CH4 minb2", kv<24, 4, 2>, 24, a, npts, dout);
    run("P30 CH3 minb2", kv<30, 3, 2>, 30, a, npts, dout);
    run("P32 CH4 minb2", kv<32, 4, 2>, 32, a, npts, dout);
    run("P32 CH2 minb1", kv<32, 2, 1>, 32, a, npts, dout);
    run("P20 CH4 minb2", kv<20, 4, 2>, 20, a, npts, dout);
    run("P16 CH4 minb3", kv<16, 4, 3>, 16, a, npts, dout);
    return 0;
}
