// Microbenchmark of inner-loop variants for the linear-form lattice sum
// (tools only; the product kernel is csrc/lq_kernels.cu::k_lin).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -I../../include -I../../paper_2404_08867_b200/csrc lin_variants.cu -o lin_variants
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "lq_device.cuh"

using namespace lq;
__device__ __noinline__ double outer_ni(double a);
#define EPI(a) outer_ni(a)

struct Dim { double c; uint32_t z, zs; };

enum { STEP_VIADDMNMX = 0, STEP_3OP = 1 };

template <int STEP>
__device__ __forceinline__ uint32_t stepv(uint32_t r, uint32_t z, uint32_t zm) {
    if (STEP == STEP_VIADDMNMX) return __viaddmin_u32(r, z, r + zm);
    uint32_t a = r + z, b = r + zm;
    return min(a, b);
}

// P points per thread, CH independent residue chains (chain c handles points c, c+CH, ...)
template <int P, int CH, int STEP, int MINB>
__global__ void __launch_bounds__(256, MINB) kvar(const Dim* __restrict__ dims, int d, uint32_t n, uint64_t npts,
                                                  uint32_t hmask, double* out) {
    __shared__ double sh[8];
    uint32_t H[P];
#pragma unroll
    for (int k = 0; k < P; ++k) H[k] = (threadIdx.x + k) & hmask;
    const int64_t ntiles = (npts + 256 * P - 1) / (256 * P);
    double tot = 0.0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t i0 = (uint32_t)(tile * 256 * P + threadIdx.x * P);
        double acc[P];
#pragma unroll
        for (int p = 0; p < P; ++p) acc[p] = 0.0;
#pragma unroll 1
        for (int j = 0; j < d; ++j) {
            const Dim dm = dims[j];
            const uint32_t zm = dm.z - n;
            uint32_t r[CH];
            r[0] = mulmod_shoup(i0, dm.z, dm.zs, n);
            uint32_t zc = dm.z, zcm = zm;
            if (CH > 1) {
                // stride-CH stepping: increment CH*z mod n
                uint32_t zz = 0;
#pragma unroll
                for (int c = 0; c < CH; ++c) zz = __viaddmin_u32(zz, dm.z, zz + zm);
                zc = zz; zcm = zz - n;
#pragma unroll
                for (int c = 1; c < CH; ++c) r[c] = stepv<STEP>(r[c - 1], dm.z, zm);
            }
#pragma unroll
            for (int p = 0; p < P; p += CH) {
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    acc[p + c] = fma(dm.c, denorm_of(r[c], H[p + c]), acc[p + c]);
                    r[c] = stepv<STEP>(r[c], zc, zcm);
                }
            }
        }
        double s = 0.0;
#pragma unroll
        for (int p = 0; p < P; ++p) s += EPI(acc[p]);
        tot += s;
    }
    tot = block_sum(tot, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = tot;
}


// per-j constants in kernel parameter space (constant bank): uniform operands
struct DimsParam { Dim d[1024]; };

template <int P, int CH, int MINB, int UNR>
__global__ void __launch_bounds__(256, MINB) kpar(const __grid_constant__ DimsParam dims, int d, uint32_t n, uint64_t npts,
                                                  uint32_t hmask, double* out) {
    __shared__ double sh[8];
    uint32_t H[P];
#pragma unroll
    for (int k = 0; k < P; ++k) H[k] = (threadIdx.x + k) & hmask;
    const int64_t ntiles = (npts + 256 * P - 1) / (256 * P);
    double tot = 0.0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t i0 = (uint32_t)(tile * 256 * P + threadIdx.x * P);
        double acc[P];
#pragma unroll
        for (int p = 0; p < P; ++p) acc[p] = 0.0;
#pragma unroll UNR
        for (int j = 0; j < d; ++j) {
            const double c = dims.d[j].c;
            const uint32_t z = dims.d[j].z, zs = dims.d[j].zs;
            const uint32_t zm = z - n;
            uint32_t r[CH];
            r[0] = mulmod_shoup(i0, z, zs, n);
            uint32_t zc = z, zcm = zm;
            if (CH > 1) {
                uint32_t zz = 0;
#pragma unroll
                for (int cc = 0; cc < CH; ++cc) zz = __viaddmin_u32(zz, z, zz + zm);
                zc = zz; zcm = zz - n;
#pragma unroll
                for (int cc = 1; cc < CH; ++cc) r[cc] = __viaddmin_u32(r[cc - 1], z, r[cc - 1] + zm);
            }
#pragma unroll
            for (int p = 0; p < P; p += CH) {
#pragma unroll
                for (int cc = 0; cc < CH; ++cc) {
                    acc[p + cc] = fma(c, denorm_of(r[cc], H[p + cc]), acc[p + cc]);
                    r[cc] = __viaddmin_u32(r[cc], zc, r[cc] + zcm);
                }
            }
        }
        double s = 0.0;
#pragma unroll
        for (int p = 0; p < P; ++p) s += EPI(acc[p]);
        tot += s;
    }
    tot = block_sum(tot, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = tot;
}


// MODE 0: all-uniform; 1: zm in a vector register; 2: z and zm vector; 3: alternate (even p uniform, odd p vector)
template <int P, int MINB, int MODE>
__global__ void __launch_bounds__(256, MINB) kmix(const __grid_constant__ DimsParam dims, int d, uint32_t n, uint64_t npts,
                                                  uint32_t hmask, double* out) {
    __shared__ double sh[8];
    uint32_t H[P];
#pragma unroll
    for (int k = 0; k < P; ++k) H[k] = (threadIdx.x + k) & hmask;
    const uint32_t vz = (threadIdx.x * 7) & hmask;   // opaque per-thread zero
    const int64_t ntiles = (npts + 256 * P - 1) / (256 * P);
    double tot = 0.0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t i0 = (uint32_t)(tile * 256 * P + threadIdx.x * P);
        double acc[P];
#pragma unroll
        for (int p = 0; p < P; ++p) acc[p] = 0.0;
#pragma unroll 1
        for (int j = 0; j < d; ++j) {
            const double c = dims.d[j].c;
            const uint32_t z = dims.d[j].z, zs = dims.d[j].zs;
            const uint32_t zm = z - n;
            const uint32_t zmv = zm + vz;      // vector copy
            const uint32_t zv = z + vz;
            uint32_t r = mulmod_shoup(i0, z, zs, n);
#pragma unroll
            for (int p = 0; p < P; ++p) {
                acc[p] = fma(c, denorm_of(r, H[p]), acc[p]);
                if (MODE == 0) r = __viaddmin_u32(r, z, r + zm);
                else if (MODE == 1) r = __viaddmin_u32(r, z, r + zmv);
                else if (MODE == 2) r = __viaddmin_u32(r, zv, r + zmv);
                else r = (p & 1) ? __viaddmin_u32(r, z, r + zmv) : __viaddmin_u32(r, z, r + zm);
            }
        }
        double s = 0.0;
#pragma unroll
        for (int p = 0; p < P; ++p) s += EPI(acc[p]);
        tot += s;
    }
    tot = block_sum(tot, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = tot;
}


// two dimensions per iteration, each with its own bank of zero registers: two
// independent residue chains and no re-materialised zeros
template <int P, int MINB>
__global__ void __launch_bounds__(256, MINB) kdual(const __grid_constant__ DimsParam dims, int d, uint32_t n, uint64_t npts,
                                                   uint32_t hmask, double* out) {
    __shared__ double sh[8];
    uint32_t H0[P], H1[P];
#pragma unroll
    for (int k = 0; k < P; ++k) { H0[k] = (threadIdx.x + k) & hmask; H1[k] = (threadIdx.x + 3 * k + 1) & hmask; }
    const int64_t ntiles = (npts + 256 * P - 1) / (256 * P);
    double tot = 0.0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t i0 = (uint32_t)(tile * 256 * P + threadIdx.x * P);
        double acc[P];
#pragma unroll
        for (int p = 0; p < P; ++p) acc[p] = 0.0;
        int j = 0;
#pragma unroll 1
        for (; j + 1 < d; j += 2) {
            const double ca = dims.d[j].c, cb = dims.d[j + 1].c;
            const uint32_t za = dims.d[j].z, zb = dims.d[j + 1].z;
            const uint32_t zma = za - n, zmb = zb - n;
            uint32_t ra = mulmod_shoup(i0, za, dims.d[j].zs, n);
            uint32_t rb = mulmod_shoup(i0, zb, dims.d[j + 1].zs, n);
#pragma unroll
            for (int p = 0; p < P; ++p) {
                acc[p] = fma(ca, denorm_of(ra, H0[p]), acc[p]);
                ra = __viaddmin_u32(ra, za, ra + zma);
                acc[p] = fma(cb, denorm_of(rb, H1[p]), acc[p]);
                rb = __viaddmin_u32(rb, zb, rb + zmb);
            }
        }
        for (; j < d; ++j) {
            const double c = dims.d[j].c;
            const uint32_t z = dims.d[j].z, zm = z - n;
            uint32_t r = mulmod_shoup(i0, z, dims.d[j].zs, n);
#pragma unroll
            for (int p = 0; p < P; ++p) {
                acc[p] = fma(c, denorm_of(r, H0[p]), acc[p]);
                r = __viaddmin_u32(r, z, r + zm);
            }
        }
        double s = 0.0;
#pragma unroll
        for (int p = 0; p < P; ++p) s += EPI(acc[p]);
        tot += s;
    }
    tot = block_sum(tot, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = tot;
}


__device__ __noinline__ double outer_ni(double a) { return exp(-fabs(a * 1e-3)); }
template <class K>
void runp(const char* name, K kern, const DimsParam& dp, int d, uint32_t n, uint64_t npts, double* dout, int nsm) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0);
    cudaFuncAttributes at;
    cudaFuncGetAttributes(&at, kern);
    int grid = nsm * per;
    kern<<<grid, 256>>>(dp, d, n, npts, 0u, dout);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        kern<<<grid, 256>>>(dp, d, n, npts, 0u, dout);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = fminf(best, ms);
    }
    std::vector<double> h(grid);
    cudaMemcpy(h.data(), dout, grid * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    for (double v : h) s += v;
    double pd = (double)npts * d;
    printf("%-28s regs=%3d occ=%d grid=%d  %8.3f ms  %.3e pd/s  %.2f TF(3/pd)  sum=%.15e  err=%s\n", name, at.numRegs,
           per, grid, best, pd / best * 1e3, 3.0 * pd / best * 1e-9, s, cudaGetErrorString(cudaGetLastError()));
}

template <class K>
void run(const char* name, K kern, const Dim* dd, int d, uint32_t n, uint64_t npts, double* dout, int nsm) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0);
    cudaFuncAttributes at;
    cudaFuncGetAttributes(&at, kern);
    int grid = nsm * per;
    kern<<<grid, 256>>>(dd, d, n, npts, 0u, dout);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        kern<<<grid, 256>>>(dd, d, n, npts, 0u, dout);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = fminf(best, ms);
    }
    std::vector<double> h(grid);
    cudaMemcpy(h.data(), dout, grid * 8, cudaMemcpyDeviceToHost);
    double s = 0;
    for (double v : h) s += v;
    double pd = (double)npts * d;
    printf("%-28s regs=%3d occ=%d grid=%d  %8.3f ms  %.3e pd/s  %.2f TF(3/pd)  sum=%.15e  err=%s\n", name, at.numRegs,
           per, grid, best, pd / best * 1e3, 3.0 * pd / best * 1e-9, s, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int d = 1000;
    const uint32_t n = 2147483647u;
    const uint64_t npts = 1ull << 27;
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    std::vector<Dim> h(d);
    uint64_t a = 1440510675ull, zz = 1;
    for (int j = 0; j < d; ++j) {
        h[j].z = (uint32_t)zz;
        h[j].zs = (uint32_t)(((uint64_t)zz << 32) / n);
        h[j].c = std::ldexp(0.01 / n, 1074 - 60);
        zz = zz * a % n;
    }
    Dim* dd;
    double* dout;
    cudaMalloc(&dd, d * sizeof(Dim));
    cudaMalloc(&dout, 1 << 20);
    cudaMemcpy(dd, h.data(), d * sizeof(Dim), cudaMemcpyHostToDevice);
    static DimsParam dp;
    for (int j = 0; j < d; ++j) dp.d[j] = h[j];
    runp("PAR P16 CH1 minb2", kpar<16, 1, 2, 1>, dp, d, n, npts, dout, nsm);
    runp("PAR P16 CH1 minb3", kpar<16, 1, 3, 1>, dp, d, n, npts, dout, nsm);
    runp("PAR P16 CH2 minb2", kpar<16, 2, 2, 1>, dp, d, n, npts, dout, nsm);
    runp("PAR P16 CH2 minb3", kpar<16, 2, 3, 1>, dp, d, n, npts, dout, nsm);
    runp("PAR P8 CH2 minb4", kpar<8, 2, 4, 1>, dp, d, n, npts, dout, nsm);
    runp("DUAL P16 minb2", kdual<16, 2>, dp, d, n, npts, dout, nsm);
    runp("DUAL P16 minb3", kdual<16, 3>, dp, d, n, npts, dout, nsm);
    runp("DUAL P8 minb4", kdual<8, 4>, dp, d, n, npts, dout, nsm);
    runp("DUAL P8 minb5", kdual<8, 5>, dp, d, n, npts, dout, nsm);
    runp("DUAL P12 minb3", kdual<12, 3>, dp, d, n, npts, dout, nsm);
    return 0;
}
