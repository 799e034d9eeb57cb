// liblq kernels (sm_100a).  See include/lq.h for the ABI and DESIGN.md for
// the roofline of each kernel.
#include <cooperative_groups.h>

#include "lq_device.cuh"
#include "lq_fft.cuh"

namespace cg = cooperative_groups;

namespace lq {

#include "lq_k_points_family.cuh"
#include "lq_k_orbit.cuh"
#include "lq_k_generic.cuh"
#include "lq_k_mdi.cuh"

// ============================================================ reductions
// Fixed pairwise tree over groups of 1024 consecutive values (zero padded):
// out[g] = tree(vals[1024 g .. 1024 g + 1023]).  1024 threads, 4 per thread... here
// 256 threads each fold 4 adjacent values in a fixed order first.
__global__ void __launch_bounds__(kThreads) k_reduce1024(const double* __restrict__ v, int64_t count,
                                                         double* __restrict__ out) {
    __shared__ double sh[8];
    const int64_t g = blockIdx.x;
    const int64_t i = g * 1024 + (int64_t)threadIdx.x * 4;
    double a[4];
    #pragma unroll
    for (int q = 0; q < 4; ++q) a[q] = (i + q < count) ? v[i + q] : 0.0;
    double s = (a[0] + a[1]) + (a[2] + a[3]);
    s = block_sum(s, sh);
    if (threadIdx.x == 0) out[g] = s;
}

// Fixed tree over groups of 256 consecutive values (zero padded): the
// super-chunk partials of layouts with heavy tiles (FFT form: 2 chains, ~12k
// points per tile), whose super-chunks hold 256 tiles.
__global__ void __launch_bounds__(kThreads) k_reduce256(const double* __restrict__ v, int64_t count,
                                                        double* __restrict__ out) {
    __shared__ double sh[8];
    const int64_t i = blockIdx.x * (int64_t)kThreads + threadIdx.x;
    double s = i < count ? v[i] : 0.0;
    s = block_sum(s, sh);
    if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// ============================================================ FP64 probe
__global__ void __launch_bounds__(kThreads) k_fp64_peak(int iters, double seed, double* out) {
    double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
           a6 = a0 + 6, a7 = a0 + 7;
    const double m = 0.999999, c = 1e-7;
    for (int it = 0; it < iters; ++it) {
        #pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
            a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
        }
    }
    double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 12345.678) out[0] = s;   // keep the chains live
}

}  // namespace lq

namespace lq {

// ============================================================ quality measures
// Bernoulli polynomials in numpy's operation order (lattice.py:140-149):
// B2 = (x - 1/2)^2 - 1/12, B4 = ((x - 2) x + 1) x x - 1/30, each op rounded
// (no contraction), so per-point factors match the reference bit for bit.
__device__ __forceinline__ double bern2(double x) {
    const double t = __dsub_rn(x, 0.5);
    return __dsub_rn(__dmul_rn(t, t), 1.0 / 12.0);
}

__device__ __forceinline__ double bern4(double x) {
    return __dsub_rn(__dmul_rn(__dmul_rn(__dadd_rn(__dmul_rn(__dsub_rn(x, 2.0), x), 1.0), x), x), 1.0 / 30.0);
}

// 1 + g (B + beta), as numpy evaluates `1.0 + g * (B + beta)`
__device__ __forceinline__ double bfactor(double B, double g, double beta) {
    return __dadd_rn(1.0, __dmul_rn(g, __dadd_rn(B, beta)));
}

struct QDim {
    uint32_t z, zs;   // z mod n, Shoup constant
    double g;         // weight gamma_j (or the p_alpha coefficient)
};

// sum over points of prod_j (1 + g_j (B_alpha(x_j) + beta)), x_j = RN(r/n)
// exactly: shift_avg_wce_sq (lattice.py:225-245) and p_alpha (:167-181).
// Each product is added to an exact fixed-point tile sum (Fix3, scale 2^S),
// so the total does not depend on the order of the points.
template <int ALPHA>
__global__ void __launch_bounds__(kThreads) k_bprod(const QDim* __restrict__ dims, int d, uint32_t n, double n_d,
                                                    double inv_n, double beta, uint64_t base, uint64_t end, int S,
                                                    Fix3* __restrict__ tile_out) {
    __shared__ Fix3 sh[8];
    const uint64_t i0_64 = base + (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kPts;
    const uint32_t i0 = (uint32_t)i0_64;
    double prod[kPts];
    #pragma unroll
    for (int p = 0; p < kPts; ++p) prod[p] = 1.0;
    for (int j = 0; j < d; ++j) {
        const QDim dm = dims[j];
        const uint32_t zm = dm.z - n;
        uint32_t r = mulmod_shoup(i0 % n, dm.z, dm.zs, n);
        #pragma unroll
        for (int p = 0; p < kPts; ++p) {
            const double x = exact_div((double)r, n_d, inv_n);
            const double B = ALPHA == 2 ? bern2(x) : bern4(x);
            prod[p] = __dmul_rn(prod[p], bfactor(B, dm.g, beta));
            r = step_mod(r, dm.z, zm);
        }
    }
    Fix3 acc = fix_zero();
    #pragma unroll
    for (int p = 0; p < kPts; ++p)
        if (i0_64 + p < end) fix_add(acc, fix_of(prod[p], S));
    acc = fix_block_sum<kThreads>(acc, sh);
    if (threadIdx.x == 0) tile_out[blockIdx.x] = acc;
}

// exact sum of count Fix3 partials (one CTA; integer addition, any order)
__global__ void __launch_bounds__(kThreads) k_fix_reduce(const Fix3* __restrict__ in, int64_t count,
                                                         Fix3* __restrict__ out) {
    __shared__ Fix3 sh[8];
    Fix3 acc = fix_zero();
    for (int64_t i = threadIdx.x; i < count; i += kThreads) fix_add(acc, in[i]);
    acc = fix_block_sum<kThreads>(acc, sh);
    if (threadIdx.x == 0) out[0] = acc;
}

// B2 of every residue: b2[r] = B2(RN(r/n)), as bernoulli_poly(np.arange(n)/n, 2)
// (lattice.py:272).
__global__ void k_b2_table(uint32_t n, double n_d, double inv_n, double* __restrict__ b2) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
        b2[r] = bern2(exact_div((double)r, n_d, inv_n));
}

// CBC base column: base[k] = 1 + gamma_1 (b2[k] + beta) (lattice.py:274)
__global__ void k_cbc_init(uint32_t n, const double* __restrict__ b2, double g, double beta,
                           double* __restrict__ basev) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        basev[k] = bfactor(b2[k], g, beta);
}

// CBC candidate sweep (lattice.py:280-287): for every candidate c,
// val[c] = sum_k base[k] * (1 + g (b2[(k c) mod n] + beta)), summed exactly
// (Fix3, scale 2^S): reflected candidates, whose terms are a permutation of
// each other, tie exactly (the reference sorts its terms for this,
// lattice.py:284).  Persistent CTAs hold the B2 table in shared memory when
// it fits and walk the candidates.
template <bool SMEM>
__global__ void __launch_bounds__(kThreads) k_cbc_eval(uint32_t n, const double* __restrict__ b2g,
                                                       const double* __restrict__ basev, double g, double beta,
                                                       const int64_t* __restrict__ cands, int64_t ncand, int S,
                                                       Fix3* __restrict__ vals) {
    extern __shared__ double b2s[];
    __shared__ Fix3 sh[8];
    const double* b2 = b2g;
    if (SMEM) {
        for (uint32_t r = threadIdx.x; r < n; r += kThreads) b2s[r] = b2g[r];
        __syncthreads();
        b2 = b2s;
    }
    for (int64_t ci = blockIdx.x; ci < ncand; ci += gridDim.x) {
        const uint32_t c = (uint32_t)cands[ci];
        const uint32_t step = (uint32_t)(((uint64_t)c * kThreads) % n), stepm = step - n;
        uint32_t r = (uint32_t)(((uint64_t)threadIdx.x * c) % n);
        Fix3 acc = fix_zero();
        for (uint32_t k = threadIdx.x; k < n; k += kThreads) {
            fix_add(acc, fix_of(__dmul_rn(basev[k], bfactor(b2[r], g, beta)), S));
            r = step_mod(r, step, stepm);
        }
        acc = fix_block_sum<kThreads>(acc, sh);
        if (threadIdx.x == 0) vals[ci] = acc;
    }
}

__global__ void k_cbc_update(uint32_t n, const double* __restrict__ b2, double g, double beta, uint32_t c,
                             double* __restrict__ basev) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint32_t r = (uint32_t)(((uint64_t)k * c) % n);
        basev[k] = __dmul_rn(basev[k], bfactor(b2[r], g, beta));
    }
}

// Korobov search (lattice.py:292-311): for every candidate a, sum over points
// k of prod_j (1 + g_j (b2[k a^j mod n] + beta)), exact (Fix3, scale 2^S);
// residues advance along j by a Shoup modmul with the candidate's constant.
template <bool SMEM>
__global__ void __launch_bounds__(kThreads) k_korobov(uint32_t n, int d, const double* __restrict__ b2g,
                                                      const double* __restrict__ gam, double beta,
                                                      const int64_t* __restrict__ cands, int64_t ncand, int S,
                                                      Fix3* __restrict__ vals) {
    extern __shared__ double b2s[];
    __shared__ Fix3 sh[8];
    const double* b2 = b2g;
    if (SMEM) {
        for (uint32_t r = threadIdx.x; r < n; r += kThreads) b2s[r] = b2g[r];
        __syncthreads();
        b2 = b2s;
    }
    for (int64_t ci = blockIdx.x; ci < ncand; ci += gridDim.x) {
        const uint32_t a = (uint32_t)(cands[ci] % n);
        const uint32_t as = (uint32_t)(((uint64_t)a << 32) / n);
        Fix3 acc = fix_zero();
        for (uint32_t k = threadIdx.x; k < n; k += kThreads) {
            uint32_t r = k;
            double prod = 1.0;
            for (int j = 0; j < d; ++j) {
                prod = __dmul_rn(prod, bfactor(b2[r], __ldg(gam + j), beta));
                r = mulmod_shoup(r, a, as, n);
            }
            fix_add(acc, fix_of(prod, S));
        }
        acc = fix_block_sum<kThreads>(acc, sh);
        if (threadIdx.x == 0) vals[ci] = acc;
    }
}

}  // namespace lq
