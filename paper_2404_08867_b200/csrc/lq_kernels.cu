// liblq kernels (sm_100a).  See include/lq.h for the ABI and DESIGN.md for
// the roofline of each kernel.
#include <cooperative_groups.h>

#include "lq_device.cuh"
#include "lq_fft.cuh"

namespace cg = cooperative_groups;

namespace lq {

// ============================================================ points_block
// out[e], e = row*d + col, = RN(((start+row) * z[col] mod n) / n).
// Flat mapping keeps the HBM writes fully coalesced (the kernel is bound by
// the 8 B/coordinate store); the residue comes from one FP64-estimated
// modmul per element.
__global__ void __launch_bounds__(kThreads) k_points(const uint64_t* __restrict__ z, uint32_t d, uint64_t n,
                                                     double n_d, double inv_n, double ninv_mm,
                                                     uint64_t start, uint64_t n_elem, double* __restrict__ out) {
    for (uint64_t e = blockIdx.x * (uint64_t)kThreads + threadIdx.x; e < n_elem;
         e += (uint64_t)gridDim.x * kThreads) {
        uint64_t row = e / d;
        uint32_t col = (uint32_t)(e - row * d);
        uint64_t i = start + row;
        uint64_t r = mulmod_u64(i % n, __ldg(z + col), n, ninv_mm);
        out[e] = exact_div((double)r, n_d, inv_n);
    }
}

// points_block for n <= 2^31, HBM-write bound: a CTA owns a 64-row x 64-column
// tile; thread (c, g) walks column c for 16 consecutive rows with the
// two-instruction residue step (one Shoup modmul per thread), rounds each
// coordinate exactly (Markstein) into shared memory, and the tile leaves as
// 64-double contiguous row segments written with 16-byte stores (thread pairs
// of columns; both shared-memory phases are conflict-free without padding).
constexpr int kPtRows = 64, kPtCols = 64;
// Blocks run column tile fastest, so the CTAs resident at any moment write
// whole rows of the output (contiguous d*8-byte spans) rather than one 512-byte
// segment out of every row: 4.87 -> 7.35 TB/s at d = 1000.
__global__ void __launch_bounds__(kThreads) k_points_tiled(const uint2* __restrict__ zz, uint32_t d, uint32_t n,
                                                           double n_d, double inv_n, uint64_t start, uint64_t m,
                                                           uint32_t col_tiles, double* __restrict__ out) {
    __shared__ __align__(16) double tile[kPtRows][kPtCols];
    const uint64_t row0 = (uint64_t)(blockIdx.x / col_tiles) * kPtRows;
    const uint32_t col0 = (blockIdx.x % col_tiles) * kPtCols;
    const uint32_t c = threadIdx.x & (kPtCols - 1), g = threadIdx.x / kPtCols;   // 4 row groups of 16
    const uint32_t col = col0 + c;
    if (col < d) {
        const uint2 t = __ldg(zz + col);
        const uint32_t zm = t.x - n;
        uint64_t i0 = start + row0 + (uint64_t)g * 16;
        if (i0 >= n) i0 %= n;                  // full-lattice exports never take the 64-bit division
        uint32_t r = mulmod_shoup((uint32_t)i0, t.x, t.y, n);
        const uint32_t zero = threadIdx.x & 0x80000000u;   // opaque zero (threadIdx.x < 2^31)
        #pragma unroll
        for (int k = 0; k < 16; ++k) {
            // r as a double without I2F (quarter rate): the denormal 2^-1074 r
            // scaled by 2^537 twice, both exact
            const double rd = denorm_of(r, zero) * 0x1p537 * 0x1p537;
            tile[g * 16 + k][c] = exact_div(rd, n_d, inv_n);
            r = step_mod(r, t.x, zm);
        }
    }
    __syncthreads();
    const uint32_t ncols = min(kPtCols, d - col0);
    const uint32_t c2 = 2 * (threadIdx.x & 31);          // column pair of this thread
    // 16-byte stores need an even global element offset: row*d + col0 + c2 is
    // even for every row iff d is even (col0 is a multiple of 64)
    const bool vec = (d & 1u) == 0u && ((uintptr_t)out & 15u) == 0u;
    for (int rr = threadIdx.x / 32; rr < kPtRows; rr += kThreads / 32) {
        const uint64_t row = row0 + rr;
        if (row >= m) break;
        double* dst = out + row * d + col0 + c2;
        if (vec && c2 + 1 < ncols) {
            *reinterpret_cast<double2*>(dst) = *reinterpret_cast<const double2*>(&tile[rr][c2]);
        } else {
            if (c2 < ncols) dst[0] = tile[rr][c2];
            if (c2 + 1 < ncols) dst[1] = tile[rr][c2 + 1];
        }
    }
}

// ============================================================ family sums
// Per-dimension record of the linear-form kernels.
struct LinDim {
    double c;       // beta_j / n * 2^(1074 - sigma): multiplies the denormal 2^-1074 r
    uint32_t z;     // z_j mod n
    uint32_t zs;    // floor(z * 2^32 / n)  (Shoup)
    uint32_t z2;    // 2 z_j mod n: stride of the two interleaved residue chains
    uint32_t z2m;   // z2 - n (mod 2^32), precomputed so it arrives as a uniform operand
};

struct QuadDim {
    double b;       // beta_j * 2^sigma
    double q;       // gamma_j * 2^(2 sigma)
    uint32_t z, zs, z2, z2m;
};

// Family kernels: 256 threads x kFamPts consecutive points per tile, two
// interleaved residue chains per thread (even/odd points, stride 2z): the
// second chain hides the 10-cycle VIADD->VIADDMNMX latency of the first
// (measured 8.1e12 vs 7.6e12 pd/s for 16 points, one chain).
constexpr int kFamPts = 24;
constexpr int kFamTile = kThreads * kFamPts;
#ifndef LQ_QUAD_PTS
#define LQ_QUAD_PTS 24
#endif
constexpr int kQuadPts = LQ_QUAD_PTS;     // points per thread of the Gaussian family
#ifndef LQ_QUADP_PTS
#define LQ_QUADP_PTS 12
#endif
// kind: 0 LIN, 1 QUAD, 2 QUADP (mirror-paired Gaussian: two accumulators per
// point), 3 PROD (product family: a running product and its exponent per point)
constexpr int kProdPts = 16;
__host__ __device__ constexpr int fam_pts(int kind) {
    return kind == 1 ? kQuadPts : kind == 2 ? LQ_QUADP_PTS : kind == 3 ? kProdPts : kFamPts;
}

struct LinParams {
    double alpha, scale, K, A, B, C0, kappa, pw;
};

// Outer functions g(s) of the families' inner sums s:
//   EXP K e^s | SINCOS C0 + A sin s + B cos s | EXPABS K e^(kappa |s|) | POW K s^pw
enum : int { OUT_EXP = 0, OUT_SINCOS = 1, OUT_EXPABS = 2, OUT_POW = 3, OUT_PROG = 4 };

// numpy's b**k for integer k (exprcore.py:466-468; square for k == 2, libm pow
// otherwise; a negative k is 1 / b**(-k), as the reference's pow nodes).
// Integer |k| <= 32 by repeated squaring (at most 9 multiplications, a few ulp
// from libm's pow: far inside the 1e-10 parity bar, ~4x cheaper than pow).
__device__ __forceinline__ double int_pow(double b, double k) {
    const double ak = fabs(k);
    double r;
    if (ak <= 32.0 && ak == rint(ak)) {
        unsigned e = (unsigned)ak;
        double x = b;
        r = 1.0;
        while (e) {
            if (e & 1u) r *= x;
            e >>= 1;
            if (e) x *= x;
        }
    } else {
        r = pow(b, ak);
    }
    return k >= 0.0 ? r : 1.0 / r;
}

template <int OUTER>
__device__ __forceinline__ double outer_val(double s, const LinParams& p) {
    if (OUTER == OUT_EXP) return p.K * exp(s);
    if (OUTER == OUT_EXPABS) return p.K * exp(p.kappa * fabs(s));
    if (OUTER == OUT_POW) return p.K * int_pow(s, p.pw);
    double sn, cs;
    sincos(s, &sn, &cs);
    return p.C0 + p.A * sn + p.B * cs;
}

// Outer functions run once per point (not per point-dim): kept out of line so
// their temporaries do not inflate the register budget of the j-loop.
// Linear families: s = alpha + acc * scale (alpha = 0 for SINCOS, folded into A, B).
template <int OUTER>
__device__ __noinline__ double outer_fn(double acc, const LinParams p) {
    return outer_val<OUTER>(fma(acc, p.scale, p.alpha), p);
}

// Quadratic families: s = alpha + acc.
template <int OUTER>
__device__ __noinline__ double quad_outer(double acc, const LinParams p) {
    return outer_val<OUTER>(p.alpha + acc, p);
}

// A point and its mirror from one range reduction.  With
// s1 = alpha + l, s2 = alphaB - l = D - s1 and y = ym l + ya:
//   EXP     e^s1 + e^s2 = e^y + e^D e^-y                       (y = s1)
//   EXPABS  e^-|y| + e^-|E - y|, y = lambda s1, E = lambda D   (kappa = -lambda <= 0)
//   SINCOS  2 C0 + A' sin y + B' cos y                         (y = s1)
// e^z = 2^k e^r and e^-z = 2^-k e^-r share r, r^2 and the even/odd halves of
// one Taylor polynomial; the constants are split on the host as c 2^k.  The
// host enables it only where every value stays a normal double (|y| <= 700).
struct PairFast {
    double ym, ya, E;
    double c0, c1, c2;   // EXP: e^D; EXPABS: e^-E, e^E; SINCOS: A', B', 2 C0
    double post;         // multiplier after the sum (K; 1 for SINCOS)
    int32_t k0, k1;      // binary exponents of c0, c1
    int32_t on;          // the host enabled the form (else two outer evaluations)
    // centred EXPABS form (pair_expabs_c): u = fma(l, ym, yc), threshold c = |E|/2,
    // e^{-c} = cm 2^ke (cm folded into the exp table), e^{2c} = c2m 2^k2
    int32_t ke, k2;
    double yc, cth, c2m;
};

// v 2^j by exponent arithmetic (v 2^j must be a normal double)
__device__ __forceinline__ double scale2(double v, int j) {
    return __hiloint2double(__double2hiint(v) + (j << 20), __double2loint(v));
}

// f(s1) + f(s2) without the factor q.post (see PairFast)
template <int OUTER>
__device__ __forceinline__ double pair_fast(double l, const PairFast& q) {
    const double y = fma(l, q.ym, q.ya);
    if constexpr (OUTER == OUT_SINCOS) {
        double sn, cs;
        sincos(y, &sn, &cs);
        return fma(q.c0, sn, fma(q.c1, cs, q.c2));
    } else {
        const double z = OUTER == OUT_EXPABS ? -fabs(y) : y;
        const double t = fma(z, 1.4426950408889634, 6755399441055744.0);   // 1.5 2^52: round to integer
        const int k = __double2loint(t);
        const double kf = t - 6755399441055744.0;
        double r = fma(kf, -6.93147180559945286e-01, z);                    // z - k ln2, two-part ln2
        r = fma(kf, -2.319046813846299558e-17, r);
        const double r2 = r * r;
        double e = fma(r2, 2.08767569878681e-09, 2.755731922398589e-07);   // sum r^2i / (2i)!, i <= 6
        e = fma(r2, e, 2.48015873015873e-05);
        e = fma(r2, e, 0.001388888888888889);
        e = fma(r2, e, 0.041666666666666664);
        e = fma(r2, e, 0.5);
        e = fma(r2, e, 1.0);
        double o = fma(r2, 2.505210838544172e-08, 2.7557319223985893e-06);   // sum r^2i / (2i + 1)!, i <= 5
        o = fma(r2, o, 0.0001984126984126984);
        o = fma(r2, o, 0.008333333333333333);
        o = fma(r2, o, 0.16666666666666666);
        o = fma(r2, o, 1.0);
        const double p = fma(r, o, e), m = fma(-r, o, e);                    // e^r, e^-r
        const double f1 = scale2(p, k);
        if constexpr (OUTER == OUT_EXP) {
            return f1 + scale2(m * q.c0, q.k0 - k);
        } else {
            const bool s1 = y >= 0.0, s2 = y <= q.E, same = s1 == s2;
            return f1 + scale2((same ? m : p) * (s2 ? q.c0 : q.c1), (s2 ? q.k0 : q.k1) + (same ? -k : k));
        }
    }
}

// pair_fast with a 2^EB-entry shared table T[j] = (2^(j/2^EB), 2^(-j/2^EB)):
// the range reduction z = (2^EB k + j) ln2/2^EB + r leaves |r| <= ln2/2^(EB+1),
// where the even/odd Taylor halves need degree 4/5 (EB = 6), 6/7 (EB = 4) or
// 8/7 (EB = 3) for a truncation below 4e-17
template <int OUTER>
__device__ __forceinline__ double pair_fast_tab(double l, const PairFast& q, const double2* __restrict__ T) {
    if constexpr (OUTER == OUT_SINCOS) return pair_fast<OUTER>(l, q);
    constexpr int EB = kFftExpBits;
    const double y = fma(l, q.ym, q.ya);
    const double z = OUTER == OUT_EXPABS ? -fabs(y) : y;
    const double t = fma(z, (double)(1 << EB) * 1.4426950408889634, 6755399441055744.0);   // 2^EB/ln2; 1.5 2^52
    const int K = __double2loint(t);
    const double kf = t - 6755399441055744.0;
    double r = fma(kf, -(6.93147180559945286e-01 / (1 << EB)), z);     // ln2/2^EB, two parts
    r = fma(kf, -(2.319046813846299558e-17 / (1 << EB)), r);
    const int k = K >> EB;
    const double2 tj = T[K & ((1 << EB) - 1)];
    const double r2 = r * r;
    double e, o;
    if constexpr (EB >= 6) {
        e = fma(r2, 4.1666666666666664e-02, 0.5);
        o = fma(r2, 8.3333333333333332e-03, 0.16666666666666666);
    } else {
        if constexpr (EB >= 4) {
            e = fma(r2, 1.3888888888888889e-03, 4.1666666666666664e-02);
        } else {
            e = fma(r2, 2.48015873015873e-05, 1.3888888888888889e-03);
            e = fma(r2, e, 4.1666666666666664e-02);
        }
        e = fma(r2, e, 0.5);
        o = fma(r2, 1.984126984126984e-04, 8.3333333333333332e-03);
        o = fma(r2, o, 0.16666666666666666);
    }
    e = fma(r2, e, 1.0);
    o = fma(r2, o, 1.0);
    const double p = fma(r, o, e) * tj.x, m = fma(-r, o, e) * tj.y;     // e^(z - k ln2), e^(-z + k ln2)
    const double f1 = scale2(p, k);
    if constexpr (OUTER == OUT_EXP) {
        return f1 + scale2(m * q.c0, q.k0 - k);
    } else {
        const bool s1 = y >= 0.0, s2 = y <= q.E, same = s1 == s2;
        return f1 + scale2((same ? m : p) * (s2 ? q.c0 : q.c1), (s2 ? q.k0 : q.k1) + (same ? -k : k));
    }
}

// Centred exp-abs pair: with u = y - E/2, w = |u| and c = |E|/2 the point and
// its mirror give e^{-|y|} + e^{-|E-y|} = e^{-c} e^{-w} + (w >= c ? e^{c} e^{-w}
// : e^{-c} e^{w}) -- one range reduction of -w, one comparison, one select.
// T[j] = (2^(j/2^EB) e^{-c}, 2^(-j/2^EB) e^{-c}) (host; normal while c <= 700).
__device__ __forceinline__ double pair_expabs_c(double l, const PairFast& q, const double2* __restrict__ T) {
    constexpr int EB = kFftExpBits;
    static_assert(EB >= 6, "degree-5 polynomial halves need |r| <= ln2/128");
    const double u = fma(l, q.ym, q.yc);
    const double t = fma(-fabs(u), (double)(1 << EB) * 1.4426950408889634, 6755399441055744.0);
    const int K = __double2loint(t);
    const double kf = t - 6755399441055744.0;
    double r = fma(kf, -(6.93147180559945286e-01 / (1 << EB)), -fabs(u));
    r = fma(kf, -(2.319046813846299558e-17 / (1 << EB)), r);
    const int k = K >> EB;
    const double2 tj = T[K & ((1 << EB) - 1)];
    const double r2 = r * r;
    double e = fma(r2, 4.1666666666666664e-02, 0.5);
    double o = fma(r2, 8.3333333333333332e-03, 0.16666666666666666);
    e = fma(r2, e, 1.0);
    o = fma(r2, o, 1.0);
    const double p = fma(r, o, e) * tj.x;    // e^{-w} e^{-c} 2^-k
    const double m = fma(-r, o, e) * tj.y;   // e^{w} e^{-c} 2^k
    const bool ge = fabs(u) >= q.cth;
    const double t2 = ge ? p * q.c2m : m;
    const int e2 = ge ? k + q.k2 : -k;
    return scale2(p, k) + scale2(t2, e2);
}

#ifndef LQ_FFT_CENTRED
#define LQ_FFT_CENTRED 1
#endif

#ifndef LQ_FFT_FULLTILE
#define LQ_FFT_FULLTILE 1
#endif

template <int OUTER>
__device__ __forceinline__ double pair_outer_fft(double l, const PairFast& q, const double2* __restrict__ T) {
#if LQ_FFT_EXPTAB
    if constexpr (OUTER == OUT_EXPABS && LQ_FFT_CENTRED) return pair_expabs_c(l, q, T);
    else return pair_fast_tab<OUTER>(l, q, T);
#else
    return pair_fast<OUTER>(l, q);
#endif
}

__global__ void __launch_bounds__(kThreads) k_fft_twiddles(double2* __restrict__ W) {
    for (int k = blockIdx.x * kThreads + threadIdx.x; k < kFftN; k += gridDim.x * kThreads) {
        double sn, cs;
        sincospi(-2.0 * (double)k / (double)kFftN, &sn, &cs);
        W[k] = make_double2(cs, sn);
    }
}

// Hc = conj(FFT(c_pad)) / N, one CTA of kFftThreads.
__global__ void __launch_bounds__(kFftThreads) k_fft_coeffs(const double* __restrict__ c, int d,
                                                             const double2* __restrict__ W, double2* __restrict__ Hc) {
    extern __shared__ double2 buf[];
    double2* tw = buf + kFftPad;
    fft_load_twiddles(tw, W);
    for (int t = threadIdx.x; t < kFftN; t += kFftThreads) buf[fpad(t)] = make_double2(t < d ? c[t] : 0.0, 0.0);
    __syncthreads();
    fft4096(buf, kFftR == 16 ? tw : W);
    const double inv = 1.0 / (double)kFftN;
    for (int t = threadIdx.x; t < kFftN; t += kFftThreads) {
        const double2 v = buf[fpad(t)];
        Hc[t] = make_double2(v.x * inv, -v.y * inv);
    }
}

// H+- = (conj(FFT(b)) +- conj(FFT(q))) / (2N) for the Gaussian family: b and q
// share one transform (b + i q) and are separated by symmetry.  One CTA.
__global__ void __launch_bounds__(kFftThreads) k_fft_coeffs_pm(const double* __restrict__ b,
                                                                const double* __restrict__ q, int d,
                                                                const double2* __restrict__ W,
                                                                double2* __restrict__ Hp, double2* __restrict__ Hm) {
    extern __shared__ double2 buf[];
    double2* tw = buf + kFftPad;
    fft_load_twiddles(tw, W);
    for (int t = threadIdx.x; t < kFftN; t += kFftThreads)
        buf[fpad(t)] = t < d ? make_double2(b[t], q[t]) : make_double2(0.0, 0.0);
    __syncthreads();
    fft4096(buf, kFftR == 16 ? tw : W);
    const double h = 0.5 / (double)kFftN;
    for (int m = threadIdx.x; m < kFftN; m += kFftThreads) {
        const double2 x = buf[fpad(m)], xr = buf[fpad((kFftN - m) & (kFftN - 1))];
        const double2 sb = make_double2(x.x + xr.x, x.y - xr.y);    // 2 FFT(b)[m]
        const double2 sq = make_double2(x.y + xr.y, xr.x - x.x);    // 2 FFT(q)[m]  ((x - conj xr) / i)
        const double2 hb = make_double2(sb.x * h, -sb.y * h);       // conj(FFT(b)) / N
        const double2 hq = make_double2(sq.x * h, -sq.y * h);       // conj(FFT(q)) / N
        Hp[m] = make_double2(0.5 * (hb.x + hq.x), 0.5 * (hb.y + hq.y));
        Hm[m] = make_double2(0.5 * (hb.x - hq.x), 0.5 * (hb.y - hq.y));
    }
}

// Mirror pairs (x and 1 - x): f at both points from one
// inner sum; `two` is false for the self-mirrored points 0 and n/2.
// Linear: s(1 - x) = (alpha + sum beta) - acc * scale.
template <int OUTER>
__device__ __noinline__ double outer_pair(double acc, const LinParams p, const double alphaB, bool two) {
    const double f1 = outer_val<OUTER>(fma(acc, p.scale, p.alpha), p);
    const double f2 = outer_val<OUTER>(fma(-acc, p.scale, alphaB), p);
    return two ? f1 + f2 : f1;
}

// Quadratic, centred form: s = alphaC + even +- odd at x and 1 - x.
template <int OUTER>
__device__ __noinline__ double quad_pair(double odd, double even, double alphaC, const LinParams p, bool two) {
    const double t = alphaC + even;
    const double f1 = outer_val<OUTER>(t + odd, p), f2 = outer_val<OUTER>(t - odd, p);
    return two ? f1 + f2 : f1;
}

// Per-dimension tables travel in kernel parameter space (constant bank 0) when
// they fit: the j-loop then reads c_j, z_j, zs_j as uniform-register operands
// (LDCU), which frees the vector register file ports for the residue chain
// (measured +30% over LDG-fed operands).
#ifndef LQ_PARAM_DIMS
#define LQ_PARAM_DIMS 1000
#endif
constexpr int kParamDims = LQ_PARAM_DIMS;   // 1000 x 32 B + header < 32764 B of kernel parameters

// Kernel arguments: everything the j-loop reads is warp-uniform and lives in
// kernel parameter space, so ptxas keeps the loop counter and per-dimension
// constants in uniform registers (LDCU + UR operands).
template <class Dim, int N>
struct FamArgs {
    int d;
    uint32_t n;
    uint64_t base, end;
    double alpha, scale, K, A, B, C0, kappa, M;
    double alphaB, bsum, half;   // mirror pairs: alpha + sum beta (QUADP: alpha + C), sum beta, 2^-sigma / 2
    double pw;                   // OUT_POW exponent
    PairFast pf;                 // linear mirror pairs from one range reduction
    Dim dims[N];
};

template <class Dim>
struct FamArgsG {   // d > kParamDims: per-dimension records in global memory
    int d;
    uint32_t n;
    uint64_t base, end;
    double alpha, scale, K, A, B, C0, kappa, M;
    double alphaB, bsum, half;
    double pw;
    PairFast pf;
    const Dim* __restrict__ dims;
};

// Plain lattice sum of f = outer(alpha + <beta, x>), n <= 2^31.
// One CTA per tile of 256 threads x 16 consecutive points.  Dimension-outer
// loop: per (thread, j) one Shoup modmul gives the first residue, then each of
// the 16 points costs VIADD + VIADDMNMX (next residue) + one DFMA with the
// residue read as a denormal -- x_j/n folded into the coefficient, no
// conversion, no division.  tile_out[t] = sum over tile t
// (fixed tree).
enum : int { FAM_LIN = 0, FAM_QUAD = 1, FAM_QUADP = 2, FAM_PROD = 3 };

// Accumulate dimensions [j0, j1) of the family's per-point inner sum for the
// P consecutive points starting at i0 (two residue chains: even/odd points).
//  LIN:  acc += c_j * (2^-1074 r)                 (one DFMA per point-dim)
//  QUAD: xs = (2^-1074 r) * M; acc += (q_j xs + b_j) xs   (three FP64 ops)
//  QUADP: u = (2^-1074 r) * M - 2^-sigma/2 (the centred coordinate x - 1/2);
//        acc += b'_j u, acc2 += q_j u^2  (odd and even parts)
template <int KIND, class Args, int P>
__device__ __forceinline__ void fam_accumulate(const Args& a, uint32_t i0, int j0, int j1, const uint32_t (&H)[P],
                                               double (&acc)[P], double (&acc2)[P]) {
    const uint32_t n = a.n;
    #pragma unroll 1
    for (int j = j0; j < j1; ++j) {
        const uint32_t z = a.dims[j].z, zm = z - n;
        const uint32_t z2 = a.dims[j].z2, z2m = a.dims[j].z2m;
        uint32_t r0 = mulmod_shoup(i0, z, a.dims[j].zs, n);
        uint32_t r1 = step_mod(r0, z, zm);
        if constexpr (KIND == FAM_LIN) {
            const double c = a.dims[j].c;
            // z2 - n as a per-thread (vector) value: the add then issues as
            // IMAD.IADD on the FMA-heavy pipe, which co-issues with the DFMAs
            // better than VIADD with a uniform operand (measured +1.5%)
            const uint32_t z2mv = z2m + H[0];
            #pragma unroll
            for (int p = 0; p < P; p += 2) {
                acc[p] = fma(c, denorm_of(r0, H[p]), acc[p]);
                acc[p + 1] = fma(c, denorm_of(r1, H[p + 1]), acc[p + 1]);
                if (p + 2 < P) {
                    r0 = step_mod(r0, z2, z2mv);
                    r1 = step_mod(r1, z2, z2mv);
                }
            }
        } else if constexpr (KIND == FAM_QUADP) {
            const double b = a.dims[j].b, q = a.dims[j].q, M = a.M, hf = a.half;
            #pragma unroll
            for (int p = 0; p < P; p += 2) {
                const double u0 = fma(denorm_of(r0, H[p]), M, -hf), u1 = fma(denorm_of(r1, H[p + 1]), M, -hf);
                acc[p] = fma(b, u0, acc[p]);
                acc2[p] = fma(q * u0, u0, acc2[p]);
                acc[p + 1] = fma(b, u1, acc[p + 1]);
                acc2[p + 1] = fma(q * u1, u1, acc2[p + 1]);
                if (p + 2 < P) {
                    r0 = step_mod(r0, z2, z2m);
                    r1 = step_mod(r1, z2, z2m);
                }
            }
        } else {
            const double b = a.dims[j].b, q = a.dims[j].q, M = a.M;
            #pragma unroll
            for (int p = 0; p < P; p += 2) {
                const double x0 = denorm_of(r0, H[p]) * M, x1 = denorm_of(r1, H[p + 1]) * M;
                acc[p] = fma(fma(q, x0, b), x0, acc[p]);
                acc[p + 1] = fma(fma(q, x1, b), x1, acc[p + 1]);
                if (p + 2 < P) {
                    r0 = step_mod(r0, z2, z2m);
                    r1 = step_mod(r1, z2, z2m);
                }
            }
        }
    }
}

template <class Args>
__device__ __forceinline__ LinParams lin_params(const Args& a) {
    return LinParams{a.alpha, a.scale, a.K, a.A, a.B, a.C0, a.kappa, a.pw};
}

template <int KIND, int OUTER, class Args>
__device__ __forceinline__ double fam_outer(double acc, const Args& a) {
    if constexpr (KIND == FAM_QUAD) return quad_outer<OUTER>(acc, lin_params(a));
    else return outer_fn<OUTER>(acc, lin_params(a));
}

// Plain lattice sum of a closed family, n <= 2^31: one tile of 256 threads x
// 24 consecutive points per CTA (S == 1), or per cluster of S CTAs (S > 1, small
// n): CTA rank s of the cluster accumulates the s-th slice of the dimensions,
// parks its partial inner sums in shared memory, and rank 0 adds the S slices
// in rank order through distributed shared memory before the outer function.
// tile_out[t] = sum over tile t (fixed tree).
template <int KIND, int OUTER, class Args, int S, bool PAIR>
__global__ void __launch_bounds__(kThreads, 2) k_fam(const __grid_constant__ Args a, uint32_t hmask,
                                                      double* __restrict__ tile_out) {
    constexpr int P = fam_pts(KIND);
    constexpr int NA = KIND == FAM_QUADP ? 2 : 1;   // accumulators per point
    extern __shared__ double part[];   // [NA][P][kThreads] when S > 1
    __shared__ double sh[8];
    uint32_t H[P];
    #pragma unroll
    for (int k = 0; k < P; ++k) H[k] = (threadIdx.x + k) & hmask;   // opaque zeros
    const int64_t tile = blockIdx.x;
    const uint64_t i0_64 = a.base + (uint64_t)tile * (kThreads * P) + (uint64_t)threadIdx.x * P;
    const uint32_t i0 = (uint32_t)i0_64;   // < 2^32 (n <= 2^31)
    double acc[P], acc2[P];
    #pragma unroll
    for (int p = 0; p < P; ++p) {
        acc[p] = 0.0;
        acc2[p] = 0.0;
    }
    int rank = 0;
    if constexpr (S == 1) {
        fam_accumulate<KIND>(a, i0, 0, a.d, H, acc, acc2);
    } else {
        cg::cluster_group cluster = cg::this_cluster();
        rank = (int)cluster.block_rank();
        fam_accumulate<KIND>(a, i0, (int)((int64_t)a.d * rank / S), (int)((int64_t)a.d * (rank + 1) / S), H, acc,
                             acc2);
        #pragma unroll
        for (int p = 0; p < P; ++p) {
            part[p * kThreads + threadIdx.x] = acc[p];
            if (NA == 2) part[(P + p) * kThreads + threadIdx.x] = acc2[p];
        }
        cluster.sync();
        if (rank == 0) {
            #pragma unroll
            for (int p = 0; p < P; ++p) {
                double v = acc[p], v2 = acc2[p];
                #pragma unroll
                for (int r = 1; r < S; ++r) {
                    const double* pr = cluster.map_shared_rank(part, r);
                    v += pr[p * kThreads + threadIdx.x];
                    if (NA == 2) v2 += pr[(P + p) * kThreads + threadIdx.x];
                }
                acc[p] = v;
                acc2[p] = v2;
            }
        }
        cluster.sync();   // peers keep their shared memory until rank 0 has read it
    }
    if (rank != 0) return;
    double s = 0.0;
    #pragma unroll
    for (int p = 0; p < P; ++p) {
        const uint64_t i = i0_64 + p;
        double f;
        if constexpr (KIND == FAM_QUADP) {
            f = quad_pair<OUTER>(acc[p], acc2[p], a.alphaB, lin_params(a), i != 0 && 2 * i != a.n);
        } else if constexpr (PAIR) {
            const bool two = i != 0 && 2 * i != a.n;
            if (OUTER != OUT_POW && a.pf.on && two)   // inline: reads a.pf from parameter space
                f = a.pf.post * pair_fast<OUTER == OUT_POW ? OUT_EXP : OUTER>(acc[p], a.pf);
            else
                f = outer_pair<OUTER>(acc[p], lin_params(a), a.alphaB, two);
        } else {
            f = fam_outer<KIND, OUTER>(acc[p], a);
        }
        s += (i < a.end) ? f : 0.0;
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) tile_out[tile] = s;
}

// ============================================================ product family
// f = K prod_j ((x_j - w_j)^2 + c_j)^p (Genz product peak, config 4's
// integrand, corpus ratprod).  Per point-dim: t = x 2^-g - w_j 2^-g and
// D *= t*t + c_j 2^-2g -- the coordinate is again the denormal residue times a
// scale, so three FP64 ops and the two-op residue step.  D is renormalised to
// [1, 2) every R factors (host-chosen so R scaled factors cannot leave
// 2^(+-1000)) with its exponent kept in an integer.
struct ProdDim {
    double w;       // w_j 2^-g
    double c;       // c_j 2^-2g
    uint32_t z, zs, z2, z2m;
};

template <int N>
struct ProdArgs {
    int nf;              // factors (dimensions that carry one)
    uint32_t n;
    uint64_t base, end;
    double K, pw;
    double m;            // 2^(1074 - g) / n: denormal residue -> x 2^-g
    int32_t off;         // 2 g nf: D_true = D 2^(E + off)
    int32_t rmask;       // renormalise after factor j when (j & rmask) == rmask
    ProdDim dims[N];
};

struct ProdArgsG {   // more factors than kProdParamDims: records in global memory
    int nf;
    uint32_t n;
    uint64_t base, end;
    double K, pw, m;
    int32_t off, rmask;
    const ProdDim* __restrict__ dims;
};

constexpr int kProdParamDims = 1000;  // 1000 x 32 B + header < 32 KB

__device__ __forceinline__ void renorm(double& D, int& E) {
    const int hi = __double2hiint(D), lo = __double2loint(D);
    const int e = (hi >> 20) - 1023;   // D > 0 normal
    D = __hiloint2double(hi - (e << 20), lo);
    E += e;
}

__device__ __noinline__ double prod_outer(double D, int E, double K, double pw, int off) {
    renorm(D, E);
    return ldexp(K * int_pow(D, pw), (int)pw * (E + off));
}

template <class Args>
__global__ void __launch_bounds__(kThreads, 2) k_prod(const __grid_constant__ Args a, uint32_t hmask,
                                                       double* __restrict__ tile_out) {
    constexpr int P = kProdPts;
    __shared__ double sh[8];
    uint32_t H[P];
    #pragma unroll
    for (int k = 0; k < P; ++k) H[k] = (threadIdx.x + k) & hmask;   // opaque zeros
    const uint64_t i0_64 = a.base + (uint64_t)blockIdx.x * (kThreads * P) + (uint64_t)threadIdx.x * P;
    const uint32_t i0 = (uint32_t)i0_64, n = a.n;
    double D[P];
    int E[P];
    #pragma unroll
    for (int p = 0; p < P; ++p) {
        D[p] = 1.0;
        E[p] = 0;
    }
    // m is the same for every factor: one vector register for the whole loop,
    // so each FP64 op below has at most one uniform operand (w_j or c_j) and
    // the per-factor records stay LDCU/UR operands
    double m;
    asm("mov.b64 %0, %1;" : "=d"(m) : "d"(a.m));
    #pragma unroll 1
    for (int j = 0; j < a.nf; ++j) {
        const uint32_t z = a.dims[j].z, z2 = a.dims[j].z2, z2m = a.dims[j].z2m;
        const double w = a.dims[j].w, c = a.dims[j].c;
        uint32_t r0 = mulmod_shoup(i0, z, a.dims[j].zs, n);
        uint32_t r1 = step_mod(r0, z, z - n);
        #pragma unroll
        for (int p = 0; p < P; p += 2) {
            const double t0 = fma(denorm_of(r0, H[p]), m, -w), t1 = fma(denorm_of(r1, H[p + 1]), m, -w);
            D[p] *= fma(t0, t0, c);
            D[p + 1] *= fma(t1, t1, c);
            if (p + 2 < P) {
                r0 = step_mod(r0, z2, z2m);
                r1 = step_mod(r1, z2, z2m);
            }
        }
        if ((j & a.rmask) == a.rmask) {
            #pragma unroll
            for (int p = 0; p < P; ++p) renorm(D[p], E[p]);
        }
    }
    double s = 0.0;
    #pragma unroll
    for (int p = 0; p < P; ++p) {
        const double f = prod_outer(D[p], E[p], a.K, a.pw, a.off);
        s += (i0_64 + p < a.end) ? f : 0.0;
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) tile_out[blockIdx.x] = s;
}

// ============================================================ Korobov orbits
// Full-lattice sums for a Korobov rule z_j = a^(j-1) mod n, n prime (DESIGN.md
// §4.1b).  Two symmetries of the point set cut the work:
//  * shift: point i*a has residues r_j(i*a) = r_(j+1)(i), so a chain of m
//    points i0, i0 a, ..., i0 a^(m-1) needs only the m + d - 1 residues
//    P[t] = i0 a^t mod n -- one Shoup modmul per step instead of one residue
//    step per point-dim; the inner sums of the chain are a sliding
//    correlation of the coefficients with P;
//  * mirror: x(n - i) = 1 - x(i) for i != 0, so the linear (or centred
//    quadratic) form of the mirror point follows from the same sums.
// The nonzero points are enumerated as g^s a^e (g a primitive root, cosets s
// of <a>) over half of the exponents, mirrors covering the rest; point 0 is
// added once by chain 0.
struct OrbHead {
    uint32_t n, a, as;      // modulus, Korobov base, Shoup constant floor(a 2^32 / n)
    int32_t dpad;           // coefficient count padded to a multiple of the chain length
    uint64_t units;         // chains
    uint32_t qc, h;         // chains per coset, exponents per coset
    const uint32_t* G;      // coset representatives g^s
    const uint32_t* Alo;    // a^(m q) for q < 4096
    const uint32_t* Ahi;    // a^(m 4096 q)
    double alpha, alphaB, scale, bsum, K, A, B, C0, kappa, M, half, pw;
    PairFast pf;            // linear families: point and mirror from one range reduction
    int32_t zero;           // unit 0 also adds the point x = 0 (not for the levels of n = 2^k)
};

constexpr int kOrbParamBytes = 32000;
constexpr int kOrbLinDims = (kOrbParamBytes - (int)sizeof(OrbHead)) / 8 / 24 * 24;
constexpr int kOrbQuadDims = (kOrbParamBytes - (int)sizeof(OrbHead)) / 16 / 24 * 24;
#ifndef LQ_ORB_LIN_M
#define LQ_ORB_LIN_M 24
#endif
#ifndef LQ_ORB_QUAD_M
#define LQ_ORB_QUAD_M 12
#endif
__host__ __device__ constexpr int orb_len(int kind) { return kind == 1 ? LQ_ORB_QUAD_M : LQ_ORB_LIN_M; }

template <int N = kOrbLinDims>
struct OrbLinArgs {
    OrbHead h;
    double c[N];                  // beta_j / n * 2^(1074 - sigma), zero padded
};
template <int N = kOrbQuadDims>
struct OrbQuadArgs {
    OrbHead h;
    double2 bq[N];                // ((beta_j + gamma_j) 2^sigma, gamma_j 2^(2 sigma)), zero padded
};

__device__ __forceinline__ uint32_t mulmod32(uint32_t x, uint32_t y, uint32_t n) {
    return (uint32_t)(((uint64_t)x * y) % n);
}

// One thread = one chain of M points (and their mirrors); 256 chains per CTA.
// tile_out[blockIdx.x] = sum over the CTA's chains (fixed tree); chain units
// [unit0 + 256 b, unit0 + 256 (b + 1)).
template <int KIND, int OUTER, class Args>
__global__ void __launch_bounds__(kThreads, 2) k_orbit(const __grid_constant__ Args a, uint64_t unit0,
                                                        uint32_t hmask, double* __restrict__ tile_out) {
    constexpr int M = orb_len(KIND);
    __shared__ double sh[8];
    const OrbHead& H = a.h;
    const uint32_t n = H.n;
    const uint64_t u = unit0 + (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    double s = 0.0;
    if (u < H.units) {
        const uint32_t cs = (uint32_t)(u / H.qc), q = (uint32_t)(u - (uint64_t)cs * H.qc);
        const uint32_t i0 = mulmod32(mulmod32(H.G[cs], H.Alo[q & 4095u], n), H.Ahi[q >> 12], n);
        const int valid = (int)min((uint32_t)M, H.h - q * (uint32_t)M);
        const uint32_t za = H.a, zs = H.as;
        if constexpr (KIND == FAM_LIN) {
            uint32_t W[M], Z[M];
            double acc[M];
            W[0] = i0;
            #pragma unroll
            for (int k = 0; k < M; ++k) {
                Z[k] = (threadIdx.x + k) & hmask;   // opaque zeros (hi words of the denormals)
                acc[k] = 0.0;
                if (k) W[k] = mulmod_shoup(W[k - 1], za, zs, n);
            }
            // (a window of denormal doubles, as in k_orbit_prod, measured 70.4 vs
            // 67.9 ms on cfg5: ptxas then loses the residue-major schedule)
            #pragma unroll 1
            for (int j0 = 0; j0 < H.dpad; j0 += M) {
                #pragma unroll
                for (int v = 0; v < M; ++v) {
                    const double c = a.c[j0 + v];
                    #pragma unroll
                    for (int k = 0; k < M; ++k) acc[k] = fma(c, denorm_of(W[(v + k) % M], Z[(v + k) % M]), acc[k]);
                    W[v] = mulmod_shoup(W[(v + M - 1) % M], za, zs, n);
                }
            }
            const LinParams prm{H.alpha, H.scale, H.K, H.A, H.B, H.C0, H.kappa, H.pw};
            if (OUTER != OUT_POW && H.pf.on) {   // one range reduction per pair, inline (§4.1e)
                double t = 0.0;
                #pragma unroll
                for (int k = 0; k < M; ++k)
                    t += k < valid ? pair_fast<OUTER == OUT_POW ? OUT_EXP : OUTER>(acc[k], H.pf) : 0.0;
                s += H.pf.post * t;
            } else {
                #pragma unroll
                for (int k = 0; k < M; ++k) s += k < valid ? outer_pair<OUTER>(acc[k], prm, H.alphaB, true) : 0.0;
            }
            if (u == 0 && H.zero) s += outer_fn<OUTER>(0.0, prm);   // point 0
        } else {
            const double Ms = H.M, hf = H.half;
            double U[M], V[M], ao[M], ae[M];
            uint32_t r = i0;
            const uint32_t zero = threadIdx.x & hmask;
            #pragma unroll
            for (int k = 0; k < M; ++k) {
                const double x = fma(denorm_of(r, zero), Ms, -hf);
                U[k] = x;
                V[k] = x * x;
                ao[k] = 0.0;
                ae[k] = 0.0;
                r = mulmod_shoup(r, za, zs, n);
            }
            #pragma unroll 1
            for (int j0 = 0; j0 < H.dpad; j0 += M) {
                #pragma unroll
                for (int v = 0; v < M; ++v) {
                    const double2 bq = a.bq[j0 + v];
                    #pragma unroll
                    for (int k = 0; k < M; ++k) {
                        ao[k] = fma(bq.x, U[(v + k) % M], ao[k]);
                        ae[k] = fma(bq.y, V[(v + k) % M], ae[k]);
                    }
                    const double x = fma(denorm_of(r, zero), Ms, -hf);
                    U[v] = x;
                    V[v] = x * x;
                    r = mulmod_shoup(r, za, zs, n);
                }
            }
            const LinParams prm{H.alpha, H.scale, H.K, H.A, H.B, H.C0, H.kappa, H.pw};
            #pragma unroll
            for (int k = 0; k < M; ++k) s += k < valid ? quad_pair<OUTER>(ao[k], ae[k], H.alphaB, prm, true) : 0.0;
            if (u == 0 && H.zero) s += quad_outer<OUTER>(0.0, prm);   // point 0
        }
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) tile_out[blockIdx.x] = s;
}

// Product family over Korobov orbits (no mirror pairs: a factor's mirror has
// the other shift 1 - w_j): the plan enumerates every nonzero point once,
// chains of kOrbProdM points share the residue window as in k_orbit, and each
// point keeps its running product and exponent as in k_prod.
constexpr int kOrbProdM = 16;
constexpr int kOrbProdDims = (kOrbParamBytes - (int)sizeof(OrbHead) - 16) / 16 / kOrbProdM * kOrbProdM;

template <int N>
struct OrbProdArgs {
    OrbHead h;                  // uses n, a, as, dpad, units, qc, h, G, Alo, Ahi, K, pw, M (= 2^(1074-g)/n)
    int32_t nf, off, rmask;     // factors (= d), as ProdArgs
    double2 wc[N];              // (w_j 2^-g, c_j 2^-2g); entries past nf are skipped
};

template <class Args>
__global__ void __launch_bounds__(kThreads, 2) k_orbit_prod(const __grid_constant__ Args a, uint64_t unit0,
                                                             uint32_t hmask, double* __restrict__ tile_out) {
    constexpr int M = kOrbProdM;
    __shared__ double sh[8];
    const OrbHead& H = a.h;
    const uint32_t n = H.n;
    const uint64_t u = unit0 + (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    double s = 0.0;
    if (u < H.units) {
        const uint32_t cs = (uint32_t)(u / H.qc), q = (uint32_t)(u - (uint64_t)cs * H.qc);
        const uint32_t i0 = mulmod32(mulmod32(H.G[cs], H.Alo[q & 4095u], n), H.Ahi[q >> 12], n);
        const int valid = (int)min((uint32_t)M, H.h - q * (uint32_t)M);
        const uint32_t za = H.a, zs = H.as;
        // the residue window is kept as denormal doubles X = {r, 0}: a new
        // residue is written straight into the low word of its slot, so the
        // DFMAs read the pair without per-use moves
        const uint32_t zero = threadIdx.x & hmask;
        double X[M], D[M];
        int E[M];
        uint32_t r = i0;
        #pragma unroll
        for (int k = 0; k < M; ++k) {
            X[k] = denorm_of(r, zero);
            D[k] = 1.0;
            E[k] = 0;
            if (k + 1 < M) r = mulmod_shoup(r, za, zs, n);
        }
        double m;
        asm("mov.b64 %0, %1;" : "=d"(m) : "d"(H.M));   // one vector register: a single uniform operand per op
        #pragma unroll 1
        for (int j0 = 0; j0 < H.dpad; j0 += M) {
            #pragma unroll
            for (int v = 0; v < M; ++v) {
                const double2 wc = a.wc[j0 + v];
                if (j0 + v < a.nf) {   // uniform: the padded tail of the last block is skipped
                    #pragma unroll
                    for (int k = 0; k < M; ++k) {
                        const double t = fma(X[(v + k) % M], m, -wc.x);
                        D[k] *= fma(t, t, wc.y);
                    }
                }
                r = mulmod_shoup(r, za, zs, n);
                X[v] = denorm_of(r, zero);
                if (((j0 + v) & a.rmask) == a.rmask) {
                    #pragma unroll
                    for (int k = 0; k < M; ++k) renorm(D[k], E[k]);
                }
            }
        }
        #pragma unroll
        for (int k = 0; k < M; ++k) s += k < valid ? prod_outer(D[k], E[k], H.K, H.pw, a.off) : 0.0;
        if (u == 0 && H.zero) {   // point 0 (x = 0): the same factors at t = -w_j
            double D0 = 1.0;
            int E0 = 0;
            for (int j = 0; j < a.nf; ++j) {
                const double2 wc = a.wc[j];
                D0 *= fma(wc.x, wc.x, wc.y);
                if ((j & a.rmask) == a.rmask) renorm(D0, E0);
            }
            s += prod_outer(D0, E0, H.K, H.pw, a.off);
        }
    }
    s = block_sum(s, sh);
    if (threadIdx.x == 0) tile_out[blockIdx.x] = s;
}

// ---------------------------------------------------- Korobov orbits, FFT form
// The chain sums L_k = sum_j c_j P[k + j] (k < B) are a correlation of the
// coefficients with the residue sequence P[t] = i0 a^t mod n, t < N = B + d - 1:
// one forward FFT of P, a product with conj(FFT(c)), one inverse FFT give all
// B linear forms of a chain (overlap-save), O(log N) FP64 work per point
// instead of O(d).  Two chains ride in one complex FFT
// (real and imaginary parts); c is real, so their correlations separate.
struct FftHead {
    uint32_t n, B;                     // modulus, chain length N - d + 1
    uint64_t units;                    // chains
    uint32_t qc, h;                    // chains per coset, exponents per coset
    const uint32_t* G;                 // coset representatives
    const uint32_t* Alo;               // a^(B q), q < 4096
    const uint32_t* Ahi;               // a^(B 4096 q)
    const uint2* apow;                 // (a^t mod n, floor(a^t 2^32 / n)), t < N
    const uint32_t* starts;            // first point of every chain
    const double2* W;                  // e^{-2 pi i k / N}
    const double2* Hc;                 // conj(FFT(c zero-padded)) / N, c_j = beta_j / n
    double alpha, alphaB, K, A, Bc, C0, kappa, pw;
    PairFast pf;
    const lq_insn* g_insn;             // OUT_PROG: the outer G as bytecode (variable 0)
    int32_t g_n, g_result;
    int32_t zero;                      // unit 0 also adds the point x = 0
    double2 etab[kFftExpTab > 0 ? kFftExpTab : 1];          // (2^(j/2^EB), 2^(-j/2^EB)), correctly rounded on the host
};

// H[m] of a real sequence's spectrum from the lower half only: H[N - m] =
// conj(H[m]), which halves the table's cache footprint (32 KB).
// Filter-spectrum reads with an L1 evict-last hint: the 32 KB half table must
// stay in the 60 KB of L1 the shared-memory carveout leaves (7.106 -> 7.089 ms)
#ifndef LQ_FFT_HLOAD
#define LQ_FFT_HLOAD 1
#endif
__device__ __forceinline__ double2 ldg_last(const double2* p) {
#if LQ_FFT_HLOAD
    double2 v;
    asm volatile("ld.global.nc.L1::evict_last.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ double2 hermitian_load(const double2* __restrict__ H, int m) {
    if (m <= kFftN / 2) return ldg_last(H + m);
    const double2 h = ldg_last(H + (kFftN - m));
    return make_double2(h.x, -h.y);
}

// first point of chain u (host-computed table: no 64-bit divisions here)
__device__ __forceinline__ uint32_t fft_chain_start(const FftHead& a, uint64_t u) { return __ldg(a.starts + u); }

// points of chain u that belong to the enumeration (the last chain of a coset is short)
__device__ __forceinline__ int fft_chain_valid(const FftHead& a, uint64_t u) {
    if (u >= a.units) return 0;
    const uint32_t q = (uint32_t)u % a.qc;   // units < 2^32
    return (int)min(a.B, a.h - q * a.B);
}

// Deterministic CTA sum for NT threads (fixed tree).  Result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum_n(double v, double* sh /* >= NT / 32 */) {
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < (NT / 32) ? sh[lane] : 0.0;
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;
}


// Per-tile CTA sums without their own barriers: each warp leaves its partial
// in a slot of the tile's parity, and thread 0 sums the previous tile's eight
// slots after the next tile's first FFT barrier (measured 7.50 -> 7.33 ms on cfg5)
#ifndef LQ_FFT_DEFER
#define LQ_FFT_DEFER 1
#endif

// p < 2^32 as a double: (2^52 + p) - 2^52, one DADD instead of an I2F.F64
// (cfg5 7.26 -> 7.20 ms)
__device__ __forceinline__ double u32_to_double(uint32_t p) {
    return __hiloint2double(0x43300000, (int)p) - 4503599627370496.0;
}
// the eight warp partials of a 256-thread CTA in block_sum_n's xor-tree order
__device__ __forceinline__ double defer_sum8(const double* w) {
    return ((w[0] + w[4]) + (w[2] + w[6])) + ((w[1] + w[5]) + (w[3] + w[7]));
}

// Tile b = two chains (units 2b, 2b + 1 after unit0); tile_out[b] = their sum.
// A CTA runs tiles per_cta blockIdx.x .. + per_cta - 1 (< ntiles), so the
// twiddle tables are filled once per per_cta tiles.
// RM (FAST only): the chains have at most RM * N/R points, so the outputs
// r >= RM of the last inverse pass are dead and the compiler drops them (and
// their registers) -- d = 769..1024: RM = 13 (cfg5 7.20 -> 7.10 ms).
template <int OUTER, bool FAST, int RM = kFftR>
__global__ void __launch_bounds__(kFftThreads, 2) k_orbit_fft(const __grid_constant__ FftHead a, uint64_t unit0,
                                                               int64_t ntiles, int per_cta,
                                                               double* __restrict__ tile_out) {
    constexpr int R = kFftR;
    extern __shared__ double2 buf[];   // kFftPad, then the twiddle tables
    __shared__ double sh[32];
    double2* tw = buf + kFftPad;
    fft_load_twiddles(tw, a.W);          // visible after the first pass's barrier
    const double2* Wt = kFftR == 16 ? tw : a.W;
#if LQ_FFT_EXPTAB
    double2* et = tw + kFftTwAll;
    if (threadIdx.x < kFftExpTab) et[threadIdx.x] = a.etab[threadIdx.x];   // visible after the first barrier
#endif
    const uint32_t n = a.n;
    const int64_t b0 = (int64_t)blockIdx.x * per_cta;
    const int64_t b1 = min(b0 + per_cta, ntiles);
    #pragma unroll 1
    for (int64_t tb = b0; tb < b1; ++tb) {
    const uint64_t u0 = unit0 + 2ull * (uint64_t)tb, u1 = u0 + 1;
    const uint32_t s0 = u0 < a.units ? fft_chain_start(a, u0) : 0u;
    const uint32_t s1 = u1 < a.units ? fft_chain_start(a, u1) : 0u;
    // residues of both chains straight into the registers of the first pass:
    // thread j holds positions t = j + (N/R) r, P[t] = s a^j (a^(N/R))^r --
    // one table load per thread, then a Shoup step per position
    double2 v[R];
    {
        const uint2 aj = __ldg(a.apow + threadIdx.x), as = __ldg(a.apow + kFftThreads);
        uint32_t p0 = mulmod_shoup(s0, aj.x, aj.y, n), p1 = mulmod_shoup(s1, aj.x, aj.y, n);
        #pragma unroll
        for (int r = 0; r < R; ++r) {
            v[r] = make_double2(u32_to_double(p0), u32_to_double(p1));
            p0 = mulmod_shoup(p0, as.x, as.y, n);
            p1 = mulmod_shoup(p1, as.x, as.y, n);
        }
    }
    fft4096_regs<false>(v, buf, Wt);
#if LQ_FFT_DEFER
    // the previous tile's warp partials (written before this tile's first
    // barrier) summed in block_sum_n's fixed order
    if (threadIdx.x == 0 && tb > b0) tile_out[tb - 1] = defer_sum8(sh + 8 * ((tb - 1) & 1));
#endif
    // Y = X conj(C) / N, conjugated so that the forward transform inverts it;
    // the last forward pass left positions j + (N/R) r in this thread, which
    // are exactly the inputs of the first inverse pass
    #pragma unroll
    for (int r = 0; r < R; ++r) {
        const double2 y = cmul(v[r], hermitian_load(a.Hc, threadIdx.x + r * kFftThreads));
        v[r] = make_double2(y.x, -y.y);
    }
    const LinParams prm{a.alpha, 1.0, a.K, a.A, a.Bc, a.C0, a.kappa, a.pw};
    double s = 0.0;
    if constexpr (FAST) {
        // inverse transform with its outputs left in registers (positions
        // j + (N/R) r, natural order): the lean pair outer runs on them
        // directly, skipping warps whose positions are all past the chains
        fft4096_regs<false>(v, buf, Wt);
        const int v0 = fft_chain_valid(a, u0), v1 = fft_chain_valid(a, u1);
#if LQ_FFT_EXPTAB
        const double2* T = et;
#else
        const double2* T = nullptr;
#endif
        const int B = (int)a.B;
        if (LQ_FFT_FULLTILE && v0 == B && v1 == B && (RM - 1) * kFftThreads < B) {
            // both chains full (every tile but the last of a coset): positions
            // r < RM - 1 are all inside the chains -- no masks, no branches
            #pragma unroll
            for (int r = 0; r < RM - 1; ++r)
                s += pair_outer_fft<OUTER>(v[r].x, a.pf, T) + pair_outer_fft<OUTER>(-v[r].y, a.pf, T);
            if ((threadIdx.x & ~31) + (RM - 1) * kFftThreads < B) {
                const int k = threadIdx.x + (RM - 1) * kFftThreads;
                const double g = pair_outer_fft<OUTER>(v[RM - 1].x, a.pf, T) +
                                 pair_outer_fft<OUTER>(-v[RM - 1].y, a.pf, T);
                s += k < B ? g : 0.0;
            }
        } else {
            const int vmax = max(v0, v1), wbase = threadIdx.x & ~31;
            #pragma unroll
            for (int r = 0; r < RM; ++r) {
                if (wbase + r * kFftThreads < vmax) {
                    const int k = threadIdx.x + r * kFftThreads;
                    const double g0 = pair_outer_fft<OUTER>(v[r].x, a.pf, T),
                                 g1 = pair_outer_fft<OUTER>(-v[r].y, a.pf, T);
                    s += (k < v0 ? g0 : 0.0) + (k < v1 ? g1 : 0.0);
                }
            }
        }
        s *= a.pf.post;
    } else {
    // inverse transform; its last pass writes the correlations to shared memory
    // so the out-of-line outer function runs with no transform state live
    fft4096_regs<true>(v, buf, Wt);
    const int v0 = fft_chain_valid(a, u0), v1 = fft_chain_valid(a, u1);   // recomputed: not live across the FFTs
    if constexpr (OUTER == OUT_PROG) {
        // G(s) + G(sum beta - s) by the bytecode interpreter: nothing of the
        // transforms is live here, so its slots cost only local memory
        double slot[32];
        #pragma unroll 1
        for (int k = threadIdx.x; k < v0 || k < v1; k += kFftThreads) {
            const double2 y = buf[fpad(k)];
            const double l0 = y.x, l1 = -y.y;
            double g = 0.0;
            if (k < v0)
                g += run_program<32>(a.g_insn, a.g_n, a.g_result, UnivSrc{l0}, slot) +
                     run_program<32>(a.g_insn, a.g_n, a.g_result, UnivSrc{a.alphaB - l0}, slot);
            if (k < v1)
                g += run_program<32>(a.g_insn, a.g_n, a.g_result, UnivSrc{l1}, slot) +
                     run_program<32>(a.g_insn, a.g_n, a.g_result, UnivSrc{a.alphaB - l1}, slot);
            s += g;
        }
        if (u0 == 0 && a.zero && threadIdx.x == 0) s += run_program<32>(a.g_insn, a.g_n, a.g_result, UnivSrc{0.0}, slot);
    } else {
    #pragma unroll 1
    for (int k = threadIdx.x; k < v0 || k < v1; k += kFftThreads) {
        const double2 y = buf[fpad(k)];             // conj of the correlation: (L0, -L1)
        // inlined (no call): nothing else is live here
        const double l0 = y.x, l1 = -y.y;
        const double f00 = outer_val<OUTER>(l0 + prm.alpha, prm), f01 = outer_val<OUTER>(a.alphaB - l0, prm);
        const double f10 = outer_val<OUTER>(l1 + prm.alpha, prm), f11 = outer_val<OUTER>(a.alphaB - l1, prm);
        s += (k < v0 ? f00 + f01 : 0.0) + (k < v1 ? f10 + f11 : 0.0);
    }
    }
    }
    if constexpr (OUTER != OUT_PROG)
        if (u0 == 0 && a.zero && threadIdx.x == 0) s += outer_fn<OUTER>(0.0, prm);   // point 0
#if LQ_FFT_DEFER
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[8 * (tb & 1) + (threadIdx.x >> 5)] = s;
#else
    s = block_sum_n<kFftThreads>(s, sh);
    if (threadIdx.x == 0) tile_out[tb] = s;
#endif
    }
#if LQ_FFT_DEFER
    __syncthreads();
    if (threadIdx.x == 0 && b1 > b0) tile_out[b1 - 1] = defer_sum8(sh + 8 * ((b1 - 1) & 1));
#endif
}

// Gaussian family in FFT form: one chain per CTA.  The centred coordinates
// u_t = P[t]/n - 1/2 and their squares ride as x = u + i u^2 in one transform;
// with X = FFT(x), the odd/even correlations (b' with u, q with u^2) come back
// as Re/Im of IFFT(Z), Z[m] = X[m] H+[m] + conj(X[N-m]) H-[m],
// H+- = (conj(FFT(b')) +- conj(FFT(q))) / (2N) (spectra of the real parts
// separated by symmetry).  Point and mirror: exp(alpha' + even +- odd).
template <int OUTER>
__global__ void __launch_bounds__(kFftThreads, 2) k_orbit_fft_quad(const __grid_constant__ FftHead a,
                                                                    const double2* __restrict__ Hm,
                                                                    uint64_t unit0, int64_t ntiles, int per_cta,
                                                                    double* __restrict__ tile_out) {
    constexpr int R = kFftR;
    extern __shared__ double2 buf[];   // kFftPad, then the twiddle tables
    __shared__ double sh[32];
    double2* tw = buf + kFftPad;
    fft_load_twiddles(tw, a.W);
    const double2* Wt = kFftR == 16 ? tw : a.W;
    const uint32_t n = a.n;
    const int64_t b0 = (int64_t)blockIdx.x * per_cta;
    const int64_t b1 = min(b0 + per_cta, ntiles);
    #pragma unroll 1
    for (int64_t tb = b0; tb < b1; ++tb) {
    const uint64_t u0 = unit0 + (uint64_t)tb;
    const uint32_t s0 = u0 < a.units ? fft_chain_start(a, u0) : 0u;
    const double inv_n = 1.0 / (double)n;
    double2 v[R];
    #pragma unroll
    for (int r = 0; r < R; ++r) {
        const int t = threadIdx.x + r * kFftThreads;
        const uint2 ap = __ldg(a.apow + t);
        const double u = fma(u32_to_double(mulmod_shoup(s0, ap.x, ap.y, n)), inv_n, -0.5);
        v[r] = make_double2(u, u * u);
    }
    fft4096_regs<true>(v, buf, Wt);        // X in shared memory, natural order
#if LQ_FFT_DEFER
    if (threadIdx.x == 0 && tb > b0) tile_out[tb - 1] = defer_sum8(sh + 8 * ((tb - 1) & 1));
#endif
    #pragma unroll
    for (int r = 0; r < R; ++r) {
        const int m = threadIdx.x + r * kFftThreads;
        const double2 x = buf[fpad(m)], xr = buf[fpad((kFftN - m) & (kFftN - 1))];
        const double2 z = cadd(cmul(x, __ldg(a.Hc + m)), cmul(make_double2(xr.x, -xr.y), __ldg(Hm + m)));
        v[r] = make_double2(z.x, -z.y);     // conjugated: the forward transform inverts it
    }
    fft4096_regs<false>(v, buf, Wt);       // (first pass stores only after its barrier); outputs stay in v
    const LinParams prm{a.alpha, 1.0, a.K, a.A, a.Bc, a.C0, a.kappa, a.pw};
    const int v0 = fft_chain_valid(a, u0), wbase = threadIdx.x & ~31;
    double s = 0.0;
    #pragma unroll
    for (int r = 0; r < R; ++r) {
        if (wbase + r * kFftThreads < v0) {
            const double2 y = v[r];             // conj: (odd, -even) at position j + (N/R) r
            const double t = a.alphaB - y.y;
            const double g = outer_val<OUTER>(t + y.x, prm) + outer_val<OUTER>(t - y.x, prm);
            s += threadIdx.x + r * kFftThreads < v0 ? g : 0.0;
        }
    }
    if (u0 == 0 && a.zero && threadIdx.x == 0) s += quad_outer<OUTER>(0.0, prm);   // point 0
#if LQ_FFT_DEFER
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sh[8 * (tb & 1) + (threadIdx.x >> 5)] = s;
#else
    s = block_sum_n<kFftThreads>(s, sh);
    if (threadIdx.x == 0) tile_out[tb] = s;
#endif
    }
#if LQ_FFT_DEFER
    __syncthreads();
    if (threadIdx.x == 0 && b1 > b0) tile_out[b1 - 1] = defer_sum8(sh + 8 * ((b1 - 1) & 1));
#endif
}

// ============================================================ generic bytecode
struct LatSrc32 {   // n <= 2^31: Shoup modmul per variable access
    uint32_t i, n;
    double n_d, inv_n;
    const uint2* zz;   // (z, zs)
    __device__ __forceinline__ double x(int b) const {
        const uint2 t = __ldg(zz + b);
        return exact_div((double)mulmod_shoup(i, t.x, t.y, n), n_d, inv_n);
    }
};

struct LatSrc64 {   // n < 2^53
    uint64_t i, n;
    double n_d, inv_n, ninv_mm;
    const uint64_t* z;
    __device__ __forceinline__ double x(int b) const {
        return exact_div((double)mulmod_u64(i, __ldg(z + b), n, ninv_mm), n_d, inv_n);
    }
};

template <int NS, bool WIDE>
__global__ void __launch_bounds__(kThreads) k_prog_lattice(const lq_insn* __restrict__ prog, int n_insn, int result,
                                                          uint64_t n, double n_d, double inv_n, double ninv_mm,
                                                          const void* __restrict__ ztab, uint64_t base, uint64_t end,
                                                          int64_t ntiles, double* __restrict__ tile_out) {
    __shared__ double sh[8];
    double slot[NS];
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t i0 = base + (uint64_t)tile * kTile + (uint64_t)threadIdx.x * kPts;
        double s = 0.0;
        for (int p = 0; p < kPts; ++p) {
            const uint64_t i = i0 + p;
            double f = 0.0;
            if (i < end) {
                if (WIDE) {
                    LatSrc64 src{i % n, n, n_d, inv_n, ninv_mm, (const uint64_t*)ztab};
                    f = run_program<NS>(prog, n_insn, result, src, slot);
                } else {
                    LatSrc32 src{(uint32_t)i, (uint32_t)n, n_d, inv_n, (const uint2*)ztab};
                    f = run_program<NS>(prog, n_insn, result, src, slot);
                }
            }
            s += f;
        }
        s = block_sum(s, sh);
        if (threadIdx.x == 0) tile_out[tile] = s;
    }
}

// ============================================================ Monte Carlo
// quad.mc_integrate (quad.py:79-93) draws numpy's default_rng(seed).random((rows, d))
// row-major: PCG64 (128-bit LCG s <- M s + inc, XSL-RR 128/64 output of the new
// state), random() = (out >> 11) 2^-53.  Draw k of the stream is an affine
// jump of the seed state, so every coordinate is generated in place: thread
// state S = state before its point's first draw, coordinate b = output of
// A_(b+1) S + C_(b+1) (host-computed jump table), next point S <- A_d S + C_d.
typedef unsigned __int128 u128;

struct Jump {        // s -> A s + C (mod 2^128)
    uint64_t alo, ahi, clo, chi;
};

__device__ __forceinline__ u128 jump_apply(const Jump& j, u128 s) {
    const u128 A = ((u128)j.ahi << 64) | j.alo, C = ((u128)j.chi << 64) | j.clo;
    return A * s + C;
}

__device__ __forceinline__ double pcg_double(u128 s) {
    const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    const unsigned rot = (unsigned)(hi >> 58);
    const uint64_t x = hi ^ lo;
    const uint64_t out = (x >> rot) | (x << ((64u - rot) & 63u));
    return (double)(out >> 11) * (1.0 / 9007199254740992.0);
}

struct McSrc {
    u128 S;
    const Jump* __restrict__ jt;   // jt[b] advances by b draws, b = 0..d
    __device__ __forceinline__ double x(int b) const {
        const Jump j = jt[b + 1];
        return pcg_double(jump_apply(j, S));
    }
};

// Points [base, end) in tiles of 4096 (256 threads x 16 consecutive points).
// pow2[k] jumps by 2^k draws (k < 64).
template <int NS>
__global__ void __launch_bounds__(kThreads) k_prog_mc(const lq_insn* __restrict__ prog, int n_insn, int result, int d,
                                                      const Jump* __restrict__ jt, const Jump* __restrict__ pow2,
                                                      uint64_t s0lo, uint64_t s0hi, uint64_t base, uint64_t end,
                                                      int64_t ntiles, double* __restrict__ tile_out) {
    __shared__ double sh[8];
    double slot[NS];
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t i0 = base + (uint64_t)tile * kTile + (uint64_t)threadIdx.x * kPts;
        u128 S = ((u128)s0hi << 64) | s0lo;
        const uint64_t k0 = i0 * (uint64_t)d;   // draws before point i0
        for (int k = 0; k < 64; ++k)
            if ((k0 >> k) & 1ull) S = jump_apply(pow2[k], S);
        const Jump jd = jt[d];
        double s = 0.0;
        for (int p = 0; p < kPts; ++p) {
            if (i0 + p < end) {
                McSrc src{S, jt};
                s += run_program<NS>(prog, n_insn, result, src, slot);
            }
            S = jump_apply(jd, S);
        }
        s = block_sum(s, sh);
        if (threadIdx.x == 0) tile_out[tile] = s;
    }
}

// ============================================================ tensor grid
constexpr int kMaxAxes = 128;

struct TensorSrc {
    const double* nodes;
    const int64_t* off;
    const uint32_t* digit;
    __device__ __forceinline__ double x(int b) const { return __ldg(nodes + off[b] + digit[b]); }
};

// Direct sum over the tensor grid, flat index s = s_1 + s_2 n_1 + ... (first
// axis fastest, mdi.py:118-124).  Each thread decodes its first index and
// advances an odometer over its 16 consecutive nodes.
template <int NS>
__global__ void __launch_bounds__(kThreads) k_prog_tensor(const lq_insn* __restrict__ prog, int n_insn, int result,
                                                          int d, const int64_t* __restrict__ counts,
                                                          const int64_t* __restrict__ off,
                                                          const double* __restrict__ nodes,
                                                          uint64_t base, uint64_t end, int64_t ntiles,
                                                          double* __restrict__ tile_out) {
    __shared__ double sh[8];
    double slot[NS];
    uint32_t digit[kMaxAxes];
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t s0 = base + (uint64_t)tile * kTile + (uint64_t)threadIdx.x * kPts;
        uint64_t rem = s0;
        for (int k = 0; k < d; ++k) {
            const uint64_t c = (uint64_t)counts[k];
            digit[k] = (uint32_t)(rem % c);
            rem /= c;
        }
        TensorSrc src{nodes, off, digit};
        double s = 0.0;
        for (int p = 0; p < kPts; ++p) {
            if (s0 + p < end) s += run_program<NS>(prog, n_insn, result, src, slot);
            for (int k = 0; k < d; ++k) {   // odometer
                if (++digit[k] < (uint64_t)counts[k]) break;
                digit[k] = 0;
            }
        }
        s = block_sum(s, sh);
        if (threadIdx.x == 0) tile_out[tile] = s;
    }
}

// ============================================================ element-wise
// eval_array (exprcore.py:442-480): one row per thread, grid-stride; variable
// b of row i is cols[b][i] (coalesced across the warp)
struct ColSrc {
    const double* const* __restrict__ cols;
    int64_t i;
    __device__ __forceinline__ double x(int b) const { return __ldg(cols[b] + i); }
};

template <int NS>
__global__ void __launch_bounds__(kThreads) k_prog_eval(const lq_insn* __restrict__ prog, int n_insn, int result,
                                                        const double* const* __restrict__ cols, int64_t m,
                                                        double* __restrict__ out) {
    double slot[NS];
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < m; i += (int64_t)gridDim.x * kThreads) {
        ColSrc src{cols, i};
        out[i] = run_program<NS>(prog, n_insn, result, src, slot);
    }
}

__global__ void k_midpoint_nodes(const int64_t* __restrict__ counts, const int64_t* __restrict__ off, int d,
                                 double* __restrict__ nodes) {
    // nodes of axis k: RN((t + 0.5) / n_k), transform.py:177
    const int k = blockIdx.y;
    if (k >= d) return;
    const int64_t c = counts[k];
    const double cd = (double)c, inv = 1.0 / cd;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < c; t += (int64_t)gridDim.x * blockDim.x)
        nodes[off[k] + t] = exact_div((double)t + 0.5, cd, inv);
}

// ============================================================ MDI cluster sums
// One CTA per (factor, node block): evaluates U_f(y_t) = R(y_t) e^{i P(y_t)}
// on the block's 256 midpoint nodes and writes the (re, im) block sums.
template <int NS>
__global__ void __launch_bounds__(kThreads) k_mdi_blocks(const lq_insn* __restrict__ insn,
                                                         const lq_factor* __restrict__ fac,
                                                         const double* __restrict__ nodes, int nblk,
                                                         int shard, int nshards, double* __restrict__ part) {
    __shared__ double sh[8];
    double slot[NS];
    const int f = blockIdx.x, b = blockIdx.y;
    const lq_factor F = fac[f];
    const int NB = (F.count + LQ_NODE_BLOCK - 1) / LQ_NODE_BLOCK;
    const int b_lo = (int)(((int64_t)shard * NB) / nshards), b_hi = (int)(((int64_t)(shard + 1) * NB) / nshards);
    if (b < b_lo || b >= b_hi) return;
    if (F.reserved == LQ_FACTOR_SUPPLIED) {
        // a core factor whose sum over its own sub-grid the host supplies
        // as (re, im) at nodes[node_off] (one block)
        if (threadIdx.x == 0) {
            part[((int64_t)f * nblk + b) * 2 + 0] = nodes[F.node_off];
            part[((int64_t)f * nblk + b) * 2 + 1] = nodes[F.node_off + 1];
        }
        return;
    }
    const int t = b * LQ_NODE_BLOCK + threadIdx.x;
    double re = 0.0, im = 0.0;
    if (t < F.count) {
        const double cd = (double)F.count;
        UnivSrc src{F.node_off < 0 ? exact_div((double)t + 0.5, cd, 1.0 / cd) : nodes[F.node_off + t]};
        double R = F.r_len ? run_program<NS>(insn + F.r_off, F.r_len, F.r_result, src, slot) : 1.0;
        if (F.p_len) {
            double P = run_program<NS>(insn + F.p_off, F.p_len, F.p_result, src, slot);
            double sn, cs;
            sincos(P, &sn, &cs);
            re = R * cs;
            im = R * sn;
        } else {
            re = R;
        }
    }
    re = block_sum(re, sh);
    im = block_sum(im, sh);
    if (threadIdx.x == 0) {
        part[((int64_t)f * nblk + b) * 2 + 0] = re;
        part[((int64_t)f * nblk + b) * 2 + 1] = im;
    }
}

// Single-CTA combine in log-polar form (fixed order everywhere).
__global__ void __launch_bounds__(kThreads) k_mdi_combine(const double* __restrict__ part, int n_factors, int nblk,
                                                          const lq_factor* __restrict__ fac,
                                                          const int32_t* __restrict__ term_ptr,
                                                          const int32_t* __restrict__ term_fac,
                                                          const double* __restrict__ coef,   // [n_terms][2]
                                                          const double* __restrict__ log_extra, int n_terms,
                                                          double* __restrict__ fwork,   // [n_factors][2]
                                                          double* __restrict__ twork,   // [n_terms][2]
                                                          double* __restrict__ out4) {
    __shared__ double sh[8];
    __shared__ double sM;
    for (int f = threadIdx.x; f < n_factors; f += kThreads) {
        const int NB = (fac[f].count + LQ_NODE_BLOCK - 1) / LQ_NODE_BLOCK;
        double re = 0.0, im = 0.0;
        for (int b = 0; b < NB; ++b) {
            re += part[((int64_t)f * nblk + b) * 2 + 0];
            im += part[((int64_t)f * nblk + b) * 2 + 1];
        }
        fwork[2 * f + 0] = log(hypot(re, im));
        fwork[2 * f + 1] = atan2(im, re);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < n_terms; t += kThreads) {
        double L = log(hypot(coef[2 * t], coef[2 * t + 1])) + log_extra[t];
        double ph = atan2(coef[2 * t + 1], coef[2 * t]);
        for (int k = term_ptr[t]; k < term_ptr[t + 1]; ++k) {
            L += fwork[2 * term_fac[k] + 0];
            ph += fwork[2 * term_fac[k] + 1];
        }
        twork[2 * t + 0] = L;
        twork[2 * t + 1] = ph;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double M = -INFINITY;
        for (int t = 0; t < n_terms; ++t) M = fmax(M, twork[2 * t]);
        sM = M;
    }
    __syncthreads();
    const double M = sM;
    double sre = 0.0, sim = 0.0;
    if (M > -INFINITY) {
        for (int t = threadIdx.x; t < n_terms; t += kThreads) {
            const double m = exp(twork[2 * t] - M);
            double sn, cs;
            sincos(twork[2 * t + 1], &sn, &cs);
            sre += m * cs;
            sim += m * sn;
        }
    }
    sre = block_sum(sre, sh);
    sim = block_sum(sim, sh);
    if (threadIdx.x == 0) {
        if (M == -INFINITY || sre == 0.0) {
            out4[0] = -INFINITY; out4[1] = 0.0; out4[2] = 0.0; out4[3] = 0.0;
        } else {
            out4[0] = M + log(fabs(sre));
            out4[1] = sre > 0.0 ? 1.0 : -1.0;
            out4[2] = sre * exp(M);
            out4[3] = sim * exp(M);
        }
    }
}

// ============================================================ MDI level collapse
// f = G(alpha + <beta, y>) on the midpoint grid with commensurate steps
// beta_j y_t = h m_j (2t + 1): the reference's level loop strips one axis per
// level and its like-term collection merges the partial sums whose constants
// coincide (mdi.py:152-165, exprcore.py:139-169, 390-402), so what it carries
// per level is the multiset of values of the partial linear form.  Here that
// multiset is a distribution over k = sum_j |m_j| t_j (t_j uniform on
// [0, N_j)): one convolution per direction, p'[s] = (1/N) sum_t p[s - |m| t],
// then one pass of G over the support.  All terms are positive, so the level
// sums carry no cancellation; four interleaved accumulators keep the rounding
// at ~N/4 ulp per level.
struct LinLevel {
    int64_t m;     // |m_j| >= 1
    int32_t n;     // N_j nodes
    int32_t pad;
    int64_t woff;  // offset of the level's N_j node weights, or -1 (uniform)
};

// p_new[s] = (1/n) sum_t w_t p_old[s - m t] (w_t = 1 without weights)
__device__ __forceinline__ double lin_conv_point(const double* __restrict__ p, int64_t k_old, int64_t s,
                                                 int64_t m, int n, const double* __restrict__ w) {
    const int64_t t_lo = s < k_old ? 0 : (s - k_old + m) / m;   // s - m t <= k_old - 1
    const int64_t t_hi = min((int64_t)n - 1, s / m);
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int64_t t = t_lo;
    const double* q = p + (s - m * t_lo);
    if (w) {
        for (; t + 3 <= t_hi; t += 4, q -= 4 * m) {
            a0 = fma(w[t], q[0], a0);
            a1 = fma(w[t + 1], q[-m], a1);
            a2 = fma(w[t + 2], q[-2 * m], a2);
            a3 = fma(w[t + 3], q[-3 * m], a3);
        }
        for (; t <= t_hi; ++t, q -= m) a0 = fma(w[t], q[0], a0);
    } else {
        for (; t + 3 <= t_hi; t += 4, q -= 4 * m) {
            a0 += q[0];
            a1 += q[-m];
            a2 += q[-2 * m];
            a3 += q[-3 * m];
        }
        for (; t <= t_hi; ++t, q -= m) a0 += q[0];
    }
    return ((a0 + a1) + (a2 + a3)) / (double)n;
}

// Every level in one CTA with both distributions in shared memory (support
// <= k_cap doubles each); the final distribution goes to p_out.
__global__ void __launch_bounds__(1024) k_linform_smem(const LinLevel* __restrict__ lv, int n_lv, int64_t k_cap,
                                                       const double* __restrict__ wts, double* __restrict__ p_out) {
    extern __shared__ double lin_sm[];
    double* a = lin_sm;
    double* b = lin_sm + k_cap;
    if (threadIdx.x == 0) a[0] = 1.0;
    int64_t K = 1;
    __syncthreads();
    for (int l = 0; l < n_lv; ++l) {
        const LinLevel L = lv[l];
        const int64_t Kn = K + L.m * (L.n - 1);
        const double* w = L.woff >= 0 ? wts + L.woff : nullptr;
        for (int64_t s = threadIdx.x; s < Kn; s += blockDim.x) b[s] = lin_conv_point(a, K, s, L.m, L.n, w);
        __syncthreads();
        double* t = a;
        a = b;
        b = t;
        K = Kn;
    }
    for (int64_t s = threadIdx.x; s < K; s += blockDim.x) p_out[s] = a[s];
}

__global__ void k_fill(double* __restrict__ p, int64_t count, double v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// One level in global memory (support past the shared-memory capacity).
__global__ void __launch_bounds__(kThreads) k_linform_level(const double* __restrict__ p, int64_t k_old,
                                                            int64_t m, int n, const double* __restrict__ w,
                                                            double* __restrict__ q) {
    const int64_t Kn = k_old + m * (n - 1);
    for (int64_t s = blockIdx.x * (int64_t)kThreads + threadIdx.x; s < Kn; s += (int64_t)gridDim.x * kThreads)
        q[s] = lin_conv_point(p, k_old, s, m, n, w);
}

// ---- two linear forms: the joint distribution on a K1 x K2 grid (row-major)
struct Lin2Level {
    int64_t m1, m2;     // |m1_j|, |m2_j| (either may be 0)
    int32_t n;          // N_j nodes
    int32_t flip;       // bit 0: form 1 takes node N-1-t (negative step), bit 1: form 2
};

// q[s1, s2] = (1/N) sum_t p[s1 - m1 t1(t), s2 - m2 t2(t)] over the new K1n x K2n grid
__global__ void __launch_bounds__(kThreads) k_linform2_level(const double* __restrict__ p, int64_t k1o, int64_t k2o,
                                                             Lin2Level L, double* __restrict__ q, int64_t k1n,
                                                             int64_t k2n) {
    const int64_t total = k1n * k2n;
    for (int64_t idx = blockIdx.x * (int64_t)kThreads + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * kThreads) {
        const int64_t s1 = idx / k2n, s2 = idx - s1 * k2n;
        double a0 = 0.0, a1 = 0.0;
        for (int t = 0; t < L.n; ++t) {
            const int64_t t1 = (L.flip & 1) ? L.n - 1 - t : t, t2 = (L.flip & 2) ? L.n - 1 - t : t;
            const int64_t k1 = s1 - L.m1 * t1, k2 = s2 - L.m2 * t2;
            if (k1 >= 0 && k1 < k1o && k2 >= 0 && k2 < k2o) {
                if (t & 1) a1 += p[k1 * k2o + k2];
                else a0 += p[k1 * k2o + k2];
            }
        }
        q[idx] = (a0 + a1) / (double)L.n;
    }
}

struct Src2 {
    double s1, s2;
    __device__ __forceinline__ double x(int b) const { return b == 0 ? s1 : s2; }
};

// sum over the K1 x K2 support of p G(h1 (m01 + 2 k1), h2 (m02 + 2 k2)), tiles of
// kTile entries [t_begin, t_end) into tiles[t - t_out0]
template <int NS>
__global__ void __launch_bounds__(kThreads) k_linform2_eval(const lq_insn* __restrict__ prog, int n_insn, int result,
                                                            const double* __restrict__ p, int64_t K1, int64_t K2,
                                                            double h1, double m01, double h2, double m02,
                                                            int64_t t_begin, int64_t t_end, int64_t t_out0,
                                                            double* __restrict__ tiles) {
    __shared__ double sh[8];
    double slot[NS];
    const int64_t K = K1 * K2;
    for (int64_t tile = t_begin + blockIdx.x; tile < t_end; tile += gridDim.x) {
        double s = 0.0;
        #pragma unroll 1
        for (int q = 0; q < kPts; ++q) {
            const int64_t k = tile * kTile + (int64_t)q * kThreads + threadIdx.x;
            if (k < K) {
                const double w = p[k];
                if (w != 0.0) {
                    const int64_t k1 = k / K2, k2 = k - k1 * K2;
                    Src2 src{h1 * (m01 + 2.0 * (double)k1), h2 * (m02 + 2.0 * (double)k2)};
                    s += w * run_program<NS>(prog, n_insn, result, src, slot);
                }
            }
        }
        s = block_sum(s, sh);
        if (threadIdx.x == 0) tiles[tile - t_out0] = s;
    }
}

// sum_k p[k] G(alpha + h (m0 + 2k)) over tiles of kTile support points
// (thread-strided inside the tile, block_sum tree): tiles [t_begin, t_end),
// partial of tile t to tiles[t - t_out0].
template <int NS>
__global__ void __launch_bounds__(kThreads) k_linform_eval(const lq_insn* __restrict__ prog, int n_insn, int result,
                                                           const double* __restrict__ p, int64_t K, double alpha,
                                                           double h, double m0, int64_t t_begin, int64_t t_end,
                                                           int64_t t_out0, double* __restrict__ tiles) {
    __shared__ double sh[8];
    double slot[NS];
    for (int64_t tile = t_begin + blockIdx.x; tile < t_end; tile += gridDim.x) {
        double s = 0.0;
        #pragma unroll 1
        for (int q = 0; q < kPts; ++q) {
            const int64_t k = tile * kTile + (int64_t)q * kThreads + threadIdx.x;
            if (k < K) {
                const double w = p[k];
                if (w != 0.0) {
                    UnivSrc src{fma(h, m0 + 2.0 * (double)k, alpha)};
                    s += w * run_program<NS>(prog, n_insn, result, src, slot);
                }
            }
        }
        s = block_sum(s, sh);
        if (threadIdx.x == 0) tiles[tile - t_out0] = s;
    }
}

// ============================================================ CF (exp-abs) MDI
// One CTA per frequency node w: each warp forms phi_j(w) = sum_t e^{i w beta_j y_t}
// for its directions j (lanes over t), accumulating log|phi_j| and arg phi_j;
// the 8 warps' (log, arg) partials combine in fixed order.  val[k] =
// weight_k * |kappa|/(kappa^2+w^2) * exp(sum log|phi|) cos(w alpha + sum arg).
__global__ void __launch_bounds__(kThreads) k_cf_expabs(const double* __restrict__ beta, const int32_t* __restrict__ counts,
                                                        int d, double alpha, const double* __restrict__ wn,
                                                        const double* __restrict__ ww, double kappa,
                                                        double* __restrict__ val, double* __restrict__ logmag) {
    __shared__ double sl[8], sa[8];
    const int k = blockIdx.x;
    const double w = wn[k];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double lsum = 0.0, asum = 0.0;
    for (int j = warp; j < d; j += kThreads / 32) {
        const int N = counts[j];
        const double cd = (double)N, inv = 1.0 / cd, th = w * beta[j];
        double re = 0.0, im = 0.0;
        for (int t = lane; t < N; t += 32) {
            const double y = exact_div((double)t + 0.5, cd, inv);
            double sn, cs;
            sincos(th * y, &sn, &cs);
            re += cs;
            im += sn;
        }
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            re += __shfl_xor_sync(0xffffffffu, re, o);
            im += __shfl_xor_sync(0xffffffffu, im, o);
        }
        lsum += log(hypot(re, im) * inv);
        asum += atan2(im, re);
    }
    if (lane == 0) { sl[warp] = lsum; sa[warp] = asum; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double L = 0.0, A = 0.0;
        for (int q = 0; q < kThreads / 32; ++q) { L += sl[q]; A += sa[q]; }
        const double ak = fabs(kappa);
        val[k] = ww[k] * ak / (kappa * kappa + w * w) * exp(L) * cos(w * alpha + A);
        logmag[k] = L;
    }
}

// Closed form of the same cluster sums on the midpoint grid y_t = (t + 1/2)/N:
// (1/N) sum_t e^{i th y_t} = e^{i th/2} sin(th/2) / (N sin(th/(2N))) (Dirichlet
// kernel), so each (w, j) costs two sines instead of N sincos; the phases sum
// to w (sum beta)/2 + pi (number of negative ratios), folded into alpha_half =
// alpha + (sum beta)/2 on the host.  One CTA per frequency node, threads over j.
__global__ void __launch_bounds__(kThreads) k_cf_expabs_closed(const double* __restrict__ beta,
                                                               const int32_t* __restrict__ counts, int d,
                                                               double alpha_half, const double* __restrict__ wn,
                                                               const double* __restrict__ ww, double kappa,
                                                               double* __restrict__ val, double* __restrict__ logmag) {
    __shared__ double sh[8];
    const int k = blockIdx.x;
    const double w = wn[k];
    double lsum = 0.0, neg = 0.0;
    for (int j = threadIdx.x; j < d; j += kThreads) {
        const double cd = (double)counts[j], h = 0.5 * w * beta[j];
        double r = 1.0;
        if (h != 0.0) r = sin(h) / (cd * sin(h / cd));
        lsum += log(fabs(r));
        neg += r < 0.0 ? 1.0 : 0.0;
    }
    lsum = block_sum(lsum, sh);
    neg = block_sum(neg, sh);
    if (threadIdx.x == 0) {
        const double ak = fabs(kappa);
        const double c = cos(w * alpha_half);
        val[k] = ww[k] * ak / (kappa * kappa + w * w) * exp(lsum) * (fmod(neg, 2.0) != 0.0 ? -c : c);
        logmag[k] = lsum;
    }
}

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
