// Device kernels of liblq, part of lq_kernels.cu's translation unit (included
// inside namespace lq): points_block, the closed-family per-index sums (k_fam) and the product family (k_prod).
#pragma once

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
