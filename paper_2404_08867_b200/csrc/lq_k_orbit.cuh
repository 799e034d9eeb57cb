// Device kernels of liblq, part of lq_kernels.cu's translation unit (included
// inside namespace lq): Korobov-orbit chain sums: direct (k_orbit, k_orbit_prod) and FFT form (k_orbit_fft, k_orbit_fft_quad).
#pragma once

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
