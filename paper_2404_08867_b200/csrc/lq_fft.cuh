// In-CTA complex FP64 FFT of N = 4096 points for the correlation form of the
// Korobov chain sums: Stockham autosort, radix R = 16 (three
// passes, 256 threads; default) or R = 8 (four passes, 512 threads: measured
// 19.7 vs 14.5 ms on cfg5), one R-point butterfly per thread per pass.
//
// Shared-memory layout: element i lives at i + i / R (one pad slot per R), so
// the stride-R stores of the first pass spread over the banks.  Radix-16
// twiddles come from small shared tables (26 KB, see fft_load_twiddles).
#pragma once
#include <cstdint>

#ifndef LQ_FFT_RADIX
#define LQ_FFT_RADIX 16
#endif

namespace lq {

constexpr int kFftN = 4096;
constexpr int kFftR = LQ_FFT_RADIX;
constexpr int kFftThreads = kFftN / kFftR;
constexpr int kFftLogR = kFftR == 16 ? 4 : 3;
constexpr int kFftPad = kFftN + kFftN / kFftR;   // padded shared-memory length (double2)
// Radix-16 twiddle tables in shared memory, laid out [q][k] so that the lanes
// of a warp (consecutive k) read consecutive entries:
//   pass Ns = 256: L3[q][k] = W^(q k), H3[q][k] = W^(4 q k), q = 1..3, k < 256;
//                  W^(r k) = L3[r mod 4] H3[r div 4] (6 loads, 9 products)
//   pass Ns = 16:  T2[r][k] = W^(16 r k), r = 1..15, k < 16 (all of them)
// (W = e^{-2 pi i / N}).
constexpr int kFftTw3 = 3 * 256, kFftTw2 = 15 * 16;
constexpr int kFftTwAll = 2 * kFftTw3 + kFftTw2;
#ifndef LQ_FFT_EXPTAB
#define LQ_FFT_EXPTAB 1
#endif
#ifndef LQ_FFT_EXPBITS
#define LQ_FFT_EXPBITS 6
#endif
constexpr int kFftExpBits = LQ_FFT_EXPBITS;
constexpr int kFftExpTab = LQ_FFT_EXPTAB ? 1 << kFftExpBits : 0;   // (2^(j/2^EB), 2^(-j/2^EB)) for the pair outer
constexpr int kFftSmem = (kFftPad + (kFftR == 16 ? kFftTwAll : 0) + kFftExpTab) * 16;   // bytes per CTA

// Build the radix-16 tables from the global table W[k] = e^{-2 pi i k / N}.
__device__ __forceinline__ void fft_load_twiddles(double2* __restrict__ tw, const double2* __restrict__ W,
                                                  int nthreads = kFftThreads) {
    if constexpr (kFftR != 16) return;   // radix 8 reads the global table directly
    for (int i = threadIdx.x; i < kFftTw3; i += nthreads) {
        const int q = i / 256 + 1, k = i & 255;
        tw[i] = __ldg(W + q * k);
        tw[kFftTw3 + i] = __ldg(W + ((4 * q * k) & (kFftN - 1)));
    }
    for (int i = threadIdx.x; i < kFftTw2; i += nthreads) {
        const int r = i / 16 + 1, k = i & 15;
        tw[2 * kFftTw3 + i] = __ldg(W + ((16 * r * k) & (kFftN - 1)));
    }
}

__device__ __forceinline__ int fpad(int i) { return i + (i >> kFftLogR); }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// a * (-i)
__device__ __forceinline__ double2 cmul_mi(double2 a) { return make_double2(a.y, -a.x); }

// forward 4-point DFT in place: X_q = sum_n a_n (-i)^(n q)
__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
    const double2 s02 = cadd(a0, a2), d02 = csub(a0, a2);
    const double2 s13 = cadd(a1, a3), d13 = cmul_mi(csub(a1, a3));
    a0 = cadd(s02, s13);
    a2 = csub(s02, s13);
    a1 = cadd(d02, d13);
    a3 = csub(d02, d13);
}

// forward 8-point DFT (2 x 4): output k = q + 4 p in v[2 q + p]
__device__ __forceinline__ void dft8(double2 (&v)[8]) {
    dft4(v[0], v[2], v[4], v[6]);   // n1 = 0: T[0][q] at v[2q]
    dft4(v[1], v[3], v[5], v[7]);   // n1 = 1: T[1][q] at v[2q + 1]
    const double c = 0.70710678118654757;
    v[3] = cmul(v[3], make_double2(c, -c));    // W8^1
    v[5] = cmul_mi(v[5]);                      // W8^2
    v[7] = cmul(v[7], make_double2(-c, -c));   // W8^3
    #pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double2 a = v[2 * q], b = v[2 * q + 1];
        v[2 * q] = cadd(a, b);
        v[2 * q + 1] = csub(a, b);
    }
}

// forward 16-point DFT (4 x 4): output k = q + 4 p in v[4 q + p].  The
// second-stage twiddles are fused into the butterflies (FMA "tangent" form):
// W^2 x = c2 (x.x + x.y, x.y - x.x) and W^1 t = c1 (t.x + tan t.y, t.y - tan t.x)
// are applied as the multiplicand of the butterfly's FMA, and a1 +- a3 =
// W^q (x1 +- W^2q x3): 148 FP64 instructions instead of 160.
__device__ __forceinline__ void dft16(double2 (&v)[16]) {
    #pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) dft4(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]);
    const double c1 = 0.92387953251128674, t1 = 0.41421356237309503;   // cos, tan(pi/8)
    const double c2 = 0.70710678118654757;                               // cos(pi/4)
    dft4(v[0], v[1], v[2], v[3]);                                        // q = 0: no twiddles
    {   // q = 2: W^2, W^4 = -i, W^6
        const double2 a0 = v[8], x1 = v[9], x2 = v[10], x3 = v[11];
        const double s02x = a0.x + x2.y, s02y = a0.y - x2.x, d02x = a0.x - x2.y, d02y = a0.y + x2.x;
        const double u1 = x1.x + x1.y, w1 = x1.y - x1.x;                // W^2 x1 = c2 (u1, w1)
        const double u3 = x3.y - x3.x, m3 = x3.x + x3.y;                // W^6 x3 = c2 (u3, -m3)
        const double Sx = u1 + u3, Sy = w1 - m3, Dx = u1 - u3, Dy = w1 + m3;
        v[8] = make_double2(fma(c2, Sx, s02x), fma(c2, Sy, s02y));
        v[10] = make_double2(fma(-c2, Sx, s02x), fma(-c2, Sy, s02y));
        v[9] = make_double2(fma(c2, Dy, d02x), fma(-c2, Dx, d02y));
        v[11] = make_double2(fma(-c2, Dy, d02x), fma(c2, Dx, d02y));
    }
    {   // q = 1: W^1, W^2, W^3 = W^1 W^2
        const double2 a0 = v[4], x1 = v[5], x2 = v[6], x3 = v[7];
        const double u2 = x2.x + x2.y, w2 = x2.y - x2.x;
        const double s02x = fma(c2, u2, a0.x), s02y = fma(c2, w2, a0.y);
        const double d02x = fma(-c2, u2, a0.x), d02y = fma(-c2, w2, a0.y);
        const double u3 = x3.x + x3.y, w3 = x3.y - x3.x;
        const double tpx = fma(c2, u3, x1.x), tpy = fma(c2, w3, x1.y);    // x1 + W^2 x3
        const double tmx = fma(-c2, u3, x1.x), tmy = fma(-c2, w3, x1.y);  // x1 - W^2 x3
        const double gx = fma(t1, tpy, tpx), gy = fma(-t1, tpx, tpy);     // W^1 tp / c1
        const double hx = fma(t1, tmy, tmx), hy = fma(-t1, tmx, tmy);     // W^1 tm / c1
        v[4] = make_double2(fma(c1, gx, s02x), fma(c1, gy, s02y));
        v[6] = make_double2(fma(-c1, gx, s02x), fma(-c1, gy, s02y));
        v[5] = make_double2(fma(c1, hy, d02x), fma(-c1, hx, d02y));
        v[7] = make_double2(fma(-c1, hy, d02x), fma(c1, hx, d02y));
    }
    {   // q = 3: W^3, W^6, W^9 = W^3 W^6
        const double2 a0 = v[12], x1 = v[13], x2 = v[14], x3 = v[15];
        const double u2 = x2.y - x2.x, w2 = -(x2.x + x2.y);            // W^6 x2 = c2 (u2, w2)
        const double s02x = fma(c2, u2, a0.x), s02y = fma(c2, w2, a0.y);
        const double d02x = fma(-c2, u2, a0.x), d02y = fma(-c2, w2, a0.y);
        const double u3 = x3.y - x3.x, w3 = -(x3.x + x3.y);
        const double tpx = fma(c2, u3, x1.x), tpy = fma(c2, w3, x1.y);    // x1 + W^6 x3
        const double tmx = fma(-c2, u3, x1.x), tmy = fma(-c2, w3, x1.y);
        const double gx = fma(t1, tpx, tpy), gy = fma(t1, tpy, -tpx);     // W^3 tp / c1
        const double hx = fma(t1, tmx, tmy), hy = fma(t1, tmy, -tmx);
        v[12] = make_double2(fma(c1, gx, s02x), fma(c1, gy, s02y));
        v[14] = make_double2(fma(-c1, gx, s02x), fma(-c1, gy, s02y));
        v[13] = make_double2(fma(c1, hy, d02x), fma(-c1, hx, d02y));
        v[15] = make_double2(fma(-c1, hy, d02x), fma(c1, hx, d02y));
    }
}

template <int R>
__device__ __forceinline__ void dftR(double2 (&v)[R]) {
    if constexpr (R == 16) dft16(v);
    else dft8(v);
}

// register slot of DFT output k after dftR
__host__ __device__ constexpr int dft_slot(int k) {
    return kFftR == 16 ? 4 * (k & 3) + (k >> 2) : 2 * (k & 3) + (k >> 2);
}

// One Stockham pass (sub-transform length Ns -> R Ns).  Thread j < N/R owns
// inputs j + (N/R) r, r < R.  W: R = 16 -> the shared tables of
// fft_load_twiddles; R = 8 -> the global table e^{-2 pi i k / N}.
//  * the inputs come from shared memory (LOAD) or are already in v;
//  * the outputs go to shared memory (STORE; positions (j / Ns) R Ns + j % Ns
//    + r Ns) or -- for the last pass, Ns = N/R, whose outputs are exactly
//    j + (N/R) r -- stay in v in natural order.
// A pass that loads must follow a __syncthreads() after the previous store.
// Barrier of the threads that share one transform: the whole CTA
// (__syncthreads) or, NAMED, the 256-thread group with barrier id `bar`
// (k_orbit_fft_dual runs two transforms per CTA).
template <bool NAMED>
__device__ __forceinline__ void fft_bar(int bar) {
    if constexpr (NAMED) asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(kFftThreads) : "memory");
    else __syncthreads();
}

template <bool LOAD, bool STORE, bool NAMED = false>
__device__ __forceinline__ void fft_pass(double2 (&v)[kFftR], double2* __restrict__ buf, int Ns,
                                         const double2* __restrict__ W, int j = threadIdx.x, int bar = 0) {
    if (LOAD) {
        #pragma unroll
        for (int r = 0; r < kFftR; ++r) v[r] = buf[fpad(j + r * kFftThreads)];
    }
    const int k = j & (Ns - 1);
    if (Ns > 1) {
        const int step = k * (kFftN / (Ns * kFftR));
        if (kFftR == 16 && Ns == 16) {
            const double2* __restrict__ T = W + 2 * kFftTw3;
            #pragma unroll
            for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], T[(r - 1) * 16 + k]);
        } else if constexpr (kFftR == 16) {
            // W^(r step), r = r0 + 4 r1, as W^(r0 step) W^(4 r1 step): six
            // conflict-free shared-table loads instead of fifteen global ones
            const double2* __restrict__ L = W;
            const double2* __restrict__ H = W + kFftTw3;
            double2 lo[4], hi[4];
            #pragma unroll
            for (int q = 1; q < 4; ++q) {
                lo[q] = L[(q - 1) * Ns + k];
                hi[q] = H[(q - 1) * Ns + k];
            }
            #pragma unroll
            for (int r = 1; r < 16; ++r) {
                const int r0 = r & 3, r1 = r >> 2;
                const double2 w = r0 == 0 ? hi[r1] : r1 == 0 ? lo[r0] : cmul(lo[r0], hi[r1]);
                v[r] = cmul(v[r], w);
            }
        } else {
            #pragma unroll
            for (int r = 1; r < kFftR; ++r) v[r] = cmul(v[r], __ldg(W + ((r * step) & (kFftN - 1))));
        }
    }
    dftR<kFftR>(v);
    if (STORE) {
        fft_bar<NAMED>(bar);   // every thread has read its inputs of this buffer
        const int idxD = (j / Ns) * Ns * kFftR + k;
        #pragma unroll
        for (int r = 0; r < kFftR; ++r) buf[fpad(idxD + r * Ns)] = v[dft_slot(r)];
        fft_bar<NAMED>(bar);
    } else {
        double2 t[kFftR];
        #pragma unroll
        for (int r = 0; r < kFftR; ++r) t[r] = v[dft_slot(r)];
        #pragma unroll
        for (int r = 0; r < kFftR; ++r) v[r] = t[r];
    }
}

// Forward FFT, inputs j + (N/R) r in v (registers).  The last pass leaves its
// outputs -- the same positions -- in v, or stores them (natural order) to buf.
template <bool LAST_TO_SMEM, bool NAMED = false>
__device__ __forceinline__ void fft4096_regs(double2 (&v)[kFftR], double2* __restrict__ buf,
                                             const double2* __restrict__ W, int j = threadIdx.x, int bar = 0) {
    fft_pass<false, true, NAMED>(v, buf, 1, W, j, bar);
    #pragma unroll
    for (int Ns = kFftR; Ns < kFftN / kFftR; Ns *= kFftR) fft_pass<true, true, NAMED>(v, buf, Ns, W, j, bar);
    fft_pass<true, LAST_TO_SMEM, NAMED>(v, buf, kFftN / kFftR, W, j, bar);
}

// Forward FFT of the N values in buf (natural order in, natural order out).
__device__ __forceinline__ void fft4096(double2* __restrict__ buf, const double2* __restrict__ W) {
    double2 v[kFftR];
    #pragma unroll
    for (int Ns = 1; Ns < kFftN; Ns *= kFftR) fft_pass<true, true>(v, buf, Ns, W);
}

}  // namespace lq
