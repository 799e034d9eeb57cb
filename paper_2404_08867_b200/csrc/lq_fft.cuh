// In-CTA complex FP64 FFT of N = 4096 points (Stockham autosort, three
// radix-16 passes, 256 threads x one 16-point butterfly per pass) for the
// correlation form of the Korobov chain sums.
//
// Shared-memory layout: element i lives at i + (i >> 4) (one pad slot per 16)
// so the stride-16 stores of the first pass spread over the banks.
#pragma once
#include <cstdint>

namespace lq {

constexpr int kFftN = 4096;
constexpr int kFftR = 16;
constexpr int kFftPad = kFftN + kFftN / 16;   // padded shared-memory length (double2)

__device__ __forceinline__ int fpad(int i) { return i + (i >> 4); }

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

// forward 16-point DFT of v (input in natural order; 4 x 4 Cooley-Tukey)
__device__ __forceinline__ void dft16(double2 (&v)[16]) {
    // 4-point DFTs over n2 for each n1: inputs v[n1 + 4 n2]
    #pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) dft4(v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]);
    // now v[n1 + 4 q] = T[n1][q]; twiddle by W16^(n1 q), W16 = e^{-2 pi i / 16}
    const double c1 = 0.92387953251128674, s1 = 0.38268343236508978;   // cos, sin(pi/8)
    const double c2 = 0.70710678118654757;                               // cos(pi/4)
    // W16^1 = (c1, -s1), W16^2 = (c2, -c2), W16^3 = (s1, -c1), W16^4 = -i,
    // W16^6 = (-c2, -c2), W16^9 = (-c1, s1)
    v[1 + 4 * 1] = cmul(v[1 + 4 * 1], make_double2(c1, -s1));
    v[1 + 4 * 2] = cmul(v[1 + 4 * 2], make_double2(c2, -c2));
    v[1 + 4 * 3] = cmul(v[1 + 4 * 3], make_double2(s1, -c1));
    v[2 + 4 * 1] = cmul(v[2 + 4 * 1], make_double2(c2, -c2));
    v[2 + 4 * 2] = cmul_mi(v[2 + 4 * 2]);
    v[2 + 4 * 3] = cmul(v[2 + 4 * 3], make_double2(-c2, -c2));
    v[3 + 4 * 1] = cmul(v[3 + 4 * 1], make_double2(s1, -c1));
    v[3 + 4 * 2] = cmul(v[3 + 4 * 2], make_double2(-c2, -c2));
    v[3 + 4 * 3] = cmul(v[3 + 4 * 3], make_double2(-c1, s1));
    // 4-point DFTs over n1 for each q: v[4 q + p] = X[q + 4 p] (digit-swapped;
    // callers read output k from v[dft16_slot(k)])
    #pragma unroll
    for (int q = 0; q < 4; ++q) dft4(v[4 * q + 0], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}

// register slot of DFT output k after dft16: k = q + 4 p lives in v[4 q + p]
__host__ __device__ constexpr int dft16_slot(int k) { return 4 * (k & 3) + (k >> 2); }

// One Stockham pass (sub-transform length Ns -> 16 Ns).  Thread j = threadIdx.x
// < N/16 owns inputs j + 256 r (r < 16).  W[k] = e^{-2 pi i k / N}.
//  * the inputs come from shared memory (LOAD) or are already in v;
//  * the outputs go to shared memory (STORE; positions (j / Ns) 16 Ns + j % Ns
//    + r Ns) or -- for the last pass, Ns = 256, whose outputs are exactly
//    j + 256 r -- stay in v in natural order.
// Callers keep the shared buffer consistent: a pass that loads must follow a
// __syncthreads() after the previous store.
template <bool LOAD, bool STORE>
__device__ __forceinline__ void fft_pass(double2 (&v)[16], double2* __restrict__ buf, int Ns,
                                         const double2* __restrict__ W) {
    const int j = threadIdx.x;
    if (LOAD) {
        #pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = buf[fpad(j + r * (kFftN / kFftR))];
    }
    const int k = j & (Ns - 1);
    if (Ns > 1) {
        const int step = k * (kFftN / (Ns * kFftR));
        #pragma unroll
        for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], __ldg(W + ((r * step) & (kFftN - 1))));
    }
    dft16(v);
    if (STORE) {
        __syncthreads();   // every thread has read its inputs of this buffer
        const int idxD = (j / Ns) * Ns * kFftR + k;
        #pragma unroll
        for (int r = 0; r < 16; ++r) buf[fpad(idxD + r * Ns)] = v[dft16_slot(r)];
        __syncthreads();
    } else {
        double2 t[16];
        #pragma unroll
        for (int r = 0; r < 16; ++r) t[r] = v[dft16_slot(r)];
        #pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = t[r];
    }
}

// Forward FFT: inputs j + 256 r in v (registers), outputs j + 256 r in v.
__device__ __forceinline__ void fft4096_regs(double2 (&v)[16], double2* __restrict__ buf,
                                             const double2* __restrict__ W) {
    fft_pass<false, true>(v, buf, 1, W);
    fft_pass<true, true>(v, buf, 16, W);
    fft_pass<true, false>(v, buf, 256, W);
}

// Forward FFT of the N values in buf (natural order in, natural order out).
__device__ __forceinline__ void fft4096(double2* __restrict__ buf, const double2* __restrict__ W) {
    double2 v[16];
    fft_pass<true, true>(v, buf, 1, W);
    fft_pass<true, true>(v, buf, 16, W);
    fft_pass<true, true>(v, buf, 256, W);
}

}  // namespace lq
