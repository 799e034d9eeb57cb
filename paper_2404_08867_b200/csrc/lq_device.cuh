// Device helpers for liblq (sm_100a): exact coordinates, modular stepping,
// deterministic reductions and the bytecode interpreter.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "lq.h"

namespace lq {

constexpr int kThreads = 256;              // every reduction kernel uses 256-thread CTAs
constexpr int kTile = LQ_TILE;             // points per tile
constexpr int kPts = kTile / kThreads;     // 16 consecutive points per thread

// ---------------------------------------------------------------- arithmetic

// RN(a / b) for doubles a >= 0, b > 0 in the normal range, given inv = RN(1/b):
// Markstein's correction step -- q within 1 ulp, the FMA residual is exact,
// and q + e*inv rounds to the correctly rounded quotient.  This reproduces
// numpy's IEEE division in lattice.points_block (lattice.py:104) and the
// Python-float node values (t+0.5)/n_i of transform.midpoint_grids
// (transform.py:177) bit for bit.
__device__ __forceinline__ double exact_div(double a, double b, double inv) {
    double q = a * inv;
    double e = fma(-q, b, a);
    return fma(e, inv, q);
}

// (a*b) mod n for a, b < 2^53, n < 2^53: quotient estimated in FP64, remainder
// exact in wrapping u64 arithmetic, then corrected (|error| is a few n).
__device__ __forceinline__ uint64_t mulmod_u64(uint64_t a, uint64_t b, uint64_t n, double ninv) {
    uint64_t lo = a * b;
    double qd = (double)a * (double)b * ninv;
    uint64_t q = qd <= 0.0 ? 0ull : (uint64_t)qd;
    int64_t r = (int64_t)(lo - q * n);
    while (r < 0) r += (int64_t)n;
    while (r >= (int64_t)n) r -= (int64_t)n;
    return (uint64_t)r;
}

// (x*z) mod n for n <= 2^31, any x < 2^32, with Shoup's precomputed
// zs = floor(z * 2^32 / n): the estimate q is floor(xz/n) or one less, so the
// wrapped difference lies in [0, 2n) and one VIADDMNMX finishes it.
__device__ __forceinline__ uint32_t mulmod_shoup(uint32_t x, uint32_t z, uint32_t zs, uint32_t n) {
    uint32_t q = __umulhi(x, zs);
    uint32_t r = x * z - q * n;
    return __viaddmin_u32(r, 0u - n, r);   // min(r - n, r) as unsigned
}

// One lattice step r <- (r + z) mod n for r, z < n <= 2^31: min(r+z, r+z-n)
// as unsigned, i.e. IADD + VIADDMNMX.  zm = z - n (mod 2^32).
__device__ __forceinline__ uint32_t step_mod(uint32_t r, uint32_t z, uint32_t zm) {
    return __viaddmin_u32(r, z, r + zm);
}

// The denormal 2^-1074 * r for integer r < 2^52, formed without a conversion
// instruction: bits {lo = r, hi = h} with h an opaque zero kept live in a
// register so ptxas does not re-materialise it per use.
__device__ __forceinline__ double denorm_of(uint32_t r, uint32_t h) {
    double x;
    asm("mov.b64 %0, {%1, %2};" : "=d"(x) : "r"(r), "r"(h));
    return x;
}

// ----------------------------------------------------------- reductions

// Deterministic CTA sum (256 threads).  Result valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double* sh /* >= 8 */) {
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < (kThreads / 32) ? sh[lane] : 0.0;
        #pragma unroll
        for (int o = 4; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;
}

// ------------------------------------------------ exact (order-free) sums
// A 192-bit two's-complement fixed-point accumulator with 2^-S resolution:
// every term is truncated to the grid once (deterministically), after which
// integer addition is associative, so the sum is the same for any order of
// the terms -- a permutation of the points, a reflected or inverted lattice
// (the reference sorts its terms for the same purpose, lattice.py:236-239)
// -- and for any tiling, block shape or rank count.  The host picks S so that
// n * max|term| < 2^188 (fix_scale) and rounds the result once (fix_to_double).
struct Fix3 {
    uint64_t w0, w1, w2;   // little-endian limbs
};

__device__ __forceinline__ Fix3 fix_zero() { return Fix3{0ull, 0ull, 0ull}; }

__device__ __forceinline__ void fix_add(Fix3& a, const Fix3& b) {
    asm("add.cc.u64 %0, %0, %3;\n\t"
        "addc.cc.u64 %1, %1, %4;\n\t"
        "addc.u64 %2, %2, %5;"
        : "+l"(a.w0), "+l"(a.w1), "+l"(a.w2)
        : "l"(b.w0), "l"(b.w1), "l"(b.w2));
}

// v * 2^S truncated toward zero, as 192-bit two's complement
__device__ __forceinline__ Fix3 fix_of(double v, int S) {
    const uint64_t bits = (uint64_t)__double_as_longlong(v);
    const int ex = (int)((bits >> 52) & 0x7ff);
    uint64_t m = bits & 0xfffffffffffffull;
    int sh;                                   // v = m 2^(sh - S) after the next two lines
    if (ex == 0) sh = -1074 + S;
    else { m |= 1ull << 52; sh = ex - 1075 + S; }
    Fix3 t = fix_zero();
    if (ex == 0x7ff || m == 0) return t;      // inf/nan never occur (finite products); zero
    if (sh < 0) {
        m = sh <= -64 ? 0ull : m >> -sh;
        sh = 0;
    }
    const int limb = sh >> 6, off = sh & 63;
    const uint64_t lo = m << off, hi = off ? m >> (64 - off) : 0ull;
    if (limb == 0) { t.w0 = lo; t.w1 = hi; }
    else if (limb == 1) { t.w1 = lo; t.w2 = hi; }
    else { t.w2 = lo; }
    if (bits >> 63) {                         // negate: ~t + 1
        t.w0 = ~t.w0; t.w1 = ~t.w1; t.w2 = ~t.w2;
        fix_add(t, Fix3{1ull, 0ull, 0ull});
    }
    return t;
}

__device__ __forceinline__ Fix3 fix_shfl_xor(const Fix3& a, int o) {
    return Fix3{__shfl_xor_sync(0xffffffffu, a.w0, o), __shfl_xor_sync(0xffffffffu, a.w1, o),
                __shfl_xor_sync(0xffffffffu, a.w2, o)};
}

// CTA sum of a Fix3 (NT threads); the result is valid in thread 0
template <int NT>
__device__ __forceinline__ Fix3 fix_block_sum(Fix3 a, Fix3* sh /* >= NT / 32 */) {
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) fix_add(a, fix_shfl_xor(a, o));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = a;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int w = 1; w < NT / 32; ++w) fix_add(a, sh[w]);
    return a;
}

// ----------------------------------------------------------- interpreter

enum : int32_t {
    OP_CONST = 0, OP_VAR = 1, OP_ACC_INIT = 2, OP_ACC_ADD = 3, OP_ACC_MUL = 4,
    OP_POW = 5, OP_RPOW = 6, OP_EXP = 7, OP_SIN = 8, OP_COS = 9, OP_ABS = 10,
    OP_ACC_ADDVAR = 11
};

__device__ __forceinline__ double ipow(double b, int k) {
    // numpy's b**k: square for k == 2, libm pow otherwise (exprcore.py:466-468)
    return k == 2 ? b * b : pow(b, (double)k);
}

// One-variable program input (MDI factors, outer functions G(s)).
struct UnivSrc {
    double y;
    __device__ __forceinline__ double x(int) const { return y; }
};

// Evaluate a program; Src::x(b) supplies variable b.  NS = slot capacity.
template <int NS, class Src>
__device__ __forceinline__ double run_program(const lq_insn* __restrict__ prog, int n_insn, int result,
                                              const Src& src, double* slot) {
    for (int k = 0; k < n_insn; ++k) {
        const lq_insn in = prog[k];
        double v;
        switch (in.op) {
            case OP_CONST: slot[in.a] = in.c; break;
            case OP_VAR: slot[in.a] = src.x(in.b); break;
            case OP_ACC_INIT: slot[in.a] = in.c; break;
            case OP_ACC_ADD: slot[in.a] = slot[in.a] + in.c * slot[in.b]; break;
            case OP_ACC_ADDVAR: slot[in.a] = slot[in.a] + in.c * src.x(in.b); break;
            case OP_ACC_MUL: slot[in.a] = slot[in.a] * slot[in.b]; break;
            case OP_POW: slot[in.a] = ipow(slot[in.b], in.n); break;
            case OP_RPOW: v = slot[in.b]; slot[in.a] = 1.0 / (in.n == 1 ? v : ipow(v, in.n)); break;
            case OP_EXP: slot[in.a] = exp(slot[in.b]); break;
            case OP_SIN: slot[in.a] = sin(slot[in.b]); break;
            case OP_COS: slot[in.a] = cos(slot[in.b]); break;
            case OP_ABS: slot[in.a] = fabs(slot[in.b]); break;
            default: break;
        }
    }
    return slot[result];
}

}  // namespace lq
