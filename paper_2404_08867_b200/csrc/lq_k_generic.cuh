// Device kernels of liblq, part of lq_kernels.cu's translation unit (included
// inside namespace lq): the bytecode interpreter kernels: plain sums, Monte Carlo, tensor grids, element-wise eval_array.
#pragma once

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
                    LatSrc64 src{i < n ? i : i % n, n, n_d, inv_n, ninv_mm, (const uint64_t*)ztab};
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
    __shared__ uint32_t gapd[kMaxAxes];
    double slot[NS];
    uint32_t digit[kMaxAxes];
    // each thread's odometer is set up once by division and carried to the
    // CTA's next tile by adding the mixed-radix digits of G kTile - kPts
    if (threadIdx.x == 0) {
        uint64_t rem = (uint64_t)gridDim.x * kTile - kPts;
        for (int k = 0; k < d; ++k) {
            const uint64_t c = (uint64_t)counts[k];
            gapd[k] = (uint32_t)(rem % c);
            rem /= c;
        }
    }
    __syncthreads();
    {
        uint64_t rem = base + (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kPts;
        for (int k = 0; k < d; ++k) {
            const uint64_t c = (uint64_t)counts[k];
            digit[k] = (uint32_t)(rem % c);
            rem /= c;
        }
    }
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t s0 = base + (uint64_t)tile * kTile + (uint64_t)threadIdx.x * kPts;
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
        uint32_t carry = 0;
        for (int k = 0; k < d; ++k) {
            const uint64_t c = (uint64_t)counts[k];
            const uint64_t t = (uint64_t)digit[k] + gapd[k] + carry;
            carry = t >= c;
            digit[k] = (uint32_t)(carry ? t - c : t);
        }
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
