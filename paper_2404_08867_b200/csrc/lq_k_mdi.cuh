// Device kernels of liblq, part of lq_kernels.cu's translation unit (included
// inside namespace lq): MDI-LR: cluster sums and combine, level collapse (one / weighted / two forms), the exp-abs characteristic function.
#pragma once

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
