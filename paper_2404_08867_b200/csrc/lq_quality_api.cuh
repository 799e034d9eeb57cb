// Quality measures and constructions behind the C ABI (included at the end of
// lq_api.cu): P_alpha / shift-averaged worst-case error sums (exact Fix3
// accumulation), CBC construction and the Korobov search.
#pragma once
// ============================================================ quality measures
namespace {

int b2_table(lq_ctx* c, uint32_t n, double** out) {
    void* p;
    int rc;
    if ((rc = dev_buf(c, B_AUX2, sizeof(double) * n, &p))) return rc;
    const double nd = (double)n;
    lq::k_b2_table<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, c->stream>>>(n, nd, 1.0 / nd, (double*)p);
    c->launches++;
    CK(cudaGetLastError());
    *out = (double*)p;
    return LQ_OK;
}

bool improves(double val, double best) { return val < best - 1e-9 * std::fabs(best); }   // lattice.py:248-252

// Scale 2^S of the exact fixed-point sums (lq::Fix3): count terms of
// magnitude <= bound stay below 2^186 (two bits of headroom under the sign).
int fix_scale(double bound, double count) {
    const double lb = std::log2(std::max(bound, 1e-300)) + std::log2(std::max(count, 1.0));
    return std::max(-900, std::min(1100, 186 - (int)std::ceil(lb)));
}

// The 192-bit two's-complement fixed-point value v 2^-S, rounded once to the
// nearest double (ties to even).
double fix_to_double(lq::Fix3 v, int S) {
    uint64_t w[3] = {v.w0, v.w1, v.w2};
    const bool neg = w[2] >> 63;
    if (neg) {   // magnitude: ~v + 1
        w[0] = ~w[0]; w[1] = ~w[1]; w[2] = ~w[2];
        for (int i = 0; i < 3 && ++w[i] == 0; ++i) {}
    }
    int top = -1;
    for (int i = 2; i >= 0 && top < 0; --i)
        if (w[i]) top = 64 * i + 63 - __builtin_clzll(w[i]);
    if (top < 0) return 0.0;
    auto bit = [&](int p) -> uint64_t { return p < 0 ? 0ull : (w[p >> 6] >> (p & 63)) & 1ull; };
    uint64_t m = 0;
    for (int p = top; p > top - 53; --p) m = (m << 1) | bit(p);
    int e = top - 52;   // |v| = m 2^e + (the bits below)
    if (top >= 53 && bit(top - 53)) {
        bool sticky = false;
        for (int p = top - 54; p >= 0 && !sticky; --p) sticky = bit(p);
        if (sticky || (m & 1ull)) {
            if (++m == (1ull << 53)) { m >>= 1; ++e; }
        }
    }
    const double out = std::ldexp((double)m, e - S);
    return neg ? -out : out;
}

// max |1 + g (B + beta)| over B in [lo, hi]
double bfactor_bound(double g, double beta, double lo, double hi) {
    return std::max(std::fabs(1.0 + g * (lo + beta)), std::fabs(1.0 + g * (hi + beta))) * (1.0 + 1e-12);
}

constexpr size_t kSmemTable = 200 * 1024;

template <class K>
int persistent_grid(lq_ctx* c, K kern, size_t smem) {
    if (smem > 48 * 1024) {
        cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)kern, lq::kThreads, smem);
    return c->sm_count * std::max(per_sm, 1);
}

}  // namespace

extern "C" {

int lq_bprod_sum(lq_ctx* c, int32_t alpha, int32_t d, uint64_t n, const uint64_t* z, const double* g, double beta,
                 uint64_t i_begin, uint64_t i_end, double* sum_out) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (alpha != 2 && alpha != 4) return fail(LQ_ERR_VALUE, "alpha must be 2 or 4, got %d", alpha);
    if ((rc = check_lattice(n, z, d))) return rc;
    if (n > (1ull << 31)) return fail(LQ_ERR_UNSUPPORTED, "quality sums support n <= 2^31");
    if (!g || !sum_out || i_end < i_begin) return fail(LQ_ERR_VALUE, "bad arguments");
    if (i_end == i_begin) {
        *sum_out = 0.0;
        return LQ_OK;
    }
    std::vector<lq::QDim> tab(d);
    for (int j = 0; j < d; ++j) {
        tab[j].z = (uint32_t)z[j];
        tab[j].zs = (uint32_t)(((uint64_t)z[j] << 32) / n);
        tab[j].g = g[j];
    }
    void* dt;
    if ((rc = upload(c, B_TAB, tab.data(), sizeof(lq::QDim) * d, &dt))) return rc;
    const int64_t ntiles = (int64_t)((i_end - i_begin + lq::kTile - 1) / lq::kTile);
    void *tiles, *red;
    if ((rc = dev_buf(c, B_TILES, sizeof(lq::Fix3) * ntiles, &tiles))) return rc;
    if ((rc = dev_buf(c, B_RED0, sizeof(lq::Fix3), &red))) return rc;
    const double nd = (double)n;
    // B_2 in [-1/12, 1/6], B_4 in [-1/30, 7/240]
    const double blo = alpha == 2 ? -1.0 / 12.0 : -1.0 / 30.0, bhi = alpha == 2 ? 1.0 / 6.0 : 7.0 / 240.0;
    double bound = 1.0;
    for (int j = 0; j < d; ++j) bound *= bfactor_bound(g[j], beta, blo, bhi);
    const int S = fix_scale(bound, (double)(i_end - i_begin));
    t_begin(c);
    if (alpha == 2)
        lq::k_bprod<2><<<(unsigned)ntiles, lq::kThreads, 0, c->stream>>>((const lq::QDim*)dt, d, (uint32_t)n, nd, 1.0 / nd, beta, i_begin, i_end, S, (lq::Fix3*)tiles);
    else
        lq::k_bprod<4><<<(unsigned)ntiles, lq::kThreads, 0, c->stream>>>((const lq::QDim*)dt, d, (uint32_t)n, nd, 1.0 / nd, beta, i_begin, i_end, S, (lq::Fix3*)tiles);
    t_end(c);
    CK(cudaGetLastError());
    lq::k_fix_reduce<<<1, lq::kThreads, 0, c->stream>>>((const lq::Fix3*)tiles, ntiles, (lq::Fix3*)red);
    c->launches++;
    CK(cudaGetLastError());
    lq::Fix3 tot;
    CK(cudaMemcpyAsync(&tot, red, sizeof(tot), cudaMemcpyDeviceToHost, c->stream));
    c->d2h_bytes += (int64_t)sizeof(tot);
    CK(cudaStreamSynchronize(c->stream));
    *sum_out = fix_to_double(tot, S);
    return LQ_OK;
}

int lq_cbc_construct(lq_ctx* c, uint64_t n, int32_t d, const double* gamma, double beta, const int64_t* cands,
                     int64_t ncand, int64_t* z_out) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (n < 2 || n > (1ull << 31)) return fail(LQ_ERR_VALUE, "CBC supports 2 <= n <= 2^31, got %llu", (unsigned long long)n);
    if (d < 1 || !gamma || !z_out) return fail(LQ_ERR_VALUE, "bad arguments");
    if (d > 1 && (ncand < 1 || !cands)) return fail(LQ_ERR_VALUE, "no candidates");
    for (int64_t k = 0; k < ncand; ++k)
        if (cands[k] < 1 || (uint64_t)cands[k] >= n) return fail(LQ_ERR_VALUE, "candidate out of range");
    double* b2;
    if ((rc = b2_table(c, (uint32_t)n, &b2))) return rc;
    void *basev, *dc, *dv;
    if ((rc = dev_buf(c, B_AUX3, sizeof(double) * n, &basev))) return rc;
    lq::k_cbc_init<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, c->stream>>>((uint32_t)n, b2, gamma[0], beta, (double*)basev);
    c->launches++;
    CK(cudaGetLastError());
    z_out[0] = 1;
    if (d == 1) return lq_sync(c);
    if ((rc = upload(c, B_AUX0, cands, sizeof(int64_t) * ncand, &dc))) return rc;
    if ((rc = dev_buf(c, B_OUT, sizeof(lq::Fix3) * ncand, &dv))) return rc;
    std::vector<lq::Fix3> vals(ncand);
    const bool smem = sizeof(double) * n <= kSmemTable;
    const size_t shbytes = smem ? sizeof(double) * n : 0;
    const int grid = smem ? persistent_grid(c, lq::k_cbc_eval<true>, shbytes) : persistent_grid(c, lq::k_cbc_eval<false>, 0);
    double anchor = 1.0 + gamma[0] * beta;
    double bound = bfactor_bound(gamma[0], beta, -1.0 / 12.0, 1.0 / 6.0);   // of the base column
    for (int s = 1; s < d; ++s) {
        const double g = gamma[s];
        anchor *= 1.0 + g * beta;
        const double gb = bfactor_bound(g, beta, -1.0 / 12.0, 1.0 / 6.0);
        const int S = fix_scale(bound * gb, (double)n);
        t_begin(c);
        if (smem)
            lq::k_cbc_eval<true><<<std::min<int64_t>(grid, ncand), lq::kThreads, shbytes, c->stream>>>((uint32_t)n, b2, (const double*)basev, g, beta, (const int64_t*)dc, ncand, S, (lq::Fix3*)dv);
        else
            lq::k_cbc_eval<false><<<std::min<int64_t>(grid, ncand), lq::kThreads, 0, c->stream>>>((uint32_t)n, b2, (const double*)basev, g, beta, (const int64_t*)dc, ncand, S, (lq::Fix3*)dv);
        t_end(c);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(vals.data(), dv, sizeof(lq::Fix3) * ncand, cudaMemcpyDeviceToHost, c->stream));
        c->d2h_bytes += (int64_t)(sizeof(lq::Fix3) * ncand);
        CK(cudaStreamSynchronize(c->stream));
        bound *= gb;
        int64_t best = -1;
        double best_val = INFINITY;
        for (int64_t k = 0; k < ncand; ++k) {
            const double val = fix_to_double(vals[k], S) / (double)n - anchor;
            if (best < 0 || improves(val, best_val)) {
                best = k;
                best_val = val;
            }
        }
        z_out[s] = cands[best];
        lq::k_cbc_update<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, c->stream>>>((uint32_t)n, b2, g, beta, (uint32_t)cands[best], (double*)basev);
        c->launches++;
        CK(cudaGetLastError());
    }
    return lq_sync(c);
}

int lq_korobov_values(lq_ctx* c, uint64_t n, int32_t d, const double* gamma, double beta, const int64_t* cands,
                      int64_t ncand, double* sums_out) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (n < 2 || n > (1ull << 31)) return fail(LQ_ERR_VALUE, "Korobov search supports 2 <= n <= 2^31");
    if (d < 1 || !gamma || !sums_out || ncand < 0) return fail(LQ_ERR_VALUE, "bad arguments");
    if (ncand == 0) return LQ_OK;
    for (int64_t k = 0; k < ncand; ++k)
        if (cands[k] < 1 || (uint64_t)cands[k] >= n) return fail(LQ_ERR_VALUE, "candidate out of range");
    double* b2;
    if ((rc = b2_table(c, (uint32_t)n, &b2))) return rc;
    void *dg, *dc, *dv;
    if ((rc = upload(c, B_AUX1, gamma, sizeof(double) * d, &dg))) return rc;
    if ((rc = upload(c, B_AUX0, cands, sizeof(int64_t) * ncand, &dc))) return rc;
    if ((rc = dev_buf(c, B_OUT, sizeof(lq::Fix3) * ncand, &dv))) return rc;
    double bound = 1.0;
    for (int j = 0; j < d; ++j) bound *= bfactor_bound(gamma[j], beta, -1.0 / 12.0, 1.0 / 6.0);
    const int S = fix_scale(bound, (double)n);
    const bool smem = sizeof(double) * n <= kSmemTable;
    const size_t shbytes = smem ? sizeof(double) * n : 0;
    const int grid = smem ? persistent_grid(c, lq::k_korobov<true>, shbytes) : persistent_grid(c, lq::k_korobov<false>, 0);
    t_begin(c);
    if (smem)
        lq::k_korobov<true><<<std::min<int64_t>(grid, ncand), lq::kThreads, shbytes, c->stream>>>((uint32_t)n, d, b2, (const double*)dg, beta, (const int64_t*)dc, ncand, S, (lq::Fix3*)dv);
    else
        lq::k_korobov<false><<<std::min<int64_t>(grid, ncand), lq::kThreads, 0, c->stream>>>((uint32_t)n, d, b2, (const double*)dg, beta, (const int64_t*)dc, ncand, S, (lq::Fix3*)dv);
    t_end(c);
    CK(cudaGetLastError());
    std::vector<lq::Fix3> vals(ncand);
    CK(cudaMemcpyAsync(vals.data(), dv, sizeof(lq::Fix3) * ncand, cudaMemcpyDeviceToHost, c->stream));
    c->d2h_bytes += (int64_t)(sizeof(lq::Fix3) * ncand);
    CK(cudaStreamSynchronize(c->stream));
    for (int64_t k = 0; k < ncand; ++k) sums_out[k] = fix_to_double(vals[k], S);
    return LQ_OK;
}

}  // extern "C"
