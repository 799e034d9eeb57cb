// liblq C ABI (include/lq.h): context, argument validation, table building
// and kernel launches.  Host code only; kernels live in lq_kernels.cu, which
// this translation unit includes so that template instantiations stay local.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <string>
#include <vector>
#include <unordered_map>
#include <algorithm>

#include "lq_kernels.cu"

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess)                                                        \
            return fail(LQ_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                          \
    } while (0)

enum Buf { B_TAB = 0, B_TILES, B_RED0, B_RED1, B_OUT, B_PROG, B_AUX0, B_AUX1, B_AUX2, B_AUX3, B_PART, B_FAC, B_NODES, B_FFTW, B_FFTH, B_NBUF };

}  // namespace

int lq_internal_fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

cudaKernel_t lq_jit_lattice_kernel(const lq_jit* j);
cudaKernel_t lq_jit_tensor_kernel(const lq_jit* j);

struct lq_ctx {
    int device = 0;
    int sm_count = 0;
    int cc_major = 0, cc_minor = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    void* dbuf[B_NBUF] = {};
    size_t dcap[B_NBUF] = {};
    void* hpin = nullptr;      // pinned host staging
    size_t hcap = 0;
    size_t hoff = 0;           // uploads staged since the stream last drained: [0, hoff) may be in flight
    bool timing = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    float last_ms = 0.f;
    int64_t launches = 0;
    bool fft_w = false;        // twiddles computed in dbuf[B_FFTW]
    // coefficients whose spectrum dbuf[B_FFTH] holds (the coefficient
    // transform is skipped when the next sum uses the same ones)
    std::vector<double> fft_key;
    const void* fft_key_buf = nullptr;
    // device copies of orbit-plan tables by plan id (a 2^k rule has one plan per level)
    std::map<uint64_t, std::pair<void*, size_t>> orb_tabs;
    // dynamic shared-memory opt-ins made on this context's device, per kernel
    // (cudaFuncSetAttribute is per device; a context is one device and one thread)
    std::map<const void*, int> smem_optin;
    // bytes moved between host and device by this context (cudaMemcpy*), and
    // kernel-parameter bytes of the lattice-sum launches (lq_ctx_transfer_bytes)
    int64_t h2d_bytes = 0, d2h_bytes = 0, param_bytes = 0;
};

namespace {

int set_dev(lq_ctx* c) {
    if (!c) return fail(LQ_ERR_VALUE, "null lq_ctx");
    CK(cudaSetDevice(c->device));
    return LQ_OK;
}

int dev_buf(lq_ctx* c, int which, size_t bytes, void** out) {
    if (bytes == 0) bytes = 8;
    if (c->dcap[which] < bytes) {
        if (c->dbuf[which]) {
            CK(cudaStreamSynchronize(c->stream));
            CK(cudaFree(c->dbuf[which]));
            c->dbuf[which] = nullptr;
            c->dcap[which] = 0;
        }
        size_t cap = bytes + bytes / 4;
        cudaError_t e = cudaMalloc(&c->dbuf[which], cap);
        if (e != cudaSuccess) return fail(LQ_ERR_NOMEM, "cudaMalloc(%zu): %s", cap, cudaGetErrorString(e));
        c->dcap[which] = cap;
    }
    *out = c->dbuf[which];
    return LQ_OK;
}

int pin_buf(lq_ctx* c, size_t bytes, void** out) {
    if (c->hcap < bytes) {
        if (c->hpin) {
            CK(cudaStreamSynchronize(c->stream));
            CK(cudaFreeHost(c->hpin));
            c->hpin = nullptr;
        }
        size_t cap = bytes < 4096 ? 4096 : bytes + bytes / 4;
        CK(cudaMallocHost(&c->hpin, cap));
        c->hcap = cap;
    }
    *out = c->hpin;
    return LQ_OK;
}

// H2D through the pinned staging buffer (async on the ctx stream; the
// staging buffer is reused only after the stream drains it).
// Consecutive uploads take consecutive slices of the staging buffer, so a
// call's several parameter uploads cost one stream drain, not one each; the
// slices are recycled only once the stream has drained them.
int upload(lq_ctx* c, int which, const void* src, size_t bytes, void** dst) {
    int rc = dev_buf(c, which, bytes, dst);
    if (rc) return rc;
    if (bytes == 0) return LQ_OK;
    const size_t need = (bytes + 255) & ~(size_t)255;
    if (c->hoff + need > c->hcap) {
        CK(cudaStreamSynchronize(c->stream));
        c->hoff = 0;
        void* h;
        if ((rc = pin_buf(c, std::max<size_t>(need, 1 << 20), &h))) return rc;
    }
    char* h = (char*)c->hpin + c->hoff;
    c->hoff += need;
    memcpy(h, src, bytes);
    CK(cudaMemcpyAsync(*dst, h, bytes, cudaMemcpyHostToDevice, c->stream));
    c->h2d_bytes += (int64_t)bytes;
    return LQ_OK;
}

// Opt kernel `fn` into `bytes` of dynamic shared memory on the context's device.
int smem_optin(lq_ctx* c, const void* fn, size_t bytes) {
    auto it = c->smem_optin.find(fn);
    if (it != c->smem_optin.end() && it->second >= (int)bytes) return LQ_OK;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    c->smem_optin[fn] = (int)bytes;
    return LQ_OK;
}

int grid_for(lq_ctx* c, const void* kernel, int64_t work, int fallback_per_sm = 1) {
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, lq::kThreads, 0) != cudaSuccess) {
        cudaGetLastError();
        per_sm = fallback_per_sm;   // (a grid larger than resident only queues)
    }
    if (per_sm < 1) per_sm = 1;
    int64_t g = (int64_t)c->sm_count * per_sm;
    if (work < g) g = work;
    return (int)(g < 1 ? 1 : g);
}

void t_begin(lq_ctx* c) {
    if (c->timing) cudaEventRecord(c->ev0, c->stream);
}
void t_end(lq_ctx* c) {
    if (c->timing) cudaEventRecord(c->ev1, c->stream);
    c->launches++;
}

// Fixed-tree reduction of vals[count] down to one value in device memory.
int reduce_dev(lq_ctx* c, const double* vals, int64_t count, double** result) {
    const double* cur = vals;
    int which = B_RED0;
    int64_t n = count;
    if (n <= 0) {
        void* p;
        int rc = dev_buf(c, B_RED0, 8, &p);
        if (rc) return rc;
        CK(cudaMemsetAsync(p, 0, 8, c->stream));
        *result = (double*)p;
        return LQ_OK;
    }
    // a single value is its own tree (k_reduce1024 would return it unchanged)
    while (n > 1) {
        int64_t groups = (n + 1023) / 1024;
        void* p;
        int rc = dev_buf(c, which, groups * sizeof(double), &p);
        if (rc) return rc;
        lq::k_reduce1024<<<(unsigned)groups, lq::kThreads, 0, c->stream>>>(cur, n, (double*)p);
        c->launches++;
        CK(cudaGetLastError());
        cur = (const double*)p;
        n = groups;
        which = which == B_RED0 ? B_RED1 : B_RED0;
    }
    *result = const_cast<double*>(cur);
    return LQ_OK;
}

int read_scalar(lq_ctx* c, const double* dev, double* out, int k = 1) {
    void* h = nullptr;
    int rc = pin_buf(c, sizeof(double) * k, &h);
    if (rc) return rc;
    // (staged uploads still in flight read their slices before this copy
    // writes: same stream, in order)
    CK(cudaMemcpyAsync(h, dev, sizeof(double) * k, cudaMemcpyDeviceToHost, c->stream));
    c->d2h_bytes += (int64_t)(sizeof(double) * k);
    CK(cudaStreamSynchronize(c->stream));
    c->hoff = 0;
    memcpy(out, h, sizeof(double) * k);
    return LQ_OK;
}

// ------------------------------------------------------------ lattice sums

int check_lattice(uint64_t n, const uint64_t* z, int d) {
    if (n < 1) return fail(LQ_ERR_VALUE, "point count must be positive, got %llu", (unsigned long long)n);
    if (n > (1ull << 53)) return fail(LQ_ERR_OVERFLOW, "cannot enumerate points of an n=%llu rule", (unsigned long long)n);
    if (d < 1) return fail(LQ_ERR_VALUE, "dimension must be positive, got %d", d);
    if (!z) return fail(LQ_ERR_VALUE, "null generating vector");
    for (int j = 0; j < d; ++j)
        if (z[j] >= n) return fail(LQ_ERR_VALUE, "z_reduced[%d]=%llu not reduced mod n", j, (unsigned long long)z[j]);
    return LQ_OK;
}

int pick_slots(int n_slots) {
    if (n_slots > LQ_MAX_SLOTS) return -1;
    return n_slots <= 32 ? 32 : LQ_MAX_SLOTS;
}

uint64_t tile_points(const lq_integrand* f, uint64_t n);
bool uses_family_kernel(const lq_integrand* f, uint64_t n);

bool is_quad_kind(int k) { return k == LQ_FAM_QUAD_EXP || k == LQ_FAM_QUAD_SINCOS; }
bool is_lin_kind(int k) {
    return k == LQ_FAM_LIN_EXP || k == LQ_FAM_LIN_SINCOS || k == LQ_FAM_LIN_EXPABS || k == LQ_FAM_LIN_POW;
}
int lin_outer(int k) {
    return k == LQ_FAM_LIN_EXP ? lq::OUT_EXP : k == LQ_FAM_LIN_SINCOS ? lq::OUT_SINCOS
         : k == LQ_FAM_LIN_EXPABS ? lq::OUT_EXPABS : k == LQ_FAM_LIN_PROG ? lq::OUT_PROG : lq::OUT_POW;
}
int quad_outer_of(int k) { return k == LQ_FAM_QUAD_SINCOS ? lq::OUT_SINCOS : lq::OUT_EXP; }

// Dimension split of the family kernels: lattices with fewer tiles than
// ~4 waves of CTAs run each tile on a cluster of S CTAs that split the
// dimensions (k_fam<S>).  S depends on (units, d) only, so every GPU of a
// multi-GPU run uses the same reduction structure.
int fam_split(uint64_t units, int d, int kind) {
    const uint64_t tp = (uint64_t)lq::kThreads * lq::fam_pts(kind);
    const uint64_t tiles = (units + tp - 1) / tp;
    const uint64_t want = 148ull * 2 * 4;
    int S = 1;
    while (S < 8 && tiles * S < want && d / (2 * S) >= 16) S *= 2;
    return S;
}

template <int KIND, int OUTER, bool PAIR, class Args, int S>
int launch_fam_s(lq_ctx* c, const Args& args, int64_t ntiles, double* tiles_dev) {
    auto kern = lq::k_fam<KIND, OUTER, Args, S, PAIR>;
    const int na = KIND == lq::FAM_QUADP ? 2 : 1;
    const size_t smem = S > 1 ? sizeof(double) * na * lq::fam_pts(KIND) * lq::kThreads : 0;
    if (S > 1) {
        int rc = smem_optin(c, (const void*)kern, smem);
        if (rc) return rc;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)ntiles, S, 1);
    cfg.blockDim = dim3(lq::kThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = S;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = S > 1 ? 1 : 0;
    t_begin(c);
    CK(cudaLaunchKernelEx(&cfg, kern, args, 0u, tiles_dev));
    t_end(c);
    CK(cudaGetLastError());
    return LQ_OK;
}

template <int KIND, int OUTER, bool PAIR, class Args>
int launch_fam(lq_ctx* c, const Args& args, int64_t ntiles, double* tiles_dev, uint64_t units) {
    switch (fam_split(units, args.d, KIND)) {
        case 1: return launch_fam_s<KIND, OUTER, PAIR, Args, 1>(c, args, ntiles, tiles_dev);
        case 2: return launch_fam_s<KIND, OUTER, PAIR, Args, 2>(c, args, ntiles, tiles_dev);
        case 4: return launch_fam_s<KIND, OUTER, PAIR, Args, 4>(c, args, ntiles, tiles_dev);
        default: return launch_fam_s<KIND, OUTER, PAIR, Args, 8>(c, args, ntiles, tiles_dev);
    }
}

// Full-range sums pair each point with its mirror n - i (x -> 1 - x) when every
// z_j is a unit mod n -- then only i = 0 and i = n/2 are self-mirrored -- and
// run over the pair indices [0, n/2] (LQ_PAIR=0 disables).
bool pair_ok(const lq_integrand* f, uint64_t n, const uint64_t* z) {
    const char* e = std::getenv("LQ_PAIR");
    if (e && !std::strcmp(e, "0")) return false;
    if (!z || f->kind == LQ_FAM_PROGRAM || f->kind == LQ_FAM_LIN_PROG || f->kind == LQ_FAM_PROD_QUAD || n < 3 ||
        n > (1ull << 31))
        return false;
    for (int j = 0; j < f->d; ++j) {
        uint64_t a = z[j], b = n;
        while (b) { const uint64_t t = a % b; a = b; b = t; }
        if (a != 1) return false;
    }
    return true;
}

int fam_kind(const lq_integrand* f, bool pair) {
    if (is_quad_kind(f->kind)) return pair ? lq::FAM_QUADP : lq::FAM_QUAD;
    if (f->kind == LQ_FAM_PROD_QUAD) return lq::FAM_PROD;
    return lq::FAM_LIN;
}

uint64_t tile_points(const lq_integrand* f, uint64_t n, bool pair) {
    if (!uses_family_kernel(f, n)) return (uint64_t)lq::kTile;
    return (uint64_t)lq::kThreads * lq::fam_pts(fam_kind(f, pair));
}
uint64_t tile_points(const lq_integrand* f, uint64_t n) { return tile_points(f, n, false); }

// scalar parameters of the family kernels
struct FamHead {
    double alpha = 0, scale = 1, K = 0, A = 0, B = 0, C0 = 0, kappa = 0, M = 0, alphaB = 0, bsum = 0, half = 0, pw = 0;
    lq::PairFast pf{};
};

bool pair_fast_consts(const lq_integrand* f, double bsum, lq::PairFast& q);
// PairFast for kernels whose accumulator is the linear form / scale
void pair_fast_scaled(const lq_integrand* f, double bsum, double scale, lq::PairFast& q) {
    if (pair_fast_consts(f, bsum, q)) q.ym *= scale;   // scale = 2^sigma: exact
}

template <class A>
void fill_head(A& a, int d, uint64_t n, uint64_t base, uint64_t end, const FamHead& h) {
    a.d = d; a.n = (uint32_t)n; a.base = base; a.end = end;
    a.alpha = h.alpha; a.scale = h.scale; a.K = h.K; a.A = h.A; a.B = h.B; a.C0 = h.C0; a.kappa = h.kappa;
    a.M = h.M; a.alphaB = h.alphaB; a.bsum = h.bsum; a.half = h.half; a.pw = h.pw; a.pf = h.pf;
}

// Per-dimension tables in kernel parameter space, sized to d: the launch copies
// the whole parameter struct, so small-d integrands use small instantiations
// (measured: cfg1, d = 8, 25.6 -> 12.7 us per launch with a 32 KB vs 4 KB struct).
template <int KIND, int OUTER, bool PAIR, class Dim, int N>
int fam_param_launch(lq_ctx* c, const std::vector<Dim>& tab, int d, uint64_t n, uint64_t base, uint64_t end,
                     int64_t ntiles, uint64_t units, const FamHead& h, double* tiles_dev) {
    using Args = lq::FamArgs<Dim, N>;
    static thread_local Args args;
    fill_head(args, d, n, base, end, h);
    std::memcpy(args.dims, tab.data(), sizeof(Dim) * d);
    if (N <= 32) return launch_fam_s<KIND, OUTER, PAIR, Args, 1>(c, args, ntiles, tiles_dev);   // d < 64: no split
    return launch_fam<KIND, OUTER, PAIR>(c, args, ntiles, tiles_dev, units);
}

template <int KIND, int OUTER, bool PAIR, class Dim>
int fam_dispatch(lq_ctx* c, const std::vector<Dim>& tab, int d, uint64_t n, uint64_t base, uint64_t end,
                 int64_t ntiles, uint64_t units, const FamHead& h, double* tiles_dev) {
#define LQ_FPL(N) fam_param_launch<KIND, OUTER, PAIR, Dim, N>(c, tab, d, n, base, end, ntiles, units, h, tiles_dev)
    if (d <= 32) return LQ_FPL(32);
    if (d <= 128) return LQ_FPL(128);
    if (d <= lq::kParamDims) return LQ_FPL(lq::kParamDims);
#undef LQ_FPL
    void* dt;
    int rc;
    if ((rc = upload(c, B_TAB, tab.data(), tab.size() * sizeof(Dim), &dt))) return rc;
    lq::FamArgsG<Dim> args;
    fill_head(args, d, n, base, end, h);
    args.dims = (const Dim*)dt;
    return launch_fam<KIND, OUTER, PAIR>(c, args, ntiles, tiles_dev, units);
}

// LIN_PROG has no per-index family kernel: its sub-ranges and non-Korobov
// rules run the whole expression's bytecode (f->prog) like PROGRAM.
bool uses_family_kernel(const lq_integrand* f, uint64_t n) {
    return n <= (1ull << 31) && f->kind != LQ_FAM_PROGRAM && f->kind != LQ_FAM_LIN_PROG;
}

// Product family (k_prod).  The coordinate comes out of the denormal residue
// as x 2^-g (g >= 51 - log2 n keeps 2^(1074-g)/n finite), so every scaled
// factor carries 2^-2g; the running product is renormalised every R factors,
// R the largest power of two <= 16 that keeps R worst-case scaled factors
// inside 2^(+-1000).
struct ProdScale {
    int g = 0, R = 16;
    double m = 0.0;
    int64_t off = 0;
    std::vector<int> dims;            // coordinates carrying a factor
    std::vector<double> w, c;         // scaled w_j 2^-g, c_j 2^-2g
};

int prod_scale(const lq_integrand* f, uint64_t n, ProdScale& ps) {
    if (!f->beta || !f->gamma) return fail(LQ_ERR_VALUE, "product family needs beta (w) and gamma (c)");
    ps.g = std::max(0, 51 - std::ilogb((double)n));
    ps.m = std::ldexp(1.0 / (double)n, 1074 - ps.g);
    if (!std::isfinite(ps.m)) return fail(LQ_ERR_UNSUPPORTED, "product family: scale overflow for n=%llu", (unsigned long long)n);
    double worst = 0.0;
    for (int j = 0; j < f->d; ++j) {
        const double w = f->beta[j], cj = f->gamma[j];
        if (std::isnan(cj)) continue;
        const double dist = w < 0.0 ? -w : (w > 1.0 ? w - 1.0 : 0.0);
        const double fmin = cj + dist * dist, fmax = cj + std::fmax(w * w, (1.0 - w) * (1.0 - w));
        if (!(fmin > 0.0) || !std::isfinite(fmax))
            return fail(LQ_ERR_UNSUPPORTED, "product factor %d spans [%g, %g]", j + 1, fmin, fmax);
        worst = std::fmax(worst, std::fmax(std::fabs(std::log2(fmin) - 2 * ps.g), std::fabs(std::log2(fmax) - 2 * ps.g)));
        const double cs = std::ldexp(cj, -2 * ps.g);
        if (cj != 0.0 && !std::isnormal(cs))
            return fail(LQ_ERR_UNSUPPORTED, "product factor %d out of the scaled range", j + 1);
        ps.dims.push_back(j);
        ps.w.push_back(std::ldexp(w, -ps.g));
        ps.c.push_back(cs);
    }
    ps.R = 16;
    while (ps.R > 1 && ps.R * (worst + 1.0) > 1000.0) ps.R /= 2;
    if ((worst + 1.0) > 1000.0) return fail(LQ_ERR_UNSUPPORTED, "product factors span more than 2^1000");
    ps.off = 2ll * ps.g * (int64_t)ps.dims.size();
    if (ps.off > (1ll << 30)) return fail(LQ_ERR_UNSUPPORTED, "product exponent offset too large");
    return LQ_OK;
}

int launch_prod(lq_ctx* c, const lq_integrand* f, uint64_t n, const uint64_t* z, uint64_t base, uint64_t end,
                int64_t ntiles, double* tiles_dev) {
    ProdScale ps;
    int rc0 = prod_scale(f, n, ps);
    if (rc0) return rc0;
    std::vector<lq::ProdDim> tab(ps.dims.size());
    for (size_t k = 0; k < ps.dims.size(); ++k) {
        const int j = ps.dims[k];
        lq::ProdDim& r = tab[k];
        r.w = ps.w[k];
        r.c = ps.c[k];
        r.z = (uint32_t)z[j];
        r.zs = (uint32_t)(((uint64_t)z[j] << 32) / n);
        r.z2 = (uint32_t)((2 * z[j]) % n);
        r.z2m = r.z2 - (uint32_t)n;
    }
    const double m = ps.m;
    const int64_t off = ps.off;
    const int R = ps.R;
    const int nf = (int)tab.size();
    auto head = [&](auto& a) {
        a.nf = nf; a.n = (uint32_t)n; a.base = base; a.end = end; a.K = f->K; a.pw = f->power; a.m = m;
        a.off = (int32_t)off;
        a.rmask = R - 1;
    };
    if (nf <= lq::kProdParamDims) {
        static thread_local lq::ProdArgs<lq::kProdParamDims> args;
        head(args);
        std::memcpy(args.dims, tab.data(), sizeof(lq::ProdDim) * nf);
        t_begin(c);
        lq::k_prod<<<(unsigned)ntiles, lq::kThreads, 0, c->stream>>>(args, 0u, tiles_dev);
        t_end(c);
    } else {
        void* dt;
        int rc;
        if ((rc = upload(c, B_TAB, tab.data(), tab.size() * sizeof(lq::ProdDim), &dt))) return rc;
        lq::ProdArgsG args;
        head(args);
        args.dims = (const lq::ProdDim*)dt;
        t_begin(c);
        lq::k_prod<<<(unsigned)ntiles, lq::kThreads, 0, c->stream>>>(args, 0u, tiles_dev);
        t_end(c);
    }
    CK(cudaGetLastError());
    return LQ_OK;
}

// Launch the tile kernel of integrand f over index units [base, end) writing
// ntiles tile partials to tiles_dev.  pair: units are mirror-pair indices
// [0, n/2] of a full-range sum (pair_ok), else points.
int launch_tiles(lq_ctx* c, const lq_integrand* f, uint64_t n, const uint64_t* z, uint64_t base, uint64_t end,
                 int64_t ntiles, double* tiles_dev, bool pair = false) {
    const int d = f->d;
    const bool fast = uses_family_kernel(f, n);
    const uint64_t units = pair ? n / 2 + 1 : n;
    int rc;
    if (fast && is_lin_kind(f->kind)) {
        if (!f->beta) return fail(LQ_ERR_VALUE, "family needs beta");
        double maxabs = 0.0, bsum = 0.0;
        for (int j = 0; j < d; ++j) {
            maxabs = fmax(maxabs, fabs(f->beta[j]));
            bsum += f->beta[j];
        }
        if (!std::isfinite(maxabs)) return fail(LQ_ERR_VALUE, "non-finite coefficient");
        int sigma = 0;
        if (maxabs > 0.0) {
            int e = std::ilogb(maxabs / (double)n);
            sigma = 1074 + e + 1 - 1020;
            if (sigma < 0) sigma = 0;
        }
        std::vector<lq::LinDim> tab(d);
        for (int j = 0; j < d; ++j) {
            tab[j].c = std::ldexp(f->beta[j] / (double)n, 1074 - sigma);
            tab[j].z = (uint32_t)z[j];
            tab[j].zs = (uint32_t)(((uint64_t)z[j] << 32) / n);
            tab[j].z2 = (uint32_t)((2 * z[j]) % n);
            tab[j].z2m = tab[j].z2 - (uint32_t)n;
        }
        FamHead h;
        h.alpha = f->alpha; h.scale = std::ldexp(1.0, sigma); h.K = f->K; h.A = f->A; h.B = f->B; h.C0 = f->C0;
        h.kappa = f->kappa; h.bsum = bsum; h.alphaB = f->alpha + bsum; h.pw = f->power;
        if (pair) pair_fast_scaled(f, bsum, h.scale, h.pf);
#define LQ_LIN(OUT) (pair ? fam_dispatch<lq::FAM_LIN, OUT, true>(c, tab, d, n, base, end, ntiles, units, h, tiles_dev) \
                          : fam_dispatch<lq::FAM_LIN, OUT, false>(c, tab, d, n, base, end, ntiles, units, h, tiles_dev))
        switch (lin_outer(f->kind)) {
            case lq::OUT_EXP: return LQ_LIN(lq::OUT_EXP);
            case lq::OUT_SINCOS: return LQ_LIN(lq::OUT_SINCOS);
            case lq::OUT_EXPABS: return LQ_LIN(lq::OUT_EXPABS);
            default: return LQ_LIN(lq::OUT_POW);
        }
#undef LQ_LIN
    }
    if (fast && is_quad_kind(f->kind)) {
        if (!f->beta || !f->gamma) return fail(LQ_ERR_VALUE, "quad family needs beta and gamma");
        const double inv_n = 1.0 / (double)n;
        int sigma = 1074 + std::ilogb(inv_n) - 1000;
        if (sigma < 0) sigma = 0;
        FamHead h;
        h.alpha = f->alpha; h.K = f->K; h.A = f->A; h.B = f->B; h.C0 = f->C0;
        h.M = std::ldexp(inv_n, 1074 - sigma); h.half = std::ldexp(0.5, -sigma);
        std::vector<lq::QuadDim> tab(d);
        double C0 = 0.0;
        for (int j = 0; j < d; ++j) {
            // paired: centred form b' u + q u^2 with b' = beta + gamma (u = x - 1/2)
            tab[j].b = std::ldexp(pair ? f->beta[j] + f->gamma[j] : f->beta[j], sigma);
            tab[j].q = std::ldexp(f->gamma[j], 2 * sigma);
            tab[j].z = (uint32_t)z[j];
            tab[j].zs = (uint32_t)(((uint64_t)z[j] << 32) / n);
            tab[j].z2 = (uint32_t)((2 * z[j]) % n);
            tab[j].z2m = tab[j].z2 - (uint32_t)n;
            C0 += 0.5 * f->beta[j] + 0.25 * f->gamma[j];
            if (!std::isfinite(tab[j].b) || !std::isfinite(tab[j].q))
                return fail(LQ_ERR_VALUE, "quadratic coefficient out of range");
        }
        h.alphaB = f->alpha + C0;
        if (quad_outer_of(f->kind) == lq::OUT_SINCOS) {
            if (pair) return fam_dispatch<lq::FAM_QUADP, lq::OUT_SINCOS, true>(c, tab, d, n, base, end, ntiles, units, h, tiles_dev);
            return fam_dispatch<lq::FAM_QUAD, lq::OUT_SINCOS, false>(c, tab, d, n, base, end, ntiles, units, h, tiles_dev);
        }
        if (pair) return fam_dispatch<lq::FAM_QUADP, lq::OUT_EXP, true>(c, tab, d, n, base, end, ntiles, units, h, tiles_dev);
        return fam_dispatch<lq::FAM_QUAD, lq::OUT_EXP, false>(c, tab, d, n, base, end, ntiles, units, h, tiles_dev);
    }
    if (fast && f->kind == LQ_FAM_PROD_QUAD) return launch_prod(c, f, n, z, base, end, ntiles, tiles_dev);
    // generic bytecode (any family falls back here for n > 2^31)
    const lq_program* pg = &f->prog;
    if (!pg->insn || pg->n_insn < 1)
        return fail(LQ_ERR_UNSUPPORTED, "integrand needs a bytecode program for n=%llu", (unsigned long long)n);
    const int ns = pick_slots(pg->n_slots);
    if (ns < 0) return fail(LQ_ERR_UNSUPPORTED, "program needs %d slots (max %d)", pg->n_slots, LQ_MAX_SLOTS);
    if (pg->n_vars > d) return fail(LQ_ERR_VALUE, "program uses %d variables, rule has d=%d", pg->n_vars, d);
    void* dp;
    if ((rc = upload(c, B_PROG, pg->insn, sizeof(lq_insn) * pg->n_insn, &dp))) return rc;
    const bool wide = n > (1ull << 31);
    void* dz;
    if (wide) {
        if ((rc = upload(c, B_TAB, z, sizeof(uint64_t) * d, &dz))) return rc;
    } else {
        std::vector<uint32_t> zz(2 * (size_t)d);
        for (int j = 0; j < d; ++j) {
            zz[2 * j] = (uint32_t)z[j];
            zz[2 * j + 1] = (uint32_t)(((uint64_t)z[j] << 32) / n);
        }
        if ((rc = upload(c, B_TAB, zz.data(), zz.size() * 4, &dz))) return rc;
    }
    const double n_d = (double)n, inv_n = 1.0 / n_d;
    if (cudaKernel_t jk = lq_jit_lattice_kernel(pg->jit)) {
        const void* ztab = dz;
        int wide_i = wide ? 1 : 0;
        int64_t nt = ntiles;
        void* args[] = {(void*)&ztab, (void*)&n, (void*)&n_d, (void*)&inv_n, (void*)&base, (void*)&end, (void*)&wide_i, (void*)&tiles_dev, (void*)&nt};
        // a resident grid striding over the tiles: each thread's coordinate
        // residues are set up once and carried from tile to tile
        const int grid = grid_for(c, (const void*)jk, ntiles, 2048 / lq::kThreads);
        t_begin(c);
        CK(cudaLaunchKernel((const void*)jk, dim3((unsigned)grid), dim3(lq::kThreads), args, 0, c->stream));
        t_end(c);
        return LQ_OK;
    }
    const void* kern = wide ? (ns == 32 ? (const void*)lq::k_prog_lattice<32, true> : (const void*)lq::k_prog_lattice<LQ_MAX_SLOTS, true>)
                            : (ns == 32 ? (const void*)lq::k_prog_lattice<32, false> : (const void*)lq::k_prog_lattice<LQ_MAX_SLOTS, false>);
    int grid = grid_for(c, kern, ntiles);
    t_begin(c);
#define LQ_PL(NS, W) lq::k_prog_lattice<NS, W><<<grid, lq::kThreads, 0, c->stream>>>((const lq_insn*)dp, pg->n_insn, pg->result, n, n_d, inv_n, inv_n, dz, base, end, ntiles, tiles_dev)
    if (wide) { if (ns == 32) LQ_PL(32, true); else LQ_PL(LQ_MAX_SLOTS, true); }
    else { if (ns == 32) LQ_PL(32, false); else LQ_PL(LQ_MAX_SLOTS, false); }
#undef LQ_PL
    t_end(c);
    CK(cudaGetLastError());
    return LQ_OK;
}

int check_integrand(const lq_integrand* f) {
    if (!f) return fail(LQ_ERR_VALUE, "null integrand");
    if (f->kind < LQ_FAM_PROGRAM || f->kind > LQ_FAM_LIN_PROG) return fail(LQ_ERR_VALUE, "bad family kind %d", f->kind);
    if (f->kind == LQ_FAM_LIN_PROG &&
        (!f->beta || !f->outer.insn || f->outer.n_insn < 1 || f->outer.n_vars > 1 || f->outer.n_slots > 32))
        return fail(LQ_ERR_VALUE, "LIN_PROG needs beta and a one-variable outer program of <= 32 slots");
    if ((f->kind == LQ_FAM_LIN_POW || f->kind == LQ_FAM_PROD_QUAD) &&
        (f->power != std::floor(f->power) || std::fabs(f->power) > 1e6))
        return fail(LQ_ERR_VALUE, "LIN_POW needs an integer power, got %g", f->power);
    return LQ_OK;
}

#include "lq_plans.cuh"   // orbit planners (prime n, 2^k, composite n)

// LQ_ORBIT=0 disables the orbit kernel; otherwise it runs whenever the rule
// allows (measured kernel ms, orbit vs mirror-paired index kernel: cfg1
// 0.0119 / 0.0125, cfg2 0.0231 / 0.0244, cfg3 0.053 / 0.127, cfg5 67.9 / 134.8).
int orbit_mode() {
    const char* e = std::getenv("LQ_ORBIT");
    if (!e || !*e) return 1;
    if (!std::strcmp(e, "0")) return 0;
    if (!std::strcmp(e, "always")) return 2;
    return 1;
}

// The FFT form (k_orbit_fft) for the linear families when d is large enough
// for O(log N) per point to beat O(d) and the lattice is large enough to fill
// the GPU with 4096-point tiles: LQ_FFT=0 disables, =always forces.
// (kernel ms, FFT vs direct orbit: cfg2, n = 10^4, d = 100: 0.023 vs 0.022;
// cfg3, n = 10^6, d = 300: 0.018 vs 0.054.)
// Smallest d for the FFT form (tools/fft_crossover.py: the FFT form against the
// direct orbit kernel, both with §4.1e's one-reduction pair outer): exp /
// exp-abs / sincos from d = 49 on n >= 2^22 (n = 2^31 - 1: 0.99x at d = 48,
// 1.21x at 56) and from d = 112 below (n = 1e6 + 3: 0.95x at 96, 1.40x at
// 128); power (two outer evaluations in both forms, integer powers by
// squaring) likewise (1.00x at d = 48, 1.29x at 96); the Gaussian form
// transforms one chain per CTA and wins from d = 64.
constexpr uint64_t kFftMinN = 1ull << 18;
int fft_min_d(const lq_integrand* f, uint64_t n) {
    if (is_quad_kind(f->kind)) return 64;
    if (f->kind == LQ_FAM_LIN_PROG) return 16;   // the alternative is the per-index bytecode kernel
    return n >= (1ull << 22) ? 49 : 112;
}
// Accuracy guard: the FFT's norm-wise error on a linear form is about
// eps log2(N) ||c||_2 ||P||_2 <= 1.2e-16 * 12 * ||beta||_2 * sqrt(N)
// (c = beta / n, residues < n); the FFT form is used only while that bound
// stays below 1e-11 absolute on the linear forms (||beta||_2 <= ~100), where
// the direct kernels' own rounding is of the same order.
bool fft_accurate(const lq_integrand* f) {
    double s2 = 0.0;
    for (int j = 0; j < f->d; ++j) {
        if (is_quad_kind(f->kind)) {   // centred form: b' = beta + gamma, q = gamma (|u| <= 1/2)
            const double bp = f->beta[j] + f->gamma[j];
            s2 += bp * bp + f->gamma[j] * f->gamma[j];
        } else {
            s2 += f->beta[j] * f->beta[j];
        }
    }
    const double bound = 1.2e-16 * 12.0 * std::sqrt(s2) * std::sqrt((double)lq::kFftN);
    return std::isfinite(bound) && bound <= 1e-11;
}

bool fft_wanted(const lq_integrand* f, uint64_t n) {
    const char* e = std::getenv("LQ_FFT");
    if (e && !std::strcmp(e, "0")) return false;
    if (!(is_lin_kind(f->kind) || is_quad_kind(f->kind) || f->kind == LQ_FAM_LIN_PROG) || f->d > lq::kFftN / 2 ||
        !f->beta)
        return false;
    if (is_quad_kind(f->kind) && !f->gamma) return false;
    if (!fft_accurate(f)) return false;
    if (e && !std::strcmp(e, "always")) return f->d >= 2;
    return f->d >= fft_min_d(f, n) && n >= kFftMinN;
}

std::shared_ptr<const OrbPlan> orbit_for(const lq_integrand* f, uint64_t n, const uint64_t* z, bool* fft = nullptr) {
    if (fft) *fft = false;
    const int mode = orbit_mode();
    if (mode == 0 || !z || f->kind == LQ_FAM_PROGRAM || f->d < 2) return nullptr;
    if (n > (1ull << 31) || n < 5) return nullptr;
    const bool prod = f->kind == LQ_FAM_PROD_QUAD;
    const bool quad = is_quad_kind(f->kind);
    const int m = prod ? lq::kOrbProdM : lq::orb_len(quad ? lq::FAM_QUAD : lq::FAM_LIN);
    const int cap = prod ? lq::kOrbProdDims : quad ? lq::kOrbQuadDims : lq::kOrbLinDims;
    if (!f->beta || ((quad || prod) && !f->gamma)) return nullptr;
    if (prod)
        for (int j = 0; j < f->d; ++j)
            if (std::isnan(f->gamma[j])) return nullptr;   // every coordinate must carry a factor
    if (z[0] != 1 % n) return nullptr;
    const uint64_t a = z[1];
    for (int j = 2; j < f->d; ++j)
        if (z[j] != z[j - 1] * a % n) return nullptr;   // z_j = a^(j-1) mod n
    if (fft && fft_wanted(f, n)) {   // the FFT form has its own dimension limit (d <= N/2)
        auto p = orbit_plan((uint32_t)n, (uint32_t)a, lq::kFftN - f->d + 1, true, true);
        if (p) {
            *fft = true;
            return p;
        }
    }
    if (f->kind == LQ_FAM_LIN_PROG) return nullptr;     // no direct orbit kernel for a program outer
    if ((f->d + m - 1) / m * m > cap) return nullptr;   // direct form: tables in parameter space
    return orbit_plan((uint32_t)n, (uint32_t)a, m, !prod);
}

// Device copies of the start tables, cached per context and plan.
int orbit_tables(lq_ctx* c, const OrbPlan& p, const uint32_t** G, const uint32_t** Alo, const uint32_t** Ahi,
                 const uint2** apow = nullptr, const uint32_t** starts = nullptr) {
    const size_t nG = p.G.size(), nlo = p.Alo.size(), nhi = p.Ahi.size(), np = p.apow.size();
    const size_t pad = (nG + nlo + nhi) & 1;   // keep apow 8-byte aligned
    const size_t ns = p.starts.size();
    const size_t bytes = 4 * (nG + nlo + nhi + pad + np + ns);
    auto it = c->orb_tabs.find(p.id);
    if (it == c->orb_tabs.end()) {
        // bounded cache (a composite-n layout holds one plan per divisor class,
        // 2^31 - 2: ~190): drop everything past 1024 plans or 512 MB
        size_t held = 0;
        for (auto& kv : c->orb_tabs) held += kv.second.second;
        if (c->orb_tabs.size() >= 1024 || held + bytes > (512u << 20)) {
            CK(cudaStreamSynchronize(c->stream));
            for (auto& kv : c->orb_tabs) cudaFree(kv.second.first);
            c->orb_tabs.clear();
        }
        std::vector<uint32_t> all;
        all.reserve(nG + nlo + nhi + pad + np);
        all.insert(all.end(), p.G.begin(), p.G.end());
        all.insert(all.end(), p.Alo.begin(), p.Alo.end());
        all.insert(all.end(), p.Ahi.begin(), p.Ahi.end());
        if (pad) all.push_back(0);
        all.insert(all.end(), p.apow.begin(), p.apow.end());
        all.insert(all.end(), p.starts.begin(), p.starts.end());
        void* d = nullptr;
        CK(cudaMalloc(&d, bytes));
        CK(cudaMemcpy(d, all.data(), bytes, cudaMemcpyHostToDevice));   // once per (context, plan)
        c->h2d_bytes += (int64_t)bytes;
        it = c->orb_tabs.emplace(p.id, std::make_pair(d, bytes)).first;
    }
    const uint32_t* base = (const uint32_t*)it->second.first;
    *G = base;
    *Alo = base + nG;
    *Ahi = base + nG + nlo;
    if (apow) *apow = (const uint2*)(base + nG + nlo + nhi + pad);
    if (starts) *starts = base + nG + nlo + nhi + pad + np;
    return LQ_OK;
}

// Kernel-parameter structs sized to the padded dimension (the launch copies
// the whole struct: 32 KB costs ~13 us per launch).
template <int N>
int orbit_quad(lq_ctx* c, const lq::OrbHead& head, const std::vector<double2>& bq, int outer, uint64_t unit0,
               int64_t ntiles, double* tiles_dev) {
    using Args = lq::OrbQuadArgs<N>;
    static thread_local Args args;
    args.h = head;
    std::memcpy(args.bq, bq.data(), sizeof(double2) * bq.size());
    const dim3 g((unsigned)ntiles), b(lq::kThreads);
    t_begin(c);
    if (outer == lq::OUT_SINCOS)
        lq::k_orbit<lq::FAM_QUAD, lq::OUT_SINCOS, Args><<<g, b, 0, c->stream>>>(args, unit0, 0u, tiles_dev);
    else
        lq::k_orbit<lq::FAM_QUAD, lq::OUT_EXP, Args><<<g, b, 0, c->stream>>>(args, unit0, 0u, tiles_dev);
    t_end(c);
    CK(cudaGetLastError());
    return LQ_OK;
}

template <int N>
int orbit_lin(lq_ctx* c, const lq::OrbHead& head, const std::vector<double>& cv, int outer, uint64_t unit0,
              int64_t ntiles, double* tiles_dev) {
    using Args = lq::OrbLinArgs<N>;
    static thread_local Args args;
    args.h = head;
    std::memcpy(args.c, cv.data(), sizeof(double) * cv.size());
    const dim3 g((unsigned)ntiles), b(lq::kThreads);
    t_begin(c);
    if (outer == lq::OUT_EXP)
        lq::k_orbit<lq::FAM_LIN, lq::OUT_EXP, Args><<<g, b, 0, c->stream>>>(args, unit0, 0u, tiles_dev);
    else if (outer == lq::OUT_SINCOS)
        lq::k_orbit<lq::FAM_LIN, lq::OUT_SINCOS, Args><<<g, b, 0, c->stream>>>(args, unit0, 0u, tiles_dev);
    else if (outer == lq::OUT_EXPABS)
        lq::k_orbit<lq::FAM_LIN, lq::OUT_EXPABS, Args><<<g, b, 0, c->stream>>>(args, unit0, 0u, tiles_dev);
    else
        lq::k_orbit<lq::FAM_LIN, lq::OUT_POW, Args><<<g, b, 0, c->stream>>>(args, unit0, 0u, tiles_dev);
    t_end(c);
    CK(cudaGetLastError());
    return LQ_OK;
}

template <int N>
int orbit_prod(lq_ctx* c, const lq::OrbHead& head, const std::vector<double2>& wc, int nf, int off, int rmask,
               uint64_t unit0, int64_t ntiles, double* tiles_dev) {
    using Args = lq::OrbProdArgs<N>;
    static thread_local Args args;
    args.h = head;
    args.nf = nf;
    args.off = off;
    args.rmask = rmask;
    std::memcpy(args.wc, wc.data(), sizeof(double2) * wc.size());
    t_begin(c);
    lq::k_orbit_prod<Args><<<(unsigned)ntiles, lq::kThreads, 0, c->stream>>>(args, unit0, 0u, tiles_dev);
    t_end(c);
    CK(cudaGetLastError());
    return LQ_OK;
}

int64_t kFftTilesPerCta = [] {
    const char* e = std::getenv("LQ_FFT_PER_CTA");
    return e ? std::max<int64_t>(1, std::atoll(e)) : 8;
}();

// e^x as (c, k), c 2^k = e^x, c in [0.7, 1.5) (long double reduction on the host)
void split_exp(long double x, double& cm, int32_t& k) {
    const long double ln2 = 0.693147180559945309417232121458176568L;
    const long double kk = nearbyintl(x / ln2);
    cm = (double)expl(x - kk * ln2);
    k = (int32_t)kk;
}

// Constants of the one-reduction point/mirror pair (lq::PairFast); false when
// the family has no such form or some value could leave the normal range.
// |s1| <= |alpha| + sum |beta|, |s2| <= |alphaB| + sum |beta| (x_j in [0, 1)).
bool pair_fast_consts(const lq_integrand* f, double bsum, lq::PairFast& q) {
    q = lq::PairFast{};   // on = 0
    if (std::getenv("LQ_PAIRFAST") && std::string(std::getenv("LQ_PAIRFAST")) == "0") return false;
    const int outer = lin_outer(f->kind);
    long double babs = 0.0L;
    for (int j = 0; j < f->d; ++j) babs += fabsl((long double)f->beta[j]);
    const long double alpha = f->alpha, alphaB = (long double)f->alpha + (long double)bsum;
    const long double smax = std::max(fabsl(alpha), fabsl(alphaB)) + babs;
    const long double D = alpha + alphaB;
    if (outer == lq::OUT_SINCOS) {
        if (!std::isfinite((double)smax)) return false;
        const long double sD = sinl(D), cD = cosl(D), A = f->A, B = f->B;
        q.ym = 1.0; q.ya = f->alpha; q.post = 1.0;
        q.c0 = (double)(A + B * sD - A * cD);
        q.c1 = (double)(B + A * sD + B * cD);
        q.c2 = (double)(2.0L * (long double)f->C0);
        q.on = 1;
        return true;
    }
    if (outer == lq::OUT_EXP) {
        if (!(smax <= 700.0L)) return false;
        q.ym = 1.0; q.ya = f->alpha; q.post = f->K;
        split_exp(D, q.c0, q.k0);
        q.on = 1;
        return true;
    }
    if (outer == lq::OUT_EXPABS) {
        const long double lam = -(long double)f->kappa;
        if (!(lam >= 0.0L) || !(lam * smax <= 700.0L)) return false;
        q.ym = (double)lam; q.ya = (double)(lam * alpha); q.E = (double)(lam * D); q.post = f->K;
        split_exp(-lam * D, q.c0, q.k0);
        split_exp(lam * D, q.c1, q.k1);
        // centred form (lq::pair_expabs_c): u = lam (l - sum beta / 2), c = |lam D| / 2
        const long double cth = fabsl(lam * D) / 2.0L;
        q.yc = (double)(lam * alpha - lam * D / 2.0L);
        q.cth = (double)cth;
        double cm;
        split_exp(-cth, cm, q.ke);
        split_exp(2.0L * cth, q.c2m, q.k2);
        q.on = 1;
        return true;
    }
    return false;
}

int launch_orbit_fft(lq_ctx* c, const lq_integrand* f, const OrbPlan& p, uint64_t unit0, int64_t ntiles,
                     double* tiles_dev) {
    int rc;
    const uint32_t *G, *Alo, *Ahi, *starts;
    const uint2* apow;
    if ((rc = orbit_tables(c, p, &G, &Alo, &Ahi, &apow, &starts))) return rc;
    const int d = f->d;
    const size_t smem = lq::kFftSmem;
    // the dynamic shared-memory opt-in of each kernel right before its first
    // launch: opting in all 17 instantiations up front made the lazy module
    // loader bring every one of them in (36 ms of the cold first call)
    void *W, *Hc, *dc;
    if ((rc = dev_buf(c, B_FFTW, sizeof(double2) * lq::kFftN, &W))) return rc;
    if (!c->fft_w) {
        lq::k_fft_twiddles<<<lq::kFftN / lq::kThreads, lq::kThreads, 0, c->stream>>>((double2*)W);
        c->launches++;
        CK(cudaGetLastError());
        c->fft_w = true;
    }
    const double nd = (double)p.n;
    const bool quad = is_quad_kind(f->kind);
    double bsum = 0.0;
    if ((rc = dev_buf(c, B_FFTH, sizeof(double2) * lq::kFftN * (quad ? 2 : 1), &Hc))) return rc;
    if (quad) {
        // centred form: b'_j = beta_j + gamma_j, q_j = gamma_j; alpha' = alpha + sum(beta/2 + gamma/4)
        std::vector<double> bq(2 * (size_t)d);
        for (int j = 0; j < d; ++j) {
            bq[j] = f->beta[j] + f->gamma[j];
            bq[d + j] = f->gamma[j];
            bsum += 0.5 * f->beta[j] + 0.25 * f->gamma[j];
        }
        bq.push_back(1.0);   // key tags: the Gaussian pair of spectra, d
        bq.push_back((double)d);
        if (c->fft_key != bq || c->fft_key_buf != Hc) {
            if ((rc = upload(c, B_AUX0, bq.data(), sizeof(double) * 2 * d, &dc))) return rc;
            if ((rc = smem_optin(c, (const void*)lq::k_fft_coeffs_pm, smem))) return rc;
            lq::k_fft_coeffs_pm<<<1, lq::kFftThreads, smem, c->stream>>>((const double*)dc, (const double*)dc + d, d,
                                                                        (const double2*)W, (double2*)Hc,
                                                                        (double2*)Hc + lq::kFftN);
            c->launches++;   // the coefficient transform
            CK(cudaGetLastError());
            c->fft_key.swap(bq);
            c->fft_key_buf = Hc;
        }
    } else {
        std::vector<double> cv(d);
        for (int j = 0; j < d; ++j) {
            cv[j] = f->beta[j] / nd;
            bsum += f->beta[j];
        }
        cv.push_back(0.0);   // key tags: one real spectrum, d
        cv.push_back((double)d);
        if (c->fft_key != cv || c->fft_key_buf != Hc) {
            if ((rc = upload(c, B_AUX0, cv.data(), sizeof(double) * d, &dc))) return rc;
            if ((rc = smem_optin(c, (const void*)lq::k_fft_coeffs, smem))) return rc;
            lq::k_fft_coeffs<<<1, lq::kFftThreads, smem, c->stream>>>((const double*)dc, d, (const double2*)W,
                                                                      (double2*)Hc);
            c->launches++;   // the coefficient transform
            CK(cudaGetLastError());
            c->fft_key.swap(cv);
            c->fft_key_buf = Hc;
        }
    }
    lq::FftHead h{};
    h.n = p.n; h.B = (uint32_t)p.m; h.units = p.units; h.qc = p.qc; h.h = p.h; h.zero = p.zero ? 1 : 0;
    h.G = G; h.Alo = Alo; h.Ahi = Ahi; h.apow = apow; h.starts = starts; h.W = (const double2*)W;
    h.Hc = (const double2*)Hc;
    h.alpha = f->alpha; h.alphaB = f->alpha + bsum; h.K = f->K; h.A = f->A; h.Bc = f->B; h.C0 = f->C0;
    h.kappa = f->kappa; h.pw = f->power;
    const int outer = lin_outer(f->kind);
    const bool fast = !quad && outer != lq::OUT_PROG && pair_fast_consts(f, bsum, h.pf);
    if (outer == lq::OUT_PROG) {
        void* dg;
        if ((rc = upload(c, B_PROG, f->outer.insn, sizeof(lq_insn) * f->outer.n_insn, &dg))) return rc;
        h.g_insn = (const lq_insn*)dg;
        h.g_n = f->outer.n_insn;
        h.g_result = f->outer.result;
    }
    // the exp table of the pair outer; the centred exp-abs form folds e^{-c}
    // into it (lq::pair_expabs_c)
    long double tscale = 1.0L;
    if (fast && outer == lq::OUT_EXPABS && LQ_FFT_CENTRED) {
        tscale = expl(-(long double)h.pf.cth);   // e^{-c} >= e^{-700}: a normal double
    }
    for (int j = 0; j < lq::kFftExpTab; ++j)
        h.etab[j] = make_double2((double)(exp2l(j / (long double)lq::kFftExpTab) * tscale),
                                 (double)(exp2l(-(j / (long double)lq::kFftExpTab)) * tscale));
    // several tiles per CTA once there are many waves: the twiddle fill is
    // paid once per CTA
    const int per = (int)std::max<int64_t>(1, std::min<int64_t>(kFftTilesPerCta, ntiles / (2 * 148 * 16)));
    const dim3 g((unsigned)((ntiles + per - 1) / per)), b(lq::kFftThreads);
    if (quad) {
        const double2* Hm = (const double2*)Hc + lq::kFftN;
        t_begin(c);
        if (quad_outer_of(f->kind) == lq::OUT_SINCOS) {
            if ((rc = smem_optin(c, (const void*)lq::k_orbit_fft_quad<lq::OUT_SINCOS>, smem))) return rc;
            lq::k_orbit_fft_quad<lq::OUT_SINCOS><<<g, b, smem, c->stream>>>(h, Hm, unit0, ntiles, per, tiles_dev);
        } else {
            if ((rc = smem_optin(c, (const void*)lq::k_orbit_fft_quad<lq::OUT_EXP>, smem))) return rc;
            lq::k_orbit_fft_quad<lq::OUT_EXP><<<g, b, smem, c->stream>>>(h, Hm, unit0, ntiles, per, tiles_dev);
        }
        t_end(c);
        CK(cudaGetLastError());
        return LQ_OK;
    }
    c->param_bytes += (int64_t)(sizeof(h) + sizeof(unit0) + sizeof(ntiles) + sizeof(per) + sizeof(tiles_dev));
    t_begin(c);
    // positions per thread that can hold a chain point: B <= RM N/R
    const int rm = (int)((p.m + lq::kFftThreads - 1) / lq::kFftThreads);
#define LQ_FFT_LIN(O, F, RM) do { if ((rc = smem_optin(c, (const void*)lq::k_orbit_fft<O, F, RM>, smem))) return rc; \
                                  lq::k_orbit_fft<O, F, RM><<<g, b, smem, c->stream>>>(h, unit0, ntiles, per, tiles_dev); } while (0)
#define LQ_FFT_FAST(O) do { if (rm <= 12) LQ_FFT_LIN(O, true, 12); else if (rm == 13) LQ_FFT_LIN(O, true, 13); \
                            else LQ_FFT_LIN(O, true, lq::kFftR); } while (0)
    if (outer == lq::OUT_EXP) { if (fast) LQ_FFT_FAST(lq::OUT_EXP); else LQ_FFT_LIN(lq::OUT_EXP, false, lq::kFftR); }
    else if (outer == lq::OUT_SINCOS) { if (fast) LQ_FFT_FAST(lq::OUT_SINCOS); else LQ_FFT_LIN(lq::OUT_SINCOS, false, lq::kFftR); }
    else if (outer == lq::OUT_EXPABS) { if (fast) LQ_FFT_FAST(lq::OUT_EXPABS); else LQ_FFT_LIN(lq::OUT_EXPABS, false, lq::kFftR); }
    else if (outer == lq::OUT_PROG) LQ_FFT_LIN(lq::OUT_PROG, false, lq::kFftR);
    else LQ_FFT_LIN(lq::OUT_POW, false, lq::kFftR);
#undef LQ_FFT_FAST
#undef LQ_FFT_LIN
    t_end(c);
    CK(cudaGetLastError());
    return LQ_OK;
}

int launch_orbit(lq_ctx* c, const lq_integrand* f, const OrbPlan& p, uint64_t unit0, int64_t ntiles,
                 double* tiles_dev) {
    int rc;
    const uint32_t* G;
    const uint32_t *Alo, *Ahi;
    if ((rc = orbit_tables(c, p, &G, &Alo, &Ahi))) return rc;
    const int d = f->d, m = p.m;
    const int dpad = (d + m - 1) / m * m;
    const double nd = (double)p.n;
    lq::OrbHead h{};
    h.n = p.n; h.a = p.a; h.as = p.as; h.dpad = dpad; h.units = p.units; h.qc = p.qc; h.h = p.h;
    h.zero = p.zero ? 1 : 0;
    h.G = G; h.Alo = Alo; h.Ahi = Ahi;
    h.alpha = f->alpha; h.K = f->K; h.A = f->A; h.B = f->B; h.C0 = f->C0; h.kappa = f->kappa; h.pw = f->power;
    if (f->kind == LQ_FAM_PROD_QUAD) {
        ProdScale ps;
        if ((rc = prod_scale(f, p.n, ps))) return rc;
        h.M = ps.m;
        std::vector<double2> wc(dpad);
        for (int j = 0; j < dpad; ++j) wc[j] = j < d ? make_double2(ps.w[j], ps.c[j]) : make_double2(0.0, 1.0);
        if (dpad <= 128) return orbit_prod<128>(c, h, wc, d, (int)ps.off, ps.R - 1, unit0, ntiles, tiles_dev);
        if (dpad <= 512) return orbit_prod<512>(c, h, wc, d, (int)ps.off, ps.R - 1, unit0, ntiles, tiles_dev);
        return orbit_prod<lq::kOrbProdDims>(c, h, wc, d, (int)ps.off, ps.R - 1, unit0, ntiles, tiles_dev);
    }
    if (is_quad_kind(f->kind)) {
        const int outer = quad_outer_of(f->kind);
        int sigma = 1074 + std::ilogb(1.0 / nd) - 1000;
        if (sigma < 0) sigma = 0;
        h.M = std::ldexp(1.0 / nd, 1074 - sigma);
        h.half = std::ldexp(0.5, -sigma);
        h.scale = 1.0;
        std::vector<double2> bq(dpad);
        double C0 = 0.0;
        for (int j = 0; j < dpad; ++j) {
            if (j < d) {
                bq[j].x = std::ldexp(f->beta[j] + f->gamma[j], sigma);
                bq[j].y = std::ldexp(f->gamma[j], 2 * sigma);
                if (!std::isfinite(bq[j].x) || !std::isfinite(bq[j].y))
                    return fail(LQ_ERR_VALUE, "quadratic coefficient out of range");
                C0 += 0.5 * f->beta[j] + 0.25 * f->gamma[j];
            } else {
                bq[j].x = 0.0;
                bq[j].y = 0.0;
            }
        }
        h.alphaB = f->alpha + C0;   // f = K exp(alpha + C + odd + even) at x, odd -> -odd at 1 - x
        h.bsum = 0.0;
        if (dpad <= 120) return orbit_quad<120>(c, h, bq, outer, unit0, ntiles, tiles_dev);
        if (dpad <= 504) return orbit_quad<504>(c, h, bq, outer, unit0, ntiles, tiles_dev);
        return orbit_quad<lq::kOrbQuadDims>(c, h, bq, outer, unit0, ntiles, tiles_dev);
    }
    double maxabs = 0.0, bsum = 0.0;
    for (int j = 0; j < d; ++j) {
        maxabs = fmax(maxabs, fabs(f->beta[j]));
        bsum += f->beta[j];
    }
    if (!std::isfinite(maxabs)) return fail(LQ_ERR_VALUE, "non-finite coefficient");
    int sigma = 0;
    if (maxabs > 0.0) {
        sigma = 1074 + std::ilogb(maxabs / nd) + 1 - 1020;
        if (sigma < 0) sigma = 0;
    }
    std::vector<double> cv(dpad);
    for (int j = 0; j < dpad; ++j) cv[j] = j < d ? std::ldexp(f->beta[j] / nd, 1074 - sigma) : 0.0;
    h.scale = std::ldexp(1.0, sigma);
    h.bsum = bsum;
    h.alphaB = f->alpha + bsum;   // alpha + <beta, 1 - x> = (alpha + sum beta) - <beta, x>
    h.M = 0.0;
    h.half = 0.0;
    pair_fast_scaled(f, bsum, h.scale, h.pf);
    const int outer = lin_outer(f->kind);
    if (dpad <= 120) return orbit_lin<120>(c, h, cv, outer, unit0, ntiles, tiles_dev);
    if (dpad <= 1008) return orbit_lin<1008>(c, h, cv, outer, unit0, ntiles, tiles_dev);
    return orbit_lin<lq::kOrbLinDims>(c, h, cv, outer, unit0, ntiles, tiles_dev);
}

// Reduction layout of a full-lattice sum: units are points (index kernels) or
// chains of paired points (orbit kernel); tiles of tile_units units, super-chunks
// of LQ_SUPER_TILES tiles.
struct Layout {
    uint64_t tile_units = 0, n_units = 0;
    std::shared_ptr<const OrbPlan> orb;
    bool pair = false, fft = false;
    // n = 2^k Korobov rules: level segments of tiles, then the small lattice
    std::shared_ptr<const Pow2Plan> p2;
    std::vector<int64_t> seg;          // first tile of each level, of the small lattice, and the end
    uint64_t small_n = 0, small_tp = 0;
    int64_t super_tiles = LQ_SUPER_TILES;   // tiles per super-chunk (256 for the heavy FFT tiles)
    int mode() const {
        if (p2) return LQ_LAYOUT_ORBIT_POW2;
        return orb ? (fft ? LQ_LAYOUT_ORBIT_FFT : LQ_LAYOUT_ORBIT) : pair ? LQ_LAYOUT_PAIRED : LQ_LAYOUT_INDEX;
    }
};

// n = 2^k Korobov rules of the linear and Gaussian families (mirror pairs).
std::shared_ptr<const Pow2Plan> pow2_for(const lq_integrand* f, uint64_t n, const uint64_t* z, bool* fft) {
    *fft = false;
    if (orbit_mode() == 0 || !z || f->d < 2 || !(is_lin_kind(f->kind) || is_quad_kind(f->kind))) return nullptr;
    if (n < (1ull << 12) || n > (1ull << 31) || (n & (n - 1))) return nullptr;
    if (!f->beta || (is_quad_kind(f->kind) && !f->gamma)) return nullptr;
    if (z[0] != 1) return nullptr;
    const uint64_t a = z[1];
    if (!(a & 1)) return nullptr;
    for (int j = 2; j < f->d; ++j)
        if (z[j] != z[j - 1] * a % n) return nullptr;
    int k = 0;
    while ((1ull << k) < n) ++k;
    const bool quad = is_quad_kind(f->kind);
    bool use_fft = fft_wanted(f, n);
    int len = use_fft ? lq::kFftN - f->d + 1 : lq::orb_len(quad ? lq::FAM_QUAD : lq::FAM_LIN);
    if (!use_fft) {
        const int cap = quad ? lq::kOrbQuadDims : lq::kOrbLinDims;
        if ((f->d + len - 1) / len * len > cap) return nullptr;
    }
    auto P = pow2_plan((uint32_t)a, k, len, use_fft);
    if (P) *fft = use_fft;
    return P;
}

// Chains per tile of one level: two per FFT tile (one for the Gaussian form),
// one per thread of the direct orbit kernel.
uint64_t level_units_per_tile(const lq_integrand* f, const OrbPlan& lp) {
    return lp.apow.empty() ? lq::kThreads : (is_quad_kind(f->kind) ? 1 : 2);
}

// Composite n (not a power of two) Korobov rules of the linear and Gaussian
// families with gcd(a, n) = 1: the divisor-class levels of div_plan.
std::shared_ptr<const Pow2Plan> divplan_for(const lq_integrand* f, uint64_t n, const uint64_t* z, bool* fft) {
    *fft = false;
    if (orbit_mode() == 0 || !z || f->d < 2) return nullptr;
    if (!(is_lin_kind(f->kind) || is_quad_kind(f->kind) || f->kind == LQ_FAM_LIN_PROG)) return nullptr;
    if (n < (1ull << 12) || n > (1ull << 31) || !(n & (n - 1)) || is_prime32((uint32_t)n)) return nullptr;
    if (!f->beta || (is_quad_kind(f->kind) && !f->gamma)) return nullptr;
    if (z[0] != 1) return nullptr;
    const uint64_t a = z[1];
    if (a < 2 || gcd64(a, n) != 1) return nullptr;
    for (int j = 2; j < f->d; ++j)
        if (z[j] != z[j - 1] * a % n) return nullptr;
    const bool quad = is_quad_kind(f->kind);
    const bool use_fft = fft_wanted(f, n);
    int len_direct = lq::orb_len(quad ? lq::FAM_QUAD : lq::FAM_LIN);
    const int cap = quad ? lq::kOrbQuadDims : lq::kOrbLinDims;
    if (f->kind == LQ_FAM_LIN_PROG || (f->d + len_direct - 1) / len_direct * len_direct > cap) len_direct = 0;
    if (!use_fft && len_direct == 0) return nullptr;
    auto P = div_plan((uint32_t)n, (uint32_t)a, use_fft ? lq::kFftN - f->d + 1 : len_direct, use_fft, len_direct);
    if (P) *fft = P->fft;
    return P;
}

Layout plan_layout(const lq_integrand* f, uint64_t n, const uint64_t* z);

// The layout of (f, n, z) is a pure function of n, z, f's kind, d, beta and
// gamma and the LQ_ORBIT / LQ_FFT / LQ_PAIR switches.  Deciding it costs
// O(d) 64-bit modular checks plus the planners' cache lookups (11 us at
// d = 1000), paid on every call; a repeated call (the e2e loop, sub-range
// calls of one sum) matches the last few inputs by bytes instead (~1 us).
struct LayoutMemo {
    uint64_t n = 0;
    int kind = -1, d = -1, has_gamma = 0;
    std::string env;
    std::vector<uint64_t> z;
    std::vector<double> beta, gamma;
    Layout L;
};

std::string layout_env() {
    std::string s;
    for (const char* k : {"LQ_ORBIT", "LQ_FFT", "LQ_PAIR"}) {
        const char* e = std::getenv(k);
        s += e ? e : "";
        s += '\x1f';
    }
    return s;
}

Layout layout_of(const lq_integrand* f, uint64_t n, const uint64_t* z) {
    constexpr int kMemo = 4;
    static thread_local LayoutMemo memo[kMemo];
    static thread_local int next = 0;
    if (!z || !f->beta || f->d < 1) return plan_layout(f, n, z);
    const int d = f->d;
    const int hg = f->gamma != nullptr;
    std::string env = layout_env();
    for (auto& m : memo)
        if (m.n == n && m.kind == f->kind && m.d == d && m.has_gamma == hg && m.env == env &&
            !std::memcmp(m.z.data(), z, sizeof(uint64_t) * d) &&
            !std::memcmp(m.beta.data(), f->beta, sizeof(double) * d) &&
            (!hg || !std::memcmp(m.gamma.data(), f->gamma, sizeof(double) * d)))
            return m.L;
    Layout L = plan_layout(f, n, z);
    LayoutMemo& m = memo[next];
    next = (next + 1) % kMemo;
    m.n = n; m.kind = f->kind; m.d = d; m.has_gamma = hg; m.env = std::move(env);
    m.z.assign(z, z + d);
    m.beta.assign(f->beta, f->beta + d);
    if (hg) m.gamma.assign(f->gamma, f->gamma + d); else m.gamma.clear();
    m.L = L;
    return L;
}

Layout plan_layout(const lq_integrand* f, uint64_t n, const uint64_t* z) {
    Layout L;
    bool fft2 = false;
    if ((L.p2 = pow2_for(f, n, z, &fft2)) || (L.p2 = divplan_for(f, n, z, &fft2))) {
        L.fft = fft2;
        int64_t t = 0;
        for (const auto& lp : L.p2->levels) {   // each level: FFT-form or direct chains
            const uint64_t tu = level_units_per_tile(f, *lp);
            L.seg.push_back(t);
            t += (int64_t)((lp->units + tu - 1) / tu);
        }
        L.small_n = L.p2->small_n;
        L.small_tp = tile_points(f, L.small_n);
        L.seg.push_back(t);
        t += (int64_t)((L.small_n + L.small_tp - 1) / L.small_tp);
        L.seg.push_back(t);
        L.tile_units = 1;                 // units are tiles
        L.n_units = (uint64_t)t;
        if (fft2) L.super_tiles = 256;
        return L;
    }
    L.orb = orbit_for(f, n, z, &L.fft);
    if (L.orb) {
        // FFT form: two chains per CTA (linear families) or one (Gaussian family)
        L.tile_units = L.fft ? (is_quad_kind(f->kind) ? 1 : 2) : lq::kThreads;
        if (L.fft) L.super_tiles = 256;
        L.n_units = L.orb->units;
    } else if (uses_family_kernel(f, n) && pair_ok(f, n, z)) {
        L.pair = true;
        L.tile_units = tile_points(f, n, true);
        L.n_units = n / 2 + 1;
    } else {
        L.tile_units = tile_points(f, n);
        L.n_units = n;
    }
    return L;
}

// Super-chunk partials of tiles[0 .. ntiles) (groups of L.super_tiles) into out.
int super_partials(lq_ctx* c, const Layout& L, const double* tiles, int64_t ntiles, int64_t groups, double* out) {
    if (L.super_tiles == 256)
        lq::k_reduce256<<<(unsigned)groups, lq::kThreads, 0, c->stream>>>(tiles, ntiles, out);
    else
        lq::k_reduce1024<<<(unsigned)groups, lq::kThreads, 0, c->stream>>>(tiles, ntiles, out);
    c->launches++;
    CK(cudaGetLastError());
    return LQ_OK;
}

// Full sum of a layout's tiles: the super-chunk partials, then the fixed tree
// over them -- the same association as lq_lattice_partials + lq_reduce_sum,
// so one GPU and any number of ranks agree bit for bit.
int layout_total(lq_ctx* c, const Layout& L, const double* tiles, int64_t ntiles, double** result) {
    if (L.super_tiles == LQ_SUPER_TILES) return reduce_dev(c, tiles, ntiles, result);
    const int64_t groups = (ntiles + L.super_tiles - 1) / L.super_tiles;
    void* parts;
    int rc;
    if ((rc = dev_buf(c, B_PART, sizeof(double) * groups, &parts))) return rc;
    if ((rc = super_partials(c, L, tiles, ntiles, groups, (double*)parts))) return rc;
    return reduce_dev(c, (const double*)parts, groups, result);
}

// Tiles [T0, T1) of a 2^k layout into tiles_dev[0 .. T1 - T0).
int launch_pow2_tiles(lq_ctx* c, const lq_integrand* f, const uint64_t* z, const Layout& L, int64_t T0, int64_t T1,
                      double* tiles_dev) {
    int rc;
    const int nl = (int)L.p2->levels.size();
    for (int l = 0; l <= nl; ++l) {
        const int64_t lo = std::max(T0, L.seg[l]), hi = std::min(T1, L.seg[l + 1]);
        if (hi <= lo) continue;
        double* out = tiles_dev + (lo - T0);
        if (l < nl) {
            const OrbPlan& lp = *L.p2->levels[l];
            const uint64_t unit0 = (uint64_t)(lo - L.seg[l]) * level_units_per_tile(f, lp);
            rc = lp.apow.empty() ? launch_orbit(c, f, lp, unit0, hi - lo, out)
                                 : launch_orbit_fft(c, f, lp, unit0, hi - lo, out);
        } else {
            // the small lattice (mod 2^m0, or m0 for composite n): every class
            // too short for chains, and the point 0
            std::vector<uint64_t> zs(f->d);
            for (int j = 0; j < f->d; ++j) zs[j] = z[j] % L.small_n;
            const uint64_t base = (uint64_t)(lo - L.seg[l]) * L.small_tp;
            const uint64_t end = std::min<uint64_t>((uint64_t)(hi - L.seg[l]) * L.small_tp, L.small_n);
            rc = launch_tiles(c, f, L.small_n, zs.data(), base, end, hi - lo, out);
        }
        if (rc) return rc;
    }
    return LQ_OK;
}

}  // namespace

// ======================================================================= ABI
extern "C" {

const char* lq_last_error(void) { return g_err.c_str(); }
int lq_abi_version(void) { return LQ_ABI_VERSION; }

int lq_ctx_create(int device, lq_ctx** out) {
    if (!out) return fail(LQ_ERR_VALUE, "null output pointer");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(LQ_ERR_VALUE, "device %d out of range (%d devices)", device, ndev);
    lq_ctx* c = new lq_ctx();
    c->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->cc_major, cudaDevAttrComputeCapabilityMajor, device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->cc_minor, cudaDevAttrComputeCapabilityMinor, device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
    if (e != cudaSuccess) {
        delete c;
        return fail(LQ_ERR_CUDA, "context creation failed: %s", cudaGetErrorString(e));
    }
    if (c->cc_major != 10) {
        int cc = c->cc_major * 10 + c->cc_minor;
        delete c;
        return fail(LQ_ERR_UNSUPPORTED, "liblq is built for sm_100a (B200); device has sm_%d", cc);
    }
    c->stream = c->own;
    *out = c;
    return LQ_OK;
}

int lq_ctx_destroy(lq_ctx* c) {
    if (!c) return LQ_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (int i = 0; i < B_NBUF; ++i)
        if (c->dbuf[i]) cudaFree(c->dbuf[i]);
    for (auto& kv : c->orb_tabs) cudaFree(kv.second.first);
    if (c->hpin) cudaFreeHost(c->hpin);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->own) cudaStreamDestroy(c->own);
    delete c;
    return LQ_OK;
}

int lq_ctx_set_stream(lq_ctx* c, void* stream) {
    int rc = set_dev(c);
    if (rc) return rc;
    CK(cudaStreamSynchronize(c->stream));
    c->hoff = 0;
    c->stream = stream ? (cudaStream_t)stream : c->own;
    return LQ_OK;
}

int lq_sync(lq_ctx* c) {
    int rc = set_dev(c);
    if (rc) return rc;
    CK(cudaStreamSynchronize(c->stream));
    return LQ_OK;
}

int lq_device_info(lq_ctx* c, int* sm, int* maj, int* mnr) {
    if (!c) return fail(LQ_ERR_VALUE, "null lq_ctx");
    if (sm) *sm = c->sm_count;
    if (maj) *maj = c->cc_major;
    if (mnr) *mnr = c->cc_minor;
    return LQ_OK;
}

int lq_ctx_enable_timing(lq_ctx* c, int enable) {
    if (!c) return fail(LQ_ERR_VALUE, "null lq_ctx");
    c->timing = enable != 0;
    c->launches = 0;
    return LQ_OK;
}

int lq_ctx_transfer_bytes(lq_ctx* c, int64_t* h2d, int64_t* d2h, int64_t* params) {
    if (!c) return fail(LQ_ERR_VALUE, "null lq_ctx");
    if (h2d) *h2d = c->h2d_bytes;
    if (d2h) *d2h = c->d2h_bytes;
    if (params) *params = c->param_bytes;
    return LQ_OK;
}

int lq_last_kernel_ms(lq_ctx* c, float* ms, int64_t* launches) {
    int rc = set_dev(c);
    if (rc) return rc;
    float t = 0.f;
    if (c->timing) {
        CK(cudaEventSynchronize(c->ev1));
        CK(cudaEventElapsedTime(&t, c->ev0, c->ev1));
    }
    if (ms) *ms = t;
    if (launches) *launches = c->launches;
    return LQ_OK;
}

int lq_points_block(lq_ctx* c, int32_t d, uint64_t n, const uint64_t* z, int64_t start, int64_t stop, double* out,
                    int32_t out_is_device) {
    int rc = set_dev(c);
    if (rc) return rc;
    if ((rc = check_lattice(n, z, d))) return rc;
    if (start < 0 || stop < start) return fail(LQ_ERR_VALUE, "bad index range [%lld, %lld)", (long long)start, (long long)stop);
    const uint64_t m = (uint64_t)(stop - start);
    if (m == 0) return LQ_OK;
    if (!out) return fail(LQ_ERR_VALUE, "null output");
    void* dz;
    if ((rc = upload(c, B_AUX0, z, sizeof(uint64_t) * d, &dz))) return rc;
    const uint64_t n_elem = m * (uint64_t)d;
    double* dst = out;
    if (!out_is_device) {
        void* p;
        if ((rc = dev_buf(c, B_OUT, n_elem * sizeof(double), &p))) return rc;
        dst = (double*)p;
    }
    const double n_d = (double)n, inv = 1.0 / n_d;
    if (n <= (1ull << 31)) {
        std::vector<uint32_t> zz(2 * (size_t)d);
        for (int j = 0; j < d; ++j) {
            zz[2 * j] = (uint32_t)z[j];
            zz[2 * j + 1] = (uint32_t)(((uint64_t)z[j] << 32) / n);
        }
        void* dzz;
        if ((rc = upload(c, B_TAB, zz.data(), zz.size() * 4, &dzz))) return rc;
        const uint64_t row_tiles = (m + lq::kPtRows - 1) / lq::kPtRows;
        const uint32_t col_tiles = (uint32_t)((d + lq::kPtCols - 1) / lq::kPtCols);
        if (row_tiles * col_tiles > 0x7fffffffull) return fail(LQ_ERR_VALUE, "point block too large");
        t_begin(c);
        lq::k_points_tiled<<<(unsigned)(row_tiles * col_tiles), lq::kThreads, 0, c->stream>>>(
            (const uint2*)dzz, (uint32_t)d, (uint32_t)n, n_d, inv, (uint64_t)start, m, col_tiles, dst);
        t_end(c);
    } else {
        int64_t blocks = (int64_t)((n_elem + lq::kThreads - 1) / lq::kThreads);
        int grid = grid_for(c, (const void*)lq::k_points, blocks);
        t_begin(c);
        lq::k_points<<<grid, lq::kThreads, 0, c->stream>>>((const uint64_t*)dz, (uint32_t)d, n, n_d, inv, inv, (uint64_t)start, n_elem, dst);
        t_end(c);
    }
    CK(cudaGetLastError());
    if (!out_is_device) {
        CK(cudaMemcpyAsync(out, dst, n_elem * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        c->d2h_bytes += (int64_t)(n_elem * sizeof(double));
        CK(cudaStreamSynchronize(c->stream));
    }
    return LQ_OK;
}

int lq_lattice_layout(const lq_integrand* f, uint64_t n, const uint64_t* z, int64_t* tile_units, int64_t* n_supers,
                      int64_t* n_units, int32_t* mode, int64_t* super_tiles) {
    int rc;
    if ((rc = check_integrand(f))) return rc;
    if (z && (rc = check_lattice(n, z, f->d))) return rc;
    const Layout L = layout_of(f, n, z);
    const uint64_t sp = L.tile_units * (uint64_t)L.super_tiles;
    if (tile_units) *tile_units = (int64_t)L.tile_units;
    if (n_supers) *n_supers = (int64_t)((L.n_units + sp - 1) / sp);
    if (n_units) *n_units = (int64_t)L.n_units;
    if (mode) *mode = L.mode();
    if (super_tiles) *super_tiles = L.super_tiles;
    return LQ_OK;
}

int lq_lattice_partials(lq_ctx* c, const lq_integrand* f, uint64_t n, const uint64_t* z, int64_t s_begin,
                        int64_t s_end, double* out_dev) {
    int rc = set_dev(c);
    if (rc) return rc;
    if ((rc = check_integrand(f)) || (rc = check_lattice(n, z, f->d))) return rc;
    const Layout L = layout_of(f, n, z);
    const uint64_t tp = L.tile_units, sp = tp * (uint64_t)L.super_tiles;
    const int64_t ns = (int64_t)((L.n_units + sp - 1) / sp);
    if (s_begin < 0 || s_end > ns || s_end < s_begin)
        return fail(LQ_ERR_VALUE, "super-chunk range [%lld, %lld) outside [0, %lld)", (long long)s_begin, (long long)s_end, (long long)ns);
    if (s_end == s_begin) return LQ_OK;
    const uint64_t base = (uint64_t)s_begin * sp;
    const uint64_t end = std::min<uint64_t>((uint64_t)s_end * sp, L.n_units);
    const int64_t ntiles = (int64_t)((end - base + tp - 1) / tp);
    void* tiles;
    if ((rc = dev_buf(c, B_TILES, sizeof(double) * ntiles, &tiles))) return rc;
    if (L.p2) {
        if ((rc = launch_pow2_tiles(c, f, z, L, (int64_t)base, (int64_t)end, (double*)tiles))) return rc;
    } else if (L.orb) {
        if ((rc = L.fft ? launch_orbit_fft(c, f, *L.orb, base, ntiles, (double*)tiles)
                        : launch_orbit(c, f, *L.orb, base, ntiles, (double*)tiles))) return rc;
    } else {
        if ((rc = launch_tiles(c, f, n, z, base, end, ntiles, (double*)tiles, L.pair))) return rc;
    }
    return super_partials(c, L, (const double*)tiles, ntiles, s_end - s_begin, out_dev);
}

int lq_layout_cover(const lq_integrand* f, uint64_t n, const uint64_t* z, int64_t* missed, int64_t* repeated) {
    int rc;
    if ((rc = check_integrand(f)) || (rc = check_lattice(n, z, f->d))) return rc;
    if (!missed || !repeated) return fail(LQ_ERR_VALUE, "null output");
    if (n > (1ull << 26)) return fail(LQ_ERR_UNSUPPORTED, "cover check supports n <= 2^26");
    const Layout L = layout_of(f, n, z);
    std::vector<uint8_t> hits(n, 0);
    auto mark = [&](uint64_t i) { if (hits[i] < 255) ++hits[i]; };
    auto mark_plan = [&](const OrbPlan& p, uint64_t scale) {   // points scale * u, u in the plan's unit classes
        const uint64_t m = p.n;
        for (uint64_t cs = 0; cs < p.G.size(); ++cs) {
            uint64_t u = p.G[cs];
            for (uint64_t t = 0; t < p.h; ++t) {
                const uint64_t i = scale * u % n;
                mark(i);
                if (p.mirror) mark((n - i) % n);
                u = u * p.a % m;
            }
        }
        if (p.zero) mark(0);
    };
    if (L.p2) {
        for (const auto& lp : L.p2->levels) mark_plan(*lp, n / lp->n);
        for (uint64_t t = 0; t < L.small_n; ++t) mark(n / L.small_n * t);
    } else if (L.orb) {
        mark_plan(*L.orb, 1);
    } else if (L.pair) {
        for (uint64_t i = 0; i <= n / 2; ++i) { mark(i); if (i && 2 * i != n) mark(n - i); }
    } else {
        for (uint64_t i = 0; i < n; ++i) mark(i);
    }
    int64_t miss = 0, rep = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (hits[i] == 0) ++miss;
        else if (hits[i] > 1) ++rep;
    }
    *missed = miss;
    *repeated = rep;
    return LQ_OK;
}

int lq_reduce_sum(lq_ctx* c, const double* vals, int64_t count, double* out) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (!out) return fail(LQ_ERR_VALUE, "null output");
    double* r;
    if ((rc = reduce_dev(c, vals, count, &r))) return rc;
    return read_scalar(c, r, out);
}

int lq_lattice_sum(lq_ctx* c, const lq_integrand* f, uint64_t n, const uint64_t* z, uint64_t i_begin, uint64_t i_end,
                   double* sum_out) {
    int rc = set_dev(c);
    if (rc) return rc;
    if ((rc = check_integrand(f)) || (rc = check_lattice(n, z, f->d))) return rc;
    if (!sum_out) return fail(LQ_ERR_VALUE, "null output");
    if (i_end < i_begin) return fail(LQ_ERR_VALUE, "bad index range");
    if (i_end == i_begin) {
        *sum_out = 0.0;
        return LQ_OK;
    }
    if (i_begin == 0 && i_end == n) {
        const Layout L = layout_of(f, n, z);
        if (L.p2) {
            const int64_t ntiles = (int64_t)L.n_units;
            void* tiles;
            if ((rc = dev_buf(c, B_TILES, sizeof(double) * ntiles, &tiles))) return rc;
            if ((rc = launch_pow2_tiles(c, f, z, L, 0, ntiles, (double*)tiles))) return rc;
            double* r;
            if ((rc = layout_total(c, L, (const double*)tiles, ntiles, &r))) return rc;
            return read_scalar(c, r, sum_out);
        }
        if (L.orb || L.pair) {
            const int64_t ntiles = (int64_t)((L.n_units + L.tile_units - 1) / L.tile_units);
            void* tiles;
            if ((rc = dev_buf(c, B_TILES, sizeof(double) * ntiles, &tiles))) return rc;
            if (L.orb) rc = L.fft ? launch_orbit_fft(c, f, *L.orb, 0, ntiles, (double*)tiles)
                                  : launch_orbit(c, f, *L.orb, 0, ntiles, (double*)tiles);
            else rc = launch_tiles(c, f, n, z, 0, L.n_units, ntiles, (double*)tiles, true);
            if (rc) return rc;
            double* r;
            if ((rc = layout_total(c, L, (const double*)tiles, ntiles, &r))) return rc;
            return read_scalar(c, r, sum_out);
        }
    }
    const uint64_t tp = tile_points(f, n);
    if (n <= (1ull << 31) && i_end > (1ull << 32) - 2 * tp)
        return fail(LQ_ERR_VALUE, "index range beyond 2^32 for n <= 2^31; reduce indices mod n");
    const int64_t ntiles = (int64_t)((i_end - i_begin + tp - 1) / tp);
    void* tiles;
    if ((rc = dev_buf(c, B_TILES, sizeof(double) * ntiles, &tiles))) return rc;
    if ((rc = launch_tiles(c, f, n, z, i_begin, i_end, ntiles, (double*)tiles))) return rc;
    double* r;
    if ((rc = reduce_dev(c, (const double*)tiles, ntiles, &r))) return rc;
    return read_scalar(c, r, sum_out);
}

// Monte Carlo over numpy's PCG64 stream (quad.mc_integrate, quad.py:79-93).
int lq_mc_sum(lq_ctx* c, const lq_program* pg, int32_t d, uint64_t n, const uint64_t* state, const uint64_t* inc,
              uint64_t i_begin, uint64_t i_end, double* sum_out) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (!pg || !pg->insn || pg->n_insn < 1) return fail(LQ_ERR_VALUE, "null program");
    if (!state || !inc || !sum_out) return fail(LQ_ERR_VALUE, "null argument");
    if (d < 1) return fail(LQ_ERR_VALUE, "dimension must be positive, got %d", d);
    if (n < 1) return fail(LQ_ERR_VALUE, "sample count must be >= 1, got %llu", (unsigned long long)n);
    if (i_end > n || i_end < i_begin) return fail(LQ_ERR_VALUE, "bad point range");
    if (pg->n_vars > d) return fail(LQ_ERR_VALUE, "program uses %d variables, d=%d", pg->n_vars, d);
    if ((unsigned __int128)n * (unsigned)d >= ((unsigned __int128)1 << 64))
        return fail(LQ_ERR_OVERFLOW, "n*d draws exceed 2^64");
    const int ns = pick_slots(pg->n_slots);
    if (ns < 0) return fail(LQ_ERR_UNSUPPORTED, "program needs %d slots (max %d)", pg->n_slots, LQ_MAX_SLOTS);
    if (i_end == i_begin) {
        *sum_out = 0.0;
        return LQ_OK;
    }
    typedef unsigned __int128 u128;
    const u128 M = ((u128)0x2360ED051FC65DA4ull << 64) | 0x4385DF649FCCF645ull;   // PCG_DEFAULT_MULTIPLIER_128
    const u128 I = ((u128)inc[1] << 64) | inc[0];
    auto pack = [](u128 A, u128 C) {
        return lq::Jump{(uint64_t)A, (uint64_t)(A >> 64), (uint64_t)C, (uint64_t)(C >> 64)};
    };
    std::vector<lq::Jump> tab(d + 1 + 64);
    u128 A = 1, C = 0;   // b draws: A_b = M^b, C_b = inc (M^(b-1) + ... + 1)
    for (int b = 0; b <= d; ++b) {
        tab[b] = pack(A, C);
        C = M * C + I;
        A = M * A;
    }
    u128 PA = M, PC = I;   // 2^k draws
    for (int k = 0; k < 64; ++k) {
        tab[d + 1 + k] = pack(PA, PC);
        PC = PA * PC + PC;
        PA = PA * PA;
    }
    void *dp, *dt;
    if ((rc = upload(c, B_PROG, pg->insn, sizeof(lq_insn) * pg->n_insn, &dp))) return rc;
    if ((rc = upload(c, B_AUX0, tab.data(), sizeof(lq::Jump) * tab.size(), &dt))) return rc;
    const int64_t ntiles = (int64_t)((i_end - i_begin + lq::kTile - 1) / lq::kTile);
    void* tiles;
    if ((rc = dev_buf(c, B_TILES, sizeof(double) * ntiles, &tiles))) return rc;
    const lq::Jump* jt = (const lq::Jump*)dt;
    const void* kern = ns == 32 ? (const void*)lq::k_prog_mc<32> : (const void*)lq::k_prog_mc<LQ_MAX_SLOTS>;
    const int grid = grid_for(c, kern, ntiles);
    t_begin(c);
    if (ns == 32)
        lq::k_prog_mc<32><<<grid, lq::kThreads, 0, c->stream>>>((const lq_insn*)dp, pg->n_insn, pg->result, d, jt,
                                                                 jt + d + 1, state[0], state[1], i_begin, i_end,
                                                                 ntiles, (double*)tiles);
    else
        lq::k_prog_mc<LQ_MAX_SLOTS><<<grid, lq::kThreads, 0, c->stream>>>((const lq_insn*)dp, pg->n_insn, pg->result,
                                                                          d, jt, jt + d + 1, state[0], state[1],
                                                                          i_begin, i_end, ntiles, (double*)tiles);
    t_end(c);
    CK(cudaGetLastError());
    double* r;
    if ((rc = reduce_dev(c, (const double*)tiles, ntiles, &r))) return rc;
    return read_scalar(c, r, sum_out);
}

namespace {
// Tile partials of the flat range [s_begin, s_end) (tiles of LQ_TILE nodes from
// s_begin) into tiles_out, or -- tiles_out == NULL -- their fixed-tree sum.
int tensor_tiles(lq_ctx* c, const lq_program* pg, int32_t d, const int64_t* counts, const double* nodes,
                 int32_t midpoint, uint64_t s_begin, uint64_t s_end, double* tiles_out, double* sum_out) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (!pg || !pg->insn || pg->n_insn < 1) return fail(LQ_ERR_VALUE, "null program");
    if (d < 0 || d > lq::kMaxAxes) return fail(LQ_ERR_UNSUPPORTED, "tensor sum supports 0..%d axes, got %d", lq::kMaxAxes, d);
    if (pg->n_vars > d) return fail(LQ_ERR_VALUE, "program uses %d axes, grid has %d", pg->n_vars, d);
    const int ns = pick_slots(pg->n_slots);
    if (ns < 0) return fail(LQ_ERR_UNSUPPORTED, "program needs %d slots (max %d)", pg->n_slots, LQ_MAX_SLOTS);
    std::vector<int64_t> off(d + 1, 0);
    for (int k = 0; k < d; ++k) {
        if (counts[k] < 1) return fail(LQ_ERR_VALUE, "axis %d has no nodes", k + 1);
        off[k + 1] = off[k] + counts[k];
    }
    if (s_end < s_begin) return fail(LQ_ERR_VALUE, "bad flat range");
    if (s_end == s_begin) {
        if (sum_out) *sum_out = 0.0;
        return LQ_OK;
    }
    void *dp, *dc, *doff, *dn;
    if ((rc = upload(c, B_PROG, pg->insn, sizeof(lq_insn) * pg->n_insn, &dp))) return rc;
    std::vector<int64_t> cnt(counts, counts + d);
    cnt.push_back(1);
    if ((rc = upload(c, B_AUX0, cnt.data(), sizeof(int64_t) * cnt.size(), &dc))) return rc;
    if ((rc = upload(c, B_AUX1, off.data(), sizeof(int64_t) * off.size(), &doff))) return rc;
    const int64_t total_nodes = off[d];
    if (midpoint || !nodes) {
        if ((rc = dev_buf(c, B_AUX2, sizeof(double) * (total_nodes + 1), &dn))) return rc;
        if (d > 0) {
            int64_t maxc = 1;
            for (int k = 0; k < d; ++k) maxc = std::max<int64_t>(maxc, counts[k]);
            dim3 g((unsigned)std::min<int64_t>((maxc + 255) / 256, 4096), (unsigned)d);
            lq::k_midpoint_nodes<<<g, 256, 0, c->stream>>>((const int64_t*)dc, (const int64_t*)doff, d, (double*)dn);
            c->launches++;
            CK(cudaGetLastError());
        }
    } else {
        if ((rc = upload(c, B_AUX2, nodes, sizeof(double) * total_nodes, &dn))) return rc;
    }
    const int64_t ntiles = (int64_t)((s_end - s_begin + LQ_TILE - 1) / LQ_TILE);
    void* tiles = tiles_out;
    if (!tiles && (rc = dev_buf(c, B_TILES, sizeof(double) * ntiles, &tiles))) return rc;
    const void* kern = ns == 32 ? (const void*)lq::k_prog_tensor<32> : (const void*)lq::k_prog_tensor<LQ_MAX_SLOTS>;
    int grid = grid_for(c, kern, ntiles);
    t_begin(c);
    if (cudaKernel_t jk = lq_jit_tensor_kernel(pg->jit)) {
        const void *pc = dc, *po = doff, *pn = dn;
        void* tp = tiles;
        int64_t nt = ntiles;
        void* args[] = {(void*)&d, (void*)&pc, (void*)&po, (void*)&pn, (void*)&s_begin, (void*)&s_end, (void*)&tp, (void*)&nt};
        // a resident grid striding over the tiles: the odometers are set up
        // once by division and carried from tile to tile
        const int jgrid = grid_for(c, (const void*)jk, ntiles, 2048 / lq::kThreads);
        CK(cudaLaunchKernel((const void*)jk, dim3((unsigned)jgrid), dim3(lq::kThreads), args, 0, c->stream));
    } else if (ns == 32)
        lq::k_prog_tensor<32><<<grid, lq::kThreads, 0, c->stream>>>((const lq_insn*)dp, pg->n_insn, pg->result, d, (const int64_t*)dc, (const int64_t*)doff, (const double*)dn, s_begin, s_end, ntiles, (double*)tiles);
    else
        lq::k_prog_tensor<LQ_MAX_SLOTS><<<grid, lq::kThreads, 0, c->stream>>>((const lq_insn*)dp, pg->n_insn, pg->result, d, (const int64_t*)dc, (const int64_t*)doff, (const double*)dn, s_begin, s_end, ntiles, (double*)tiles);
    t_end(c);
    CK(cudaGetLastError());
    if (tiles_out) return LQ_OK;
    double* r;
    if ((rc = reduce_dev(c, (const double*)tiles, ntiles, &r))) return rc;
    return read_scalar(c, r, sum_out);
}
}  // namespace

int lq_eval_array(lq_ctx* c, const lq_program* pg, const double* const* cols, int64_t m, int32_t on_device,
                  double* out) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (!pg || !pg->insn || pg->n_insn < 1) return fail(LQ_ERR_VALUE, "null program");
    if (m < 0) return fail(LQ_ERR_VALUE, "negative row count %lld", (long long)m);
    if (m == 0) return LQ_OK;
    if (!out) return fail(LQ_ERR_VALUE, "null output");
    if (pg->n_vars > 0 && !cols) return fail(LQ_ERR_VALUE, "null column table");
    const int ns = pick_slots(pg->n_slots);
    if (ns < 0) return fail(LQ_ERR_UNSUPPORTED, "program needs %d slots (max %d)", pg->n_slots, LQ_MAX_SLOTS);
    // every variable the bytecode reads must have a column
    for (int k = 0; k < pg->n_insn; ++k) {
        const lq_insn& in = pg->insn[k];
        if (in.op == lq::OP_VAR || in.op == lq::OP_ACC_ADDVAR) {
            if (in.b < 0 || in.b >= pg->n_vars || !cols[in.b])
                return fail(LQ_ERR_VALUE, "variable x[%d] has no column", in.b + 1);
        }
    }
    const int V = std::max(pg->n_vars, 1);
    const size_t bytes = sizeof(double) * (size_t)m;
    void *dp, *dptr, *dcols = nullptr, *dout = out;
    if ((rc = upload(c, B_PROG, pg->insn, sizeof(lq_insn) * pg->n_insn, &dp))) return rc;
    std::vector<const double*> ptrs(V, nullptr);
    if (on_device) {
        for (int b = 0; b < pg->n_vars; ++b) ptrs[b] = cols[b];
    } else {
        // host columns: one device block, V columns of m rows (pageable copies)
        if ((rc = dev_buf(c, B_AUX2, bytes * V, &dcols))) return rc;
        for (int b = 0; b < pg->n_vars; ++b) {
            if (!cols[b]) continue;
            ptrs[b] = (const double*)dcols + (size_t)b * m;
            CK(cudaMemcpyAsync((void*)ptrs[b], cols[b], bytes, cudaMemcpyHostToDevice, c->stream));
            c->h2d_bytes += (int64_t)bytes;
        }
        if ((rc = dev_buf(c, B_OUT, bytes, &dout))) return rc;
    }
    if ((rc = upload(c, B_AUX3, ptrs.data(), sizeof(void*) * V, &dptr))) return rc;
    const int64_t blocks = (m + lq::kThreads - 1) / lq::kThreads;
    const void* kern = ns == 32 ? (const void*)lq::k_prog_eval<32> : (const void*)lq::k_prog_eval<LQ_MAX_SLOTS>;
    const int grid = grid_for(c, kern, blocks);
    t_begin(c);
    if (ns == 32)
        lq::k_prog_eval<32><<<grid, lq::kThreads, 0, c->stream>>>((const lq_insn*)dp, pg->n_insn, pg->result,
                                                                  (const double* const*)dptr, m, (double*)dout);
    else
        lq::k_prog_eval<LQ_MAX_SLOTS><<<grid, lq::kThreads, 0, c->stream>>>((const lq_insn*)dp, pg->n_insn, pg->result,
                                                                            (const double* const*)dptr, m, (double*)dout);
    t_end(c);
    CK(cudaGetLastError());
    if (!on_device) {
        CK(cudaMemcpyAsync(out, dout, bytes, cudaMemcpyDeviceToHost, c->stream));
        c->d2h_bytes += (int64_t)bytes;
    }
    CK(cudaStreamSynchronize(c->stream));
    c->hoff = 0;
    return LQ_OK;
}

int lq_tensor_sum(lq_ctx* c, const lq_program* pg, int32_t d, const int64_t* counts, const double* nodes,
                  int32_t midpoint, uint64_t s_begin, uint64_t s_end, double* sum_out) {
    if (!sum_out) return fail(LQ_ERR_VALUE, "null output");
    return tensor_tiles(c, pg, d, counts, nodes, midpoint, s_begin, s_end, nullptr, sum_out);
}

int lq_tensor_partials(lq_ctx* c, const lq_program* pg, int32_t d, const int64_t* counts, const double* nodes,
                       int32_t midpoint, uint64_t total, int64_t t_begin, int64_t t_end, double* tiles_dev) {
    if (!tiles_dev) return fail(LQ_ERR_VALUE, "null output");
    const int64_t T = (int64_t)((total + LQ_TILE - 1) / LQ_TILE);
    if (t_begin < 0 || t_end > T || t_end < t_begin) return fail(LQ_ERR_VALUE, "bad tile range [%lld, %lld) of %lld",
                                                                 (long long)t_begin, (long long)t_end, (long long)T);
    const uint64_t s0 = (uint64_t)t_begin * LQ_TILE, s1 = std::min<uint64_t>((uint64_t)t_end * LQ_TILE, total);
    return tensor_tiles(c, pg, d, counts, nodes, midpoint, s0, s1, tiles_dev + t_begin, nullptr);
}

static int mdi_validate(const lq_insn* insn, int32_t n_insn, const lq_factor* fac, int32_t nf, int* nblk, int* ns) {
    if (nf < 0) return fail(LQ_ERR_VALUE, "negative factor count");
    int maxnb = 1, maxslots = 1;
    for (int f = 0; f < nf; ++f) {
        const lq_factor& F = fac[f];
        if (F.count < 1) return fail(LQ_ERR_VALUE, "factor %d has no nodes", f);
        if (F.r_len < 0 || F.p_len < 0 || F.r_off < 0 || F.p_off < 0 || F.r_off + F.r_len > n_insn || F.p_off + F.p_len > n_insn)
            return fail(LQ_ERR_VALUE, "factor %d program out of range", f);
        maxnb = std::max(maxnb, (F.count + LQ_NODE_BLOCK - 1) / LQ_NODE_BLOCK);
        maxslots = std::max(maxslots, F.n_slots);
    }
    *nblk = maxnb;
    *ns = pick_slots(maxslots);
    if (*ns < 0) return fail(LQ_ERR_UNSUPPORTED, "factor program needs %d slots", maxslots);
    if (n_insn > 0 && !insn) return fail(LQ_ERR_VALUE, "null instruction table");
    return LQ_OK;
}

int lq_mdi_block_sums(lq_ctx* c, const lq_insn* insn, int32_t n_insn, const lq_factor* fac, int32_t nf,
                      const double* nodes, int64_t n_nodes, int32_t shard, int32_t nshards, double* part_dev) {
    int rc = set_dev(c);
    if (rc) return rc;
    int nblk, ns;
    if ((rc = mdi_validate(insn, n_insn, fac, nf, &nblk, &ns))) return rc;
    if (nshards < 1 || shard < 0 || shard >= nshards) return fail(LQ_ERR_VALUE, "bad shard %d of %d", shard, nshards);
    if (nf == 0) return LQ_OK;
    for (int f = 0; f < nf; ++f) {
        const int64_t need = fac[f].reserved == LQ_FACTOR_SUPPLIED ? 2 : fac[f].count;
        if (fac[f].reserved == LQ_FACTOR_SUPPLIED && (fac[f].count != 1 || fac[f].node_off < 0))
            return fail(LQ_ERR_VALUE, "supplied factor %d needs count 1 and a node offset", f);
        if (fac[f].node_off >= 0 && (!nodes || (int64_t)fac[f].node_off + need > n_nodes))
            return fail(LQ_ERR_VALUE, "factor %d node table out of range", f);
    }
    void *dp, *dfac, *dn = nullptr;
    if ((rc = upload(c, B_PROG, insn, sizeof(lq_insn) * std::max(n_insn, 1), &dp))) return rc;
    if ((rc = upload(c, B_AUX0, fac, sizeof(lq_factor) * nf, &dfac))) return rc;
    if (nodes && n_nodes > 0 && (rc = upload(c, B_NODES, nodes, sizeof(double) * n_nodes, &dn))) return rc;
    dim3 g((unsigned)nf, (unsigned)nblk);
    t_begin(c);
    if (ns == 32)
        lq::k_mdi_blocks<32><<<g, lq::kThreads, 0, c->stream>>>((const lq_insn*)dp, (const lq_factor*)dfac, (const double*)dn, nblk, shard, nshards, part_dev);
    else
        lq::k_mdi_blocks<LQ_MAX_SLOTS><<<g, lq::kThreads, 0, c->stream>>>((const lq_insn*)dp, (const lq_factor*)dfac, (const double*)dn, nblk, shard, nshards, part_dev);
    t_end(c);
    CK(cudaGetLastError());
    return LQ_OK;
}

int lq_mdi_combine(lq_ctx* c, const double* part_dev, const lq_factor* fac, int32_t nf, int32_t nblk, const int32_t* term_ptr,
                   const int32_t* term_fac, const double* coef_re, const double* coef_im, const double* log_extra,
                   int32_t n_terms, double* out4) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (!out4 || n_terms < 0 || !term_ptr) return fail(LQ_ERR_VALUE, "bad combine arguments");
    const int32_t nk = term_ptr[n_terms];
    for (int k = 0; k < nk; ++k)
        if (term_fac[k] < 0 || term_fac[k] >= nf) return fail(LQ_ERR_VALUE, "term factor index out of range");
    // host-side packing of the small term tables
    std::vector<double> coef(2 * (size_t)std::max(n_terms, 1));
    for (int t = 0; t < n_terms; ++t) {
        coef[2 * t] = coef_re[t];
        coef[2 * t + 1] = coef_im ? coef_im[t] : 0.0;
    }
    void *dptr, *dfacidx, *dcoef, *dlog, *fw, *tw, *dout, *dfac;
    lq_factor dummy{};
    if ((rc = upload(c, B_FAC, nf > 0 ? (const void*)fac : (const void*)&dummy, sizeof(lq_factor) * std::max(nf, 1), &dfac))) return rc;
    if ((rc = upload(c, B_AUX1, term_ptr, sizeof(int32_t) * (n_terms + 1), &dptr))) return rc;
    if ((rc = upload(c, B_AUX2, term_fac, sizeof(int32_t) * std::max(nk, 1), &dfacidx))) return rc;
    if ((rc = upload(c, B_AUX3, coef.data(), sizeof(double) * coef.size(), &dcoef))) return rc;
    std::vector<double> lx(log_extra ? log_extra : coef.data(), log_extra ? log_extra + n_terms : coef.data());
    if (!log_extra) lx.assign(std::max(n_terms, 1), 0.0);
    if ((rc = upload(c, B_RED1, lx.data(), sizeof(double) * std::max<size_t>(lx.size(), 1), &dlog))) return rc;
    if ((rc = dev_buf(c, B_TILES, sizeof(double) * 2 * std::max(nf, 1), &fw))) return rc;
    if ((rc = dev_buf(c, B_RED0, sizeof(double) * 2 * std::max(n_terms, 1), &tw))) return rc;
    if ((rc = dev_buf(c, B_OUT, sizeof(double) * 4, &dout))) return rc;
    lq::k_mdi_combine<<<1, lq::kThreads, 0, c->stream>>>(part_dev, nf, nblk, (const lq_factor*)dfac,
                                                        (const int32_t*)dptr, (const int32_t*)dfacidx,
                                                        (const double*)dcoef, (const double*)dlog, n_terms,
                                                        (double*)fw, (double*)tw, (double*)dout);
    c->launches++;
    CK(cudaGetLastError());
    return read_scalar(c, (const double*)dout, out4, 4);
}

int lq_mdi_sum(lq_ctx* c, const lq_insn* insn, int32_t n_insn, const lq_factor* fac, int32_t nf,
               const double* nodes, int64_t n_nodes, const int32_t* term_ptr, const int32_t* term_fac, const double* coef_re, const double* coef_im,
               const double* log_extra, int32_t n_terms, double* out4) {
    int rc = set_dev(c);
    if (rc) return rc;
    int nblk, ns;
    if ((rc = mdi_validate(insn, n_insn, fac, nf, &nblk, &ns))) return rc;
    void* part;
    if ((rc = dev_buf(c, B_PART, sizeof(double) * 2 * (size_t)std::max(nf, 1) * nblk, &part))) return rc;
    if (nf > 0 && (rc = lq_mdi_block_sums(c, insn, n_insn, fac, nf, nodes, n_nodes, 0, 1, (double*)part))) return rc;
    return lq_mdi_combine(c, (const double*)part, fac, nf, nblk, term_ptr, term_fac, coef_re, coef_im, log_extra, n_terms, out4);
}

namespace {
// Per-node terms of the characteristic-function integral for nodes [k0, k1):
// vals[k], logmag[k] (device pointers indexed by the global node number).
int expabs_nodes(lq_ctx* c, int32_t d, const double* beta, const int32_t* counts, double alpha, const double* wn,
                 const double* ww, int32_t n_w, double kappa, int32_t k0, int32_t k1, double* vals, double* logmag) {
    int rc;
    void *db, *dc, *dw, *dww;
    if ((rc = upload(c, B_AUX0, beta, sizeof(double) * d, &db))) return rc;
    if ((rc = upload(c, B_AUX1, counts, sizeof(int32_t) * d, &dc))) return rc;
    if ((rc = upload(c, B_AUX2, wn, sizeof(double) * n_w, &dw))) return rc;
    if ((rc = upload(c, B_AUX3, ww, sizeof(double) * n_w, &dww))) return rc;
    if (k1 <= k0) return LQ_OK;
    // closed-form Dirichlet sums (default) or the direct N-term sums (LQ_CF_DIRECT=1)
    const char* direct = std::getenv("LQ_CF_DIRECT");
    const double *w0 = (const double*)dw + k0, *ww0 = (const double*)dww + k0;
    t_begin(c);
    if (direct && !std::strcmp(direct, "1")) {
        lq::k_cf_expabs<<<k1 - k0, lq::kThreads, 0, c->stream>>>((const double*)db, (const int32_t*)dc, d, alpha, w0,
                                                                 ww0, kappa, vals + k0, logmag + k0);
    } else {
        double bsum = 0.0;
        for (int j = 0; j < d; ++j) bsum += beta[j];
        lq::k_cf_expabs_closed<<<k1 - k0, lq::kThreads, 0, c->stream>>>((const double*)db, (const int32_t*)dc, d,
                                                                        alpha + 0.5 * bsum, w0, ww0, kappa,
                                                                        vals + k0, logmag + k0);
    }
    t_end(c);
    CK(cudaGetLastError());
    return LQ_OK;
}
}  // namespace

int lq_mdi_expabs(lq_ctx* c, int32_t d, const double* beta, const int32_t* counts, double alpha, const double* wn,
                  const double* ww, int32_t n_w, double kappa, double* out2, double* logmag) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (d < 1 || !beta || !counts || !wn || !ww || n_w < 1 || !out2) return fail(LQ_ERR_VALUE, "bad expabs arguments");
    if (!(kappa < 0.0)) return fail(LQ_ERR_VALUE, "kappa must be negative");
    void *dv, *dl;
    if ((rc = dev_buf(c, B_TILES, sizeof(double) * n_w, &dv))) return rc;
    if ((rc = dev_buf(c, B_PART, sizeof(double) * n_w, &dl))) return rc;
    if ((rc = expabs_nodes(c, d, beta, counts, alpha, wn, ww, n_w, kappa, 0, n_w, (double*)dv, (double*)dl))) return rc;
    double* r;
    if ((rc = reduce_dev(c, (const double*)dv, n_w, &r))) return rc;
    double s;
    if ((rc = read_scalar(c, r, &s))) return rc;
    if (logmag) {
        CK(cudaMemcpyAsync(logmag, dl, sizeof(double) * n_w, cudaMemcpyDeviceToHost, c->stream));
        c->d2h_bytes += (int64_t)(sizeof(double) * n_w);
        CK(cudaStreamSynchronize(c->stream));
    }
    out2[0] = s == 0.0 ? -INFINITY : std::log(std::fabs(s));
    out2[1] = s > 0.0 ? 1.0 : (s < 0.0 ? -1.0 : 0.0);
    return LQ_OK;
}

int lq_mdi_expabs_partials(lq_ctx* c, int32_t d, const double* beta, const int32_t* counts, double alpha,
                           const double* wn, const double* ww, int32_t n_w, double kappa, int32_t shard,
                           int32_t nshards, double* out_dev) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (d < 1 || !beta || !counts || !wn || !ww || n_w < 1 || !out_dev) return fail(LQ_ERR_VALUE, "bad expabs arguments");
    if (!(kappa < 0.0)) return fail(LQ_ERR_VALUE, "kappa must be negative");
    if (nshards < 1 || shard < 0 || shard >= nshards) return fail(LQ_ERR_VALUE, "bad shard %d of %d", shard, nshards);
    const int32_t k0 = (int32_t)((int64_t)shard * n_w / nshards), k1 = (int32_t)((int64_t)(shard + 1) * n_w / nshards);
    CK(cudaMemsetAsync(out_dev, 0, sizeof(double) * 2 * n_w, c->stream));
    return expabs_nodes(c, d, beta, counts, alpha, wn, ww, n_w, kappa, k0, k1, out_dev, out_dev + n_w);
}

// MDI level collapse for G(alpha + <beta, y>) (lq.h): the distribution of the
// partial linear form level by level, then G over its support.
int lq_mdi_linform(lq_ctx* c, const lq_program* G, int32_t n_levels, const int64_t* m, const int32_t* counts,
                   double alpha, double h, int64_t m0, int32_t shard, int32_t nshards, double* tiles_dev,
                   int64_t tiles_cap, double* out) {
    return lq_mdi_linform_w(c, G, n_levels, m, counts, nullptr, alpha, h, m0, shard, nshards, tiles_dev, tiles_cap,
                            out);
}

int lq_mdi_linform_w(lq_ctx* c, const lq_program* G, int32_t n_levels, const int64_t* m, const int32_t* counts,
                     const double* weights, double alpha, double h, int64_t m0, int32_t shard, int32_t nshards,
                     double* tiles_dev, int64_t tiles_cap, double* out) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (!G || !G->insn || G->n_insn < 1) return fail(LQ_ERR_VALUE, "null program");
    if (G->n_vars > 1) return fail(LQ_ERR_VALUE, "G must be univariate (variable 0), uses %d", G->n_vars);
    if (n_levels < 0 || (n_levels > 0 && (!m || !counts))) return fail(LQ_ERR_VALUE, "bad levels");
    if (nshards < 1 || shard < 0 || shard >= nshards) return fail(LQ_ERR_VALUE, "bad shard %d of %d", shard, nshards);
    if (!out) return fail(LQ_ERR_VALUE, "null output");
    if (!tiles_dev && nshards != 1) return fail(LQ_ERR_VALUE, "sharded calls need tiles_dev");
    const int ns = pick_slots(G->n_slots);
    if (ns < 0) return fail(LQ_ERR_UNSUPPORTED, "program needs %d slots (max %d)", G->n_slots, LQ_MAX_SLOTS);
    std::vector<lq::LinLevel> lv;
    int64_t K = 1, wtotal = 0;
    for (int l = 0; l < n_levels; ++l) {
        if (m[l] < 1 || counts[l] < 1)
            return fail(LQ_ERR_VALUE, "level %d: m = %lld, N = %d", l, (long long)m[l], counts[l]);
        if (m[l] > LQ_LINFORM_MAX_SUPPORT / counts[l]) return fail(LQ_ERR_UNSUPPORTED, "level %d step too large", l);
        K += m[l] * (counts[l] - 1);
        if (K > LQ_LINFORM_MAX_SUPPORT) return fail(LQ_ERR_UNSUPPORTED, "support exceeds %lld points", (long long)LQ_LINFORM_MAX_SUPPORT);
        lv.push_back({m[l], counts[l], 0, weights ? wtotal : -1});
        wtotal += counts[l];
    }
    if (std::fabs((double)m0) + 2.0 * (double)K > 9007199254740992.0)
        return fail(LQ_ERR_UNSUPPORTED, "support positions exceed 2^53");
    const int64_t T = (K + LQ_TILE - 1) / LQ_TILE;
    if (tiles_dev && tiles_cap < T)
        return fail(LQ_ERR_VALUE, "tiles_dev holds %lld tiles, need %lld", (long long)tiles_cap, (long long)T);
    void *dlv = nullptr, *dp, *dq = nullptr, *dg, *dw = nullptr;
    if (!lv.empty() && (rc = upload(c, B_AUX0, lv.data(), sizeof(lq::LinLevel) * lv.size(), &dlv))) return rc;
    if (weights && wtotal > 0 && (rc = upload(c, B_AUX3, weights, sizeof(double) * wtotal, &dw))) return rc;
    if ((rc = upload(c, B_PROG, G->insn, sizeof(lq_insn) * G->n_insn, &dg))) return rc;
    if ((rc = dev_buf(c, B_AUX1, sizeof(double) * K, &dp))) return rc;
    constexpr int64_t kSmemCap = (200 * 1024) / (2 * (int64_t)sizeof(double));   // 12800 support points
    const char* force_global = std::getenv("LQ_LINFORM_SMEM");   // "0": global-memory levels (tests)
    t_begin(c);
    if (K <= kSmemCap && !(force_global && !std::strcmp(force_global, "0"))) {
        if ((rc = smem_optin(c, (const void*)lq::k_linform_smem, 2 * sizeof(double) * kSmemCap))) return rc;
        lq::k_linform_smem<<<1, 1024, 2 * sizeof(double) * K, c->stream>>>((const lq::LinLevel*)dlv, n_levels, K,
                                                                           (const double*)dw, (double*)dp);
        c->launches++;
        CK(cudaGetLastError());
    } else {
        if ((rc = dev_buf(c, B_AUX2, sizeof(double) * K, &dq))) return rc;
        // ping-pong between dp and dq so that the last level lands in dp
        double* cur = (double*)(n_levels % 2 ? dq : dp);
        double* nxt = (double*)(n_levels % 2 ? dp : dq);
        lq::k_fill<<<1, 32, 0, c->stream>>>(cur, 1, 1.0);
        c->launches++;
        int64_t k_old = 1;
        for (int l = 0; l < n_levels; ++l) {
            const int64_t kn = k_old + lv[l].m * (lv[l].n - 1);
            const int grid = (int)std::min<int64_t>((kn + lq::kThreads - 1) / lq::kThreads, (int64_t)c->sm_count * 8);
            const double* w = lv[l].woff >= 0 ? (const double*)dw + lv[l].woff : nullptr;
            lq::k_linform_level<<<grid, lq::kThreads, 0, c->stream>>>(cur, k_old, lv[l].m, lv[l].n, w, nxt);
            c->launches++;
            CK(cudaGetLastError());
            std::swap(cur, nxt);
            k_old = kn;
        }
    }
    // tile partials: this shard's tiles [t0, t1) of the fixed tiling of the support
    const int64_t t0 = (int64_t)shard * T / nshards, t1 = (int64_t)(shard + 1) * T / nshards;
    void* tiles = tiles_dev;
    if (!tiles) {
        if ((rc = dev_buf(c, B_TILES, sizeof(double) * T, &tiles))) return rc;
    } else {
        CK(cudaMemsetAsync(tiles, 0, sizeof(double) * T, c->stream));
    }
    if (t1 > t0) {
        const int grid = (int)std::min<int64_t>(t1 - t0, (int64_t)c->sm_count * 4);
        if (ns == 32)
            lq::k_linform_eval<32><<<grid, lq::kThreads, 0, c->stream>>>(
                (const lq_insn*)dg, G->n_insn, G->result, (const double*)dp, K, alpha, h, (double)m0, t0, t1, 0,
                (double*)tiles);
        else
            lq::k_linform_eval<LQ_MAX_SLOTS><<<grid, lq::kThreads, 0, c->stream>>>(
                (const lq_insn*)dg, G->n_insn, G->result, (const double*)dp, K, alpha, h, (double)m0, t0, t1, 0,
                (double*)tiles);
        c->launches++;
        CK(cudaGetLastError());
    }
    t_end(c);
    if (tiles_dev) {
        *out = (double)T;
        return LQ_OK;
    }
    double* r;
    if ((rc = reduce_dev(c, (const double*)tiles, T, &r))) return rc;
    return read_scalar(c, r, out);
}

int lq_mdi_linform2(lq_ctx* c, const lq_program* G, int32_t n_levels, const int64_t* m1, const int64_t* m2,
                    const int32_t* counts, double h1, int64_t m01, double h2, int64_t m02, int32_t shard,
                    int32_t nshards, double* tiles_dev, int64_t tiles_cap, double* out) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (!G || !G->insn || G->n_insn < 1) return fail(LQ_ERR_VALUE, "null program");
    if (G->n_vars > 2) return fail(LQ_ERR_VALUE, "G must use variables 0 and 1 only, uses %d", G->n_vars);
    if (n_levels < 1 || !m1 || !m2 || !counts) return fail(LQ_ERR_VALUE, "bad levels");
    if (nshards < 1 || shard < 0 || shard >= nshards) return fail(LQ_ERR_VALUE, "bad shard %d of %d", shard, nshards);
    if (!out) return fail(LQ_ERR_VALUE, "null output");
    if (!tiles_dev && nshards != 1) return fail(LQ_ERR_VALUE, "sharded calls need tiles_dev");
    const int ns = pick_slots(G->n_slots);
    if (ns < 0) return fail(LQ_ERR_UNSUPPORTED, "program needs %d slots (max %d)", G->n_slots, LQ_MAX_SLOTS);
    int64_t K1 = 1, K2 = 1;
    std::vector<lq::Lin2Level> lv;
    for (int l = 0; l < n_levels; ++l) {
        if (counts[l] < 1) return fail(LQ_ERR_VALUE, "level %d: N = %d", l, counts[l]);
        const int64_t a1 = m1[l] < 0 ? -m1[l] : m1[l], a2 = m2[l] < 0 ? -m2[l] : m2[l];
        if (a1 > LQ_LINFORM2_MAX_SUPPORT / counts[l] || a2 > LQ_LINFORM2_MAX_SUPPORT / counts[l])
            return fail(LQ_ERR_UNSUPPORTED, "level %d step too large", l);
        K1 += a1 * (counts[l] - 1);
        K2 += a2 * (counts[l] - 1);
        if (K1 > LQ_LINFORM2_MAX_SUPPORT || K2 > LQ_LINFORM2_MAX_SUPPORT || K1 * K2 > LQ_LINFORM2_MAX_SUPPORT)
            return fail(LQ_ERR_UNSUPPORTED, "joint support exceeds %lld points", (long long)LQ_LINFORM2_MAX_SUPPORT);
        lv.push_back({a1, a2, counts[l], (m1[l] < 0 ? 1 : 0) | (m2[l] < 0 ? 2 : 0)});
    }
    const int64_t K = K1 * K2, T = (K + LQ_TILE - 1) / LQ_TILE;
    if (tiles_dev && tiles_cap < T)
        return fail(LQ_ERR_VALUE, "tiles_dev holds %lld tiles, need %lld", (long long)tiles_cap, (long long)T);
    void *dp, *dq, *dg;
    if ((rc = upload(c, B_PROG, G->insn, sizeof(lq_insn) * G->n_insn, &dg))) return rc;
    if ((rc = dev_buf(c, B_AUX1, sizeof(double) * K, &dp))) return rc;
    if ((rc = dev_buf(c, B_AUX2, sizeof(double) * K, &dq))) return rc;
    double* cur = (double*)(n_levels % 2 ? dq : dp);   // the last level lands in dp
    double* nxt = (double*)(n_levels % 2 ? dp : dq);
    t_begin(c);
    lq::k_fill<<<1, 32, 0, c->stream>>>(cur, 1, 1.0);
    c->launches++;
    int64_t k1 = 1, k2 = 1;
    for (int l = 0; l < n_levels; ++l) {
        const int64_t k1n = k1 + lv[l].m1 * (lv[l].n - 1), k2n = k2 + lv[l].m2 * (lv[l].n - 1);
        const int grid = (int)std::min<int64_t>((k1n * k2n + lq::kThreads - 1) / lq::kThreads, (int64_t)c->sm_count * 8);
        lq::k_linform2_level<<<grid, lq::kThreads, 0, c->stream>>>(cur, k1, k2, lv[l], nxt, k1n, k2n);
        c->launches++;
        CK(cudaGetLastError());
        std::swap(cur, nxt);
        k1 = k1n;
        k2 = k2n;
    }
    const int64_t t0 = (int64_t)shard * T / nshards, t1 = (int64_t)(shard + 1) * T / nshards;
    void* tiles = tiles_dev;
    if (!tiles) {
        if ((rc = dev_buf(c, B_TILES, sizeof(double) * T, &tiles))) return rc;
    } else {
        CK(cudaMemsetAsync(tiles, 0, sizeof(double) * T, c->stream));
    }
    if (t1 > t0) {
        const int grid = (int)std::min<int64_t>(t1 - t0, (int64_t)c->sm_count * 4);
        if (ns == 32)
            lq::k_linform2_eval<32><<<grid, lq::kThreads, 0, c->stream>>>(
                (const lq_insn*)dg, G->n_insn, G->result, (const double*)dp, K1, K2, h1, (double)m01, h2,
                (double)m02, t0, t1, 0, (double*)tiles);
        else
            lq::k_linform2_eval<LQ_MAX_SLOTS><<<grid, lq::kThreads, 0, c->stream>>>(
                (const lq_insn*)dg, G->n_insn, G->result, (const double*)dp, K1, K2, h1, (double)m01, h2,
                (double)m02, t0, t1, 0, (double*)tiles);
        c->launches++;
        CK(cudaGetLastError());
    }
    t_end(c);
    if (tiles_dev) {
        *out = (double)T;
        return LQ_OK;
    }
    double* r;
    if ((rc = reduce_dev(c, (const double*)tiles, T, &r))) return rc;
    return read_scalar(c, r, out);
}

int lq_fp64_peak(lq_ctx* c, int32_t iters, double* tflops, float* ms) {
    int rc = set_dev(c);
    if (rc) return rc;
    if (iters < 1) return fail(LQ_ERR_VALUE, "iters must be positive");
    void* p;
    if ((rc = dev_buf(c, B_OUT, 64, &p))) return rc;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)lq::k_fp64_peak, lq::kThreads, 0);
    const int grid = c->sm_count * std::max(per_sm, 1) * 4;
    lq::k_fp64_peak<<<grid, lq::kThreads, 0, c->stream>>>(std::max(1, iters / 16), 1.0, (double*)p);  // warm-up
    CK(cudaGetLastError());
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, c->stream));
    lq::k_fp64_peak<<<grid, lq::kThreads, 0, c->stream>>>(iters, 1.0, (double*)p);
    CK(cudaEventRecord(b, c->stream));
    CK(cudaEventSynchronize(b));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 2.0 * 8 * 16 * (double)iters * grid * lq::kThreads;
    if (tflops) *tflops = flops / (t * 1e-3) / 1e12;
    if (ms) *ms = t;
    return LQ_OK;
}

}  // extern "C"

#include "lq_quality_api.cuh"   // p_alpha / wce sums, CBC, Korobov search

