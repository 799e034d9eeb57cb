/*
 * liblq — B200-native (sm_100a) rank-1 lattice sums and MDI-LR cluster sums.
 *
 * The drop-in boundary of the hot path of latquad (arXiv 2404.08867's
 * reference package).  The reference has no FFI of its own: its boundary is
 * the Python callables listed in SURVEY.md §8(b).  Each entry point below
 * names the reference function whose inner loop it replaces
 * (paths relative to /root/reference/pkg/src/latquad/).  The Python mirror
 * (paper_2404_08867_b200/{lattice,quad,mdi}.py) binds these with ctypes;
 * INTEGRATION.md shows the binding a latquad maintainer would add.
 *
 * Conventions
 *  - Every function returns int status: LQ_OK or a negative LQ_ERR_* code;
 *    lq_last_error() (thread-local) describes the last failure.  The Python
 *    layer maps LQ_ERR_VALUE -> ValueError, LQ_ERR_OVERFLOW -> OverflowError,
 *    LQ_ERR_GRIDCAP -> GridCapError, the rest -> RuntimeError, matching the
 *    reference's exceptions (lattice.py:65-70, 99-100; mdi.py:44-45, 112-113).
 *  - Host pointers are caller-owned; "_dev" pointers are device pointers
 *    (e.g. torch tensors' data_ptr()).  Device scratch is owned by the lq_ctx.
 *  - All work is ordered on the context's stream (lq_ctx_set_stream); calls
 *    that return values to host pointers synchronise that stream.
 *  - Reductions are deterministic: fixed tiles of points, a fixed
 *    in-tile tree, fixed super-chunks of LQ_SUPER_TILES tiles and a fixed
 *    pairwise tree over super-chunk partials, independent of grid size and of
 *    how super-chunks are split across GPUs.
 */
#ifndef LQ_H
#define LQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LQ_ABI_VERSION 11

#define LQ_OK 0
#define LQ_ERR_VALUE (-1)
#define LQ_ERR_OVERFLOW (-2)
#define LQ_ERR_GRIDCAP (-3)
#define LQ_ERR_CUDA (-4)
#define LQ_ERR_UNSUPPORTED (-5)
#define LQ_ERR_NOMEM (-6)

#define LQ_TILE 4096          /* flat grid nodes per tile (tensor sums); points per
                                 tile of the bytecode lattice kernel; the family
                                 kernels use 6144-point tiles (lq_lattice_layout) */
#define LQ_SUPER_TILES 1024   /* tiles per super-chunk                          */
#define LQ_NODE_BLOCK 256     /* MDI nodes per deterministic partial block     */
#define LQ_MAX_SLOTS 512      /* bytecode live-slot limit                      */

typedef struct lq_ctx lq_ctx;
typedef struct lq_jit lq_jit;   /* an NVRTC-compiled integrand module (lq_jit_create) */

/* Bytecode instruction; slot[a] <- op(...).  Ops (see lower.py):
 * 0 CONST c | 1 VAR x[b] | 2 ACC_INIT c | 3 ACC_ADD += c*slot[b] |
 * 4 ACC_MUL *= slot[b] | 5 POW slot[b]^n | 6 RPOW 1/slot[b]^n | 7 EXP |
 * 8 SIN | 9 COS | 10 ABS (of slot[b]) | 11 ACC_ADDVAR += c*x[b]          */
typedef struct {
    int32_t op, a, b, n;
    double c;
} lq_insn;

typedef struct {
    const lq_insn* insn;   /* host array of n_insn instructions */
    int32_t n_insn;
    int32_t n_slots;
    int32_t result;        /* slot holding the value */
    int32_t n_vars;        /* variables referenced: 0..n_vars-1 */
    lq_jit* jit;           /* optional: compiled straight-line version (NULL: interpret) */
} lq_program;

enum {
    LQ_FAM_PROGRAM = 0,     /* generic bytecode (any expression)               */
    LQ_FAM_LIN_EXP = 1,     /* K exp(alpha + <beta,x>)                         */
    LQ_FAM_LIN_SINCOS = 2,  /* C0 + A sin(<beta,x>) + B cos(<beta,x>)          */
    LQ_FAM_LIN_EXPABS = 3,  /* K exp(kappa |alpha + <beta,x>|)                 */
    LQ_FAM_QUAD_EXP = 4,    /* K exp(alpha + sum_j beta_j x_j + gamma_j x_j^2) */
    LQ_FAM_LIN_POW = 5,     /* K (alpha + <beta,x>)^power, integer power       */
    LQ_FAM_QUAD_SINCOS = 6, /* C0 + A sin(Q) + B cos(Q), Q = sum_j beta_j x_j + gamma_j x_j^2 */
    LQ_FAM_PROD_QUAD = 7,   /* K prod_j ((x_j - beta_j)^2 + gamma_j)^power; gamma_j = NaN: no factor */
    LQ_FAM_LIN_PROG = 8     /* G(<beta,x>), G any one-variable program (outer); prog = the whole
                               expression (per-index kernels), outer = G (FFT-form chains)  */
};

typedef struct {
    int32_t kind;
    int32_t d;
    const double* beta;     /* [d], host (LIN_*, QUAD_*) */
    const double* gamma;    /* [d], host (QUAD_*)        */
    double alpha, K, A, B, C0, kappa;
    double power;           /* LIN_POW: integer-valued exponent */
    lq_program prog;        /* LQ_FAM_PROGRAM, LQ_FAM_LIN_PROG: the whole expression */
    lq_program outer;       /* LQ_FAM_LIN_PROG: G of one variable (variable 0 = <beta,x>) */
} lq_integrand;

/* ---- context ----------------------------------------------------------
 * Plumbing with no reference counterpart: latquad is single-process numpy
 * (quad.py:96-131 runs its loops on the host); a context holds what those
 * loops keep implicitly -- the device, a stream, scratch and cached plans.  */
int lq_ctx_create(int device, lq_ctx** out);
int lq_ctx_destroy(lq_ctx* ctx);
/* Order all work on this cudaStream_t (NULL: the context's own stream). */
int lq_ctx_set_stream(lq_ctx* ctx, void* stream);
int lq_sync(lq_ctx* ctx);
const char* lq_last_error(void);
int lq_abi_version(void);
int lq_device_info(lq_ctx* ctx, int* sm_count, int* cc_major, int* cc_minor);
/* Device time (ms) of the main kernel of the last timed call (0 if none). */
int lq_ctx_enable_timing(lq_ctx* ctx, int enable);
int lq_last_kernel_ms(lq_ctx* ctx, float* ms, int64_t* launches);
/* Cumulative bytes this context moved host->device and device->host with
 * cudaMemcpy*, and the kernel-parameter bytes of its FFT-form lattice-sum
 * launches (the e2e accounting of bench.py reads the difference per step). */
int lq_ctx_transfer_bytes(lq_ctx* ctx, int64_t* h2d, int64_t* d2h, int64_t* params);

/* ---- points: replaces lattice.points_block (lattice.py:96-105) ---------
 * out[(i-start)*d + j] = RN(((i * z_reduced[j]) mod n) / n), i in [start, stop),
 * bit-identical to the reference (int64 modmul + IEEE division).
 * n > 2^53 -> LQ_ERR_OVERFLOW (lattice.py:99-100).                          */
int lq_points_block(lq_ctx* ctx, int32_t d, uint64_t n, const uint64_t* z_reduced,
                    int64_t start, int64_t stop, double* out, int32_t out_is_device);

/* ---- plain lattice sum: replaces the block loop of quad.slr_integrate ----
 * (quad.py:96-104 -> lattice.iter_point_blocks + exprcore.eval_array + np.sum).
 * Returns sum_{i in [i_begin, i_end)} f(frac(i z / n)) (not divided by n).
 * A full range [0, n) uses the fastest exact enumeration lq_lattice_layout
 * reports (Korobov chains in direct or FFT form, 2^k unit-group levels,
 * mirror pairs, index tiles); sub-ranges use index tiles.  The choice is a
 * function of (f, n, z) only; LQ_ORBIT=0, LQ_FFT=0|always, LQ_PAIR=0 in the
 * environment override it (tests, comparisons).                             */
int lq_lattice_sum(lq_ctx* ctx, const lq_integrand* f, uint64_t n, const uint64_t* z_reduced,
                   uint64_t i_begin, uint64_t i_end, double* sum_out);
/* Multi-GPU building blocks.  A full-lattice sum is split into units: points
 * i in [0, n) for the per-index kernels (mode LQ_LAYOUT_INDEX), or -- for a
 * Korobov rule z_j = a^(j-1) over a prime n (mode LQ_LAYOUT_ORBIT) -- chains
 * of consecutive powers i0 a^k whose points are summed together with their
 * mirrors n - i, or -- when every z_j is a unit mod n
 * (mode LQ_LAYOUT_PAIRED) -- mirror-pair indices i in [0, n/2], point i
 * summed with point n - i.  Units form tiles of tile_units, tiles form
 * super-chunks of super_tiles tiles (LQ_SUPER_TILES; 256 for the FFT-form
 * layouts, whose tiles are heavy); super-chunk s covers units
 * [s*T*S, (s+1)*T*S), T = tile_units, S = super_tiles.  The layout depends on
 * (f, n, z) only, so every rank computes the same one; z may be NULL (index
 * layout).  lq_lattice_partials writes the partials of super-chunks
 * [s_begin, s_end) to out_dev[0 .. s_end-s_begin).  lq_lattice_sum over the
 * full range [0, n) uses the same layout.  (Replaces the chunk loop of
 * quad.slr_integrate, quad.py:96-104, for sharded runs.)                   */
#define LQ_LAYOUT_INDEX 0
#define LQ_LAYOUT_ORBIT 1
#define LQ_LAYOUT_PAIRED 2   /* units: mirror-pair indices i in [0, n/2] (points i and n - i) */
#define LQ_LAYOUT_ORBIT_FFT 3 /* units: Korobov chains of 4097 - d points, two per FFT tile */
#define LQ_LAYOUT_ORBIT_POW2 4 /* n = 2^k Korobov: units are tiles (levels of chains + the 2^m0 lattice) */
int lq_lattice_layout(const lq_integrand* f, uint64_t n, const uint64_t* z_reduced, int64_t* tile_units,
                      int64_t* n_supers, int64_t* n_units, int32_t* mode, int64_t* super_tiles);
int lq_lattice_partials(lq_ctx* ctx, const lq_integrand* f, uint64_t n, const uint64_t* z_reduced,
                        int64_t s_begin, int64_t s_end, double* out_dev);
/* Fixed pairwise tree over vals_dev[0..count); result to host *out. */
/* ---- MDI-LR level collapse for G(alpha1 + <beta1, y>, alpha2 + <beta2, y>):
 * two commensurate forms (exprcore.py:139-169 collects the partial sums with
 * equal pairs).  Level l moves the joint distribution of
 * k = (sum |m1_l| t, sum |m2_l| t) by node t (t -> N-1-t for a negative step),
 * on a K1 x K2 grid (K1 K2 <= LQ_LINFORM2_MAX_SUPPORT); then
 * sum_k p(k) G(h1 (m01 + 2 k1), h2 (m02 + 2 k2)) over fixed tiles of LQ_TILE
 * entries.  G: program of variables 0 and 1.  Sharding and outputs as
 * lq_mdi_linform.                                                             */
#define LQ_LINFORM2_MAX_SUPPORT (((int64_t)1) << 25)
int lq_mdi_linform2(lq_ctx* ctx, const lq_program* G, int32_t n_levels, const int64_t* m1, const int64_t* m2,
                    const int32_t* counts, double h1, int64_t m01, double h2, int64_t m02, int32_t shard,
                    int32_t nshards, double* tiles_dev, int64_t tiles_cap, double* out);

/* Host-only check of the full-lattice layout of (f, n, z) (n <= 2^26): how
 * many lattice indices the layout's units (chains and their mirrors, levels,
 * the small lattice, mirror pairs or plain indices) miss and how many they
 * cover more than once -- both 0 for a correct plan.                        */
int lq_layout_cover(const lq_integrand* f, uint64_t n, const uint64_t* z_reduced, int64_t* missed,
                    int64_t* repeated);
int lq_reduce_sum(lq_ctx* ctx, const double* vals_dev, int64_t count, double* out);

/* ---- Monte Carlo: replaces quad.mc_integrate's loop (quad.py:79-93).  Sums
 * f over points [i_begin, i_end) of numpy's default_rng(seed).random((n, d))
 * stream, reproduced bit for bit on the device: PCG64 state/increment as
 * (lo, hi) words of bit_generator.state after seeding (host bookkeeping).   */
int lq_mc_sum(lq_ctx* ctx, const lq_program* prog, int32_t d, uint64_t n, const uint64_t* state,
              const uint64_t* inc, uint64_t i_begin, uint64_t i_end, double* sum_out);

/* ---- direct tensor-grid sum: replaces mdi._numeric_sum / direct_tensor_sum
 * (mdi.py:104-136) for implr_integrate and the MDI fallback.  Flat index s
 * decodes first axis fastest.  nodes: concatenated per-axis node values
 * (host), or NULL with midpoint=1 for nodes RN((t+0.5)/counts[k])
 * (transform.py:169-178).  Sums flat indices [s_begin, s_end).              */
int lq_tensor_sum(lq_ctx* ctx, const lq_program* prog, int32_t d, const int64_t* counts,
                  const double* nodes, int32_t midpoint, uint64_t s_begin, uint64_t s_end,
                  double* sum_out);
/* Sharded form: partials of tiles [t_begin, t_end) of the fixed tiling of
 * [0, total) (LQ_TILE nodes per tile) into tiles_dev[t_begin .. t_end) (device);
 * lq_reduce_sum over all ceil(total / LQ_TILE) tiles equals lq_tensor_sum over
 * [0, total) bit for bit.  (mdi.py:104-136 sharded by flat index.) */
int lq_tensor_partials(lq_ctx* ctx, const lq_program* prog, int32_t d, const int64_t* counts,
                       const double* nodes, int32_t midpoint, uint64_t total, int64_t t_begin,
                       int64_t t_end, double* tiles_dev);

/* ---- element-wise evaluation: replaces exprcore.eval_array
 * (exprcore.py:442-480) on m rows, out[i] = f(x_1[i], ..., x_V[i]) in the
 * reference's evaluation order (the bytecode of lower.compile_program).
 * cols[b] holds the m values of variable b (b < prog->n_vars; NULL for a
 * variable the program never reads).  The table cols is host memory; the
 * columns and out are host memory, or device memory when on_device != 0.     */
int lq_eval_array(lq_ctx* ctx, const lq_program* prog, const double* const* cols, int64_t m,
                  int32_t on_device, double* out);

/* ---- MDI-LR cluster sums: replaces the symbolic level loop of
 * mdi.mdi_sum (mdi.py:139-192) for separable integrands.  Factor f is a
 * univariate U_f(y) = R_f(y) exp(i P_f(y)) on an axis with count_f midpoint
 * nodes y_t = RN((t+0.5)/count_f); S_f = sum_t U_f(y_t).                     */
typedef struct {
    int32_t count;          /* nodes on the factor's axis              */
    int32_t r_off, r_len;   /* program R in the insn table (len 0: R=1) */
    int32_t r_result;
    int32_t p_off, p_len;   /* program P (len 0: P=0)                   */
    int32_t p_result;
    int32_t n_slots;
    int32_t node_off;       /* < 0: midpoint nodes RN((t+0.5)/count); else
                               nodes[node_off + t] of the nodes table      */
    int32_t reserved;       /* 0, or LQ_FACTOR_SUPPLIED: a core factor of
                               several axes whose cluster sum the caller
                               supplies as (re, im) = nodes[node_off], nodes[node_off+1]
                               (count must be 1)                           */
} lq_factor;
#define LQ_FACTOR_SUPPLIED 1

/* Partial cluster sums of LQ_NODE_BLOCK-node blocks: part_dev[(f*nblk + b)*2 + {0,1}]
 * (re, im) for node blocks b of every factor with b*nshards/... owned by
 * shard `shard` of `nshards` (blocks [floor(shard*NB_f/nshards),
 * floor((shard+1)*NB_f/nshards)); others left untouched).  nblk = max_f NB_f. */
int lq_mdi_block_sums(lq_ctx* ctx, const lq_insn* insn, int32_t n_insn, const lq_factor* factors,
                      int32_t n_factors, const double* nodes, int64_t n_nodes, int32_t shard,
                      int32_t nshards, double* part_dev);
/* Combine: S_f = fixed tree over blocks; term t = coef_t * prod_{f in term t} S_f
 * * exp(log_extra_t), evaluated in log-polar form (sum log|S|, sum arg S).
 * term_ptr[n_terms+1] indexes term_fac (replaces the level loop's folded
 * coefficients, mdi.py:152-165, and the base sweep, mdi.py:166-179).
 * out[0]=log|raw|, out[1]=sign(Re raw)
 * (0 if raw == 0), out[2]=Re raw as a double (may under/overflow), out[3]=Im raw. */
int lq_mdi_combine(lq_ctx* ctx, const double* part_dev, const lq_factor* factors, int32_t n_factors, int32_t nblk,
                   const int32_t* term_ptr, const int32_t* term_fac, const double* coef_re,
                   const double* coef_im, const double* log_extra, int32_t n_terms,
                   double* out4);
/* Single-GPU convenience: block sums + combine -- the whole of mdi_sum
 * (mdi.py:139-192) for a separable integrand.                               */
int lq_mdi_sum(lq_ctx* ctx, const lq_insn* insn, int32_t n_insn, const lq_factor* factors,
               int32_t n_factors, const double* nodes, int64_t n_nodes, const int32_t* term_ptr, const int32_t* term_fac,
               const double* coef_re, const double* coef_im, const double* log_extra,
               int32_t n_terms, double* out4);

/* ---- characteristic-function MDI for K exp(kappa |alpha + <beta,y>|),
 * kappa < 0 (BASELINE config 5; the reference cannot express |.|, so this is
 * an extension of mdi_sum, mdi.py:139-192):  sum_grid = K prod_j N_j (|kappa|/pi) int_R Re[e^{i w alpha}
 * prod_j phi_j(w)] / (kappa^2 + w^2) dw,  phi_j(w) = (1/N_j) sum_t e^{i w beta_j y_t}.
 * w_nodes/w_weights: host quadrature on [0, W] (even integrand, factor 2
 * applied by the caller).  out2[0] = log|sum_k w_k |kappa|/(kappa^2+w_k^2)
 * Re[e^{i w_k alpha} prod_j phi_j(w_k)]|, out2[1] = its sign.                  */
int lq_mdi_expabs(lq_ctx* ctx, int32_t d, const double* beta, const int32_t* counts, double alpha,
                  const double* w_nodes, const double* w_weights, int32_t n_w, double kappa,
                  double* out2, double* logmag_out /* optional [n_w]: log|prod_j phi_j(w_k)| */);
/* Sharded form: frequency nodes [floor(shard n_w / nshards), floor((shard+1) n_w / nshards))
 * write their terms to out_dev[k] and log|prod_j phi_j(w_k)| to out_dev[n_w + k]
 * (device, 2 n_w doubles, zero elsewhere); lq_reduce_sum of out_dev[0 .. n_w)
 * after the exchange is the single-GPU sum bit for bit.                      */
int lq_mdi_expabs_partials(lq_ctx* ctx, int32_t d, const double* beta, const int32_t* counts, double alpha,
                           const double* w_nodes, const double* w_weights, int32_t n_w, double kappa,
                           int32_t shard, int32_t nshards, double* out_dev);

/* ---- MDI-LR level collapse for f = G(alpha + <beta, y>): replaces the level
 * loop of mdi.mdi_sum (mdi.py:152-165) for integrands whose coordinates enter
 * through one linear form with commensurate steps, where the reference's
 * partial_sum + like-term collection (exprcore.py:139-169, 374-402) merges
 * the partial sums with equal constants level by level (corpus invpow).
 * Direction l (levels with m_l != 0 only) contributes |m_l| t, t uniform on
 * [0, counts[l]); the engine convolves the distribution of
 * k = sum_l |m_l| t_l level by level (shared memory up to 12800 support
 * points, global memory up to LQ_LINFORM_MAX_SUPPORT) and sums
 * p(k) G(alpha + h (m0 + 2k)) over fixed tiles of LQ_TILE support points.
 * G: one-variable program (variable 0).
 * tiles_dev == NULL: out[0] = grid mean (shard 0 of 1).
 * tiles_dev != NULL: tiles_dev[0 .. T) = tile partials of this shard's tiles
 * [floor(shard T / nshards), floor((shard+1) T / nshards)), zero elsewhere;
 * out[0] = T = ceil(K / LQ_TILE), K = 1 + sum_l |m_l| (counts[l] - 1);
 * the mean is lq_reduce_sum of the (all-reduced) tile vector.              */
#define LQ_LINFORM_MAX_SUPPORT (((int64_t)1) << 28)
int lq_mdi_linform(lq_ctx* ctx, const lq_program* G, int32_t n_levels, const int64_t* m, const int32_t* counts,
                   double alpha, double h, int64_t m0, int32_t shard, int32_t nshards, double* tiles_dev,
                   int64_t tiles_cap, double* out);
/* Weighted form (f = G(alpha + <beta, y>) prod_j phi_j(y_j)): level l's
 * distribution update is p'(k) = (1/N_l) sum_t w_(l,t) p(k - |m_l| t), with
 * weights[] the levels' node weights concatenated in level order (N_l each,
 * in the order of the level's t; NULL: uniform, = lq_mdi_linform).          */
int lq_mdi_linform_w(lq_ctx* ctx, const lq_program* G, int32_t n_levels, const int64_t* m, const int32_t* counts,
                     const double* weights, double alpha, double h, int64_t m0, int32_t shard, int32_t nshards,
                     double* tiles_dev, int64_t tiles_cap, double* out);

/* ---- lattice quality measures and constructions (
 * lattice.py:140-311).  B_alpha and the factors 1 + g_j (B + beta) follow
 * numpy's operation order.  n <= 2^31.                                       */
/* sum over i in [i_begin, i_end) of prod_j (1 + g_j (B_alpha(x_ij) + beta)):
 * shift_avg_wce_sq (g = weights, beta = anchor constant) and p_alpha
 * (g = sign (2 pi)^alpha / alpha!, beta = 0).                               */
int lq_bprod_sum(lq_ctx* ctx, int32_t alpha, int32_t d, uint64_t n, const uint64_t* z_reduced,
                 const double* g, double beta, uint64_t i_begin, uint64_t i_end, double* sum_out);
/* cbc_construct (lattice.py:259-289): z_1 = 1, then for each s the candidate
 * minimising the shift-averaged worst-case error, ties to the earliest
 * (strict improvement with 1e-9 relative head-room, lattice.py:248-252).    */
int lq_cbc_construct(lq_ctx* ctx, uint64_t n, int32_t d, const double* gamma, double beta,
                     const int64_t* candidates, int64_t n_candidates, int64_t* z_out);
/* korobov_search building block (lattice.py:292-311): for each candidate a,
 * sum_k prod_j (1 + gamma_j (B_2(x_kj) + beta)) over the Korobov rule
 * z = (1, a, ..., a^(d-1)).                                                 */
int lq_korobov_values(lq_ctx* ctx, uint64_t n, int32_t d, const double* gamma, double beta,
                      const int64_t* candidates, int64_t n_candidates, double* sums_out);

/* ---- JIT: the lowering step before the path ------
 * Compile CUDA source that defines extern "C" kernels lq_jit_lattice and/or
 * lq_jit_tensor (generated from an expression by paper_2404_08867_b200/jit.py)
 * with NVRTC for sm_100a (replaces eval_array inside the sums,
 * exprcore.py:442-480).  Attach the handle to lq_program.jit: lattice and
 * tensor sums then launch the compiled kernel instead of the interpreter,
 * with the same tiles and reduction tree.  NVRTC is loaded with dlopen.     */
int lq_jit_create(const char* source, const char* name, lq_jit** out, char* log, int64_t log_cap);
int lq_jit_destroy(lq_jit* jit);

/* ---- FP64 roofline probe: DFMA chains on every SM; returns TFLOP/s -----
 * (measurement only; bench.py's roofline denominator, no reference twin) */
int lq_fp64_peak(lq_ctx* ctx, int32_t iters, double* tflops, float* ms);

#ifdef __cplusplus
}
#endif
#endif /* LQ_H */
