/*
 * hodlrgp_b200 — C ABI of the B200-native HODLR maximum-likelihood hot path.
 *
 * Drop-in boundary for the reference C++ API in /root/reference/proj/include/
 * hodlrgp (arXiv 2303.10102). Each entry point names the reference interface
 * it replaces (file:line). Plain pointers and sizes only; matrices are
 * column-major doubles. `loc` selects where X/Y live: HG_HOST (copied in/out
 * inside the call) or HG_DEVICE (device pointers on the context's device).
 *
 * Every call returns an hg_status; hg_last_error() gives the message of the
 * last failure on the calling thread. The C++ layer (include/hodlrgp_b200.hpp)
 * maps the codes back to the reference exception types.
 */
#ifndef HODLRGP_B200_H
#define HODLRGP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HG_OK = 0,
    HG_NOT_SPD = 1,   /* NotPositiveDefinite  (factorization.hpp:14-16) */
    HG_EINVAL = 2,    /* std::invalid_argument (dimension/tree/orientation) */
    HG_ELENGTH = 3,   /* std::length_error    (size guards) */
    HG_ELOGIC = 4,    /* std::logic_error     (lower() on symmetric storage) */
    HG_ENOMEM = 5,
    HG_ECUDA = 6,
    HG_EIO = 7,       /* std::runtime_error of io.cpp (missing/truncated sidecar, bad manifest) */
    HG_EOTHER = 9
} hg_status;

enum { HG_HOST = 0, HG_DEVICE = 1 };
enum { HG_RIGHT = 0, HG_LEFT = 1 }; /* Orientation (factorization.hpp:18-21) */

typedef struct hg_ctx_s* hg_ctx_t;
typedef struct hg_hodlr_s* hg_hodlr_t;
typedef struct hg_factor_s* hg_factor_t;
typedef struct hg_prodrep_s* hg_prodrep_t;
typedef struct hg_oracle_s* hg_oracle_t;
typedef struct hg_build_s* hg_build_t;

/* ---------------------------------------------------------------- context */
const char* hg_last_error(void);
/* One device + one CUDA stream (stream may be NULL: the context creates one). */
hg_status hg_ctx_create(int device, void* stream, hg_ctx_t* out);
hg_status hg_ctx_destroy(hg_ctx_t ctx);
hg_status hg_ctx_synchronize(hg_ctx_t ctx);
/* Number of kernels this context has launched so far. */
uint64_t hg_ctx_launches(hg_ctx_t ctx);
void* hg_ctx_stream(hg_ctx_t ctx);
/* Numerical options of a context (defaults 0):
 *  HG_OPT_PRODUCT_ASSOCIATION — how solve_multiply applies each Woodbury factor
 *    to the running factors. HG_ASSOC_SOLVE (default): rows -= v cap^{-T}(u^T rows),
 *    stable at the condition numbers of BASELINE's configs. HG_ASSOC_REFERENCE:
 *    p = -(cap^{-1} v^T)^T formed first, rows += p (q^T rows), exactly the
 *    association of product_rep.cpp:32-45,74-78 (parity mode).
 *  HG_OPT_COMPRESSION — truncation of the derivative blocks' cores
 *    (LowRankBlock::compressed, hodlr_matrix.cpp:42-66): HG_COMPRESS_PIVOTED_QR
 *    (default, rank-revealing pivoted QR at the same 1e-13 threshold) or
 *    HG_COMPRESS_JACOBI_SVD (singular values, as the reference).
 *  HG_OPT_Q2_BASIS — the derivative build's second basis q2 (sketch.cpp:194-233).
 *    HG_Q2_REORTHOGONALIZED (default): q2 is projected against q once more and
 *    renormalised, so [q | q2] is orthonormal to roundoff; columns kept near
 *    the w2 floor otherwise overlap q and double-count dK q in the committed
 *    derivative block (the error that dominates dK/dtheta at n = 2^20).
 *    HG_Q2_REFERENCE: q2 exactly as the reference forms it (parity mode).
 *  HG_OPT_COMPRESS_AT — when the derivative blocks are truncated
 *    (LowRankBlock::compressed at 1e-13). HG_COMPRESS_AT_LEVEL (default): as
 *    each level is committed, so finer levels peel against the compressed
 *    (rank ~3..8 instead of 2k + w2) panels. HG_COMPRESS_AT_END: after the
 *    last level, as sketch.cpp:331-341 (parity mode).
 *  HG_OPT_SKETCH_RNG — where the SketchPlan's Gaussian samplers come from.
 *    HG_SKETCH_RNG_REFERENCE (default): std::mt19937_64(seed) +
 *    std::normal_distribution<double> on the host in the reference's fill
 *    order (sketch.cpp:10-31), byte-identical to the reference's plan — a
 *    sequential stream (seconds at n = 2^20: 2.7e8 draws). HG_SKETCH_RNG_DEVICE:
 *    a counter-based generator on the device (a hash of (seed, level, row,
 *    column) through Box-Muller), milliseconds; same sparsity pattern, not the
 *    reference's bytes (no parity with a CPU run of the same seed). */
enum { HG_OPT_PRODUCT_ASSOCIATION = 1, HG_OPT_COMPRESSION = 2, HG_OPT_Q2_BASIS = 3, HG_OPT_COMPRESS_AT = 4,
       HG_OPT_SKETCH_RNG = 5 };
enum { HG_ASSOC_SOLVE = 0, HG_ASSOC_REFERENCE = 1 };
enum { HG_COMPRESS_PIVOTED_QR = 0, HG_COMPRESS_JACOBI_SVD = 1 };
enum { HG_Q2_REORTHOGONALIZED = 0, HG_Q2_REFERENCE = 1 };
enum { HG_COMPRESS_AT_LEVEL = 0, HG_COMPRESS_AT_END = 1 };
enum { HG_SKETCH_RNG_REFERENCE = 0, HG_SKETCH_RNG_DEVICE = 1 };
hg_status hg_ctx_set_option(hg_ctx_t ctx, int option, int value);
int hg_ctx_get_option(hg_ctx_t ctx, int option);

/* ----------------------------------------------------- cluster tree (host) */
/* tree_depth — cluster_tree.cpp:34-38 */
int hg_tree_depth(int64_t n, int64_t leaf_min, int64_t leaf_max);
/* ClusterTree(n, tau).level(d) for d = 0..tau, depth-major (lo,hi) pairs —
 * cluster_tree.cpp:10-22. lo_hi holds 2 * (2^(tau+1) - 1) entries. */
hg_status hg_tree_ranges(int64_t n, int tau, int64_t* lo_hi);
/* build_kd_ordering — cluster_tree.cpp:40-90; coords n x d col-major. */
hg_status hg_kd_ordering(int64_t n, int d, const double* coords, int64_t leaf_min, int64_t leaf_max,
                         int64_t* perm, int64_t* inv, int* tau);

/* ------------------------------------------------------------ HodlrMatrix */
/* HodlrMatrix::zero / identity / random_spd / random_symmetric —
 * hodlr_matrix.cpp:68-88,126-172 */
hg_status hg_hodlr_zero(hg_ctx_t ctx, int64_t n, int tau, int symmetric, hg_hodlr_t* out);
hg_status hg_hodlr_identity(hg_ctx_t ctx, int64_t n, int tau, hg_hodlr_t* out);
hg_status hg_hodlr_random(hg_ctx_t ctx, int64_t n, int tau, int64_t k, uint64_t seed, int spd, hg_hodlr_t* out);
/* Panel exchange format: for l = 1..tau, U_l then V_l (n x R[l-1] each,
 * col-major; U rows of left children = upper.left, of right children =
 * lower.left; V rows of right children = upper.right, of left children =
 * lower.right), then leaves m_b x m_b concatenated. ranks_* hold 2^tau - 1
 * entries (level-major, node order). Host pointers. */
hg_status hg_hodlr_import(hg_ctx_t ctx, int64_t n, int tau, int symmetric, const int* R, const double* flat,
                          const int* ranks_up, const int* ranks_lo, hg_hodlr_t* out);
hg_status hg_hodlr_info(hg_hodlr_t h, int64_t* n, int* tau, int* symmetric, int* R);
int64_t hg_hodlr_export_size(hg_hodlr_t h);
hg_status hg_hodlr_export(hg_ctx_t ctx, hg_hodlr_t h, double* flat, int* ranks_up, int* ranks_lo);
/* write_hodlr_debug / read_hodlr_debug — io.hpp:33-36, io.cpp:171-275. JSON
 * manifest `dir/name.json` (n, depth, symmetric, per-level upper[/lower]
 * blocks with node, rows, cols, rank, left/right sidecar names; leaves with
 * index, rows, file) + row-major little-endian float64 sidecars. The writer
 * creates `dir`; the reader rebuilds the matrix on the context's device.
 * Manifest ranges must match ClusterTree(n, depth) (HG_EINVAL); missing or
 * short files give HG_EIO. */
hg_status hg_write_hodlr_debug(hg_ctx_t ctx, const char* dir, const char* name, hg_hodlr_t h);
hg_status hg_read_hodlr_debug(hg_ctx_t ctx, const char* dir, const char* name, hg_hodlr_t* out);
hg_status hg_hodlr_copy(hg_ctx_t ctx, hg_hodlr_t h, hg_hodlr_t* out);
hg_status hg_hodlr_free(hg_hodlr_t h);
/* make_asymmetric — hodlr_matrix.cpp:187-196 */
hg_status hg_hodlr_make_asymmetric(hg_ctx_t ctx, hg_hodlr_t h);
/* Y = H X, X/Y n x s (ldx/ldy >= n) — HodlrMatrix::matvec, hodlr_matrix.cpp:198-226 */
hg_status hg_hodlr_matvec(hg_ctx_t ctx, hg_hodlr_t h, const double* X, int64_t ldx, int64_t s, double* Y,
                          int64_t ldy, int loc);
/* Y = H_sub X (or H_sub^T X) for the depth-d node `node` — sub_matvec,
 * hodlr_matrix.cpp:228-265. X/Y have the node's row count. */
hg_status hg_hodlr_sub_matvec(hg_ctx_t ctx, hg_hodlr_t h, int d, int64_t node, const double* X, int64_t ldx,
                              int64_t s, int transpose, double* Y, int64_t ldy, int loc);
/* trace — hodlr_matrix.cpp:267-271; trace_product — :294-318 */
hg_status hg_hodlr_trace(hg_ctx_t ctx, hg_hodlr_t h, double* out);
hg_status hg_trace_product(hg_ctx_t ctx, hg_hodlr_t a, hg_hodlr_t b, double* out);

/* ---------------------------------------------------------- factorization */
/* factorize — factorization.cpp:62-168 */
hg_status hg_factorize(hg_ctx_t ctx, hg_hodlr_t h, int orientation, hg_factor_t* out);
hg_status hg_factor_free(hg_factor_t f);
/* HodlrFactorization::solve — factorization.cpp:170-212 (in-place allowed on HG_DEVICE) */
hg_status hg_factor_solve(hg_ctx_t ctx, hg_factor_t f, const double* B, int64_t ldb, int64_t s, double* X,
                          int64_t ldx, int loc);
/* HodlrFactorization::logdet — factorization.cpp:214-224 (HG_NOT_SPD on a
 * non-positive capacitance or leaf determinant) */
hg_status hg_factor_logdet(hg_ctx_t ctx, hg_factor_t f, double* out);
/* Leaf decisions: 1 = LLT used, 0 = LU fallback (factorization.cpp:7-18). */
hg_status hg_factor_leaf_llt(hg_ctx_t ctx, hg_factor_t f, int* out);

/* ---------------------------------------------------------- trace algebra */
/* multiply / solve_multiply — product_rep.cpp:180-186 (pipeline :47-155) */
hg_status hg_multiply(hg_ctx_t ctx, hg_factor_t f, hg_hodlr_t b, hg_prodrep_t* out);
hg_status hg_solve_multiply(hg_ctx_t ctx, hg_factor_t f, hg_hodlr_t b, hg_prodrep_t* out);
hg_status hg_prodrep_free(hg_prodrep_t p);
/* ProductRep::densify — product_rep.cpp:9-22 (n <= 2^14; host output n x n) */
hg_status hg_prodrep_densify(hg_ctx_t ctx, hg_prodrep_t p, double* out);
/* trace_product_rep :188-194, trace_pair :204-235, trace_solve :196-202,
 * trace_quad :237-245 */
hg_status hg_trace_product_rep(hg_ctx_t ctx, hg_prodrep_t p, double* out);
hg_status hg_trace_pair(hg_ctx_t ctx, hg_prodrep_t p, hg_prodrep_t q, double* out);
hg_status hg_trace_solve(hg_ctx_t ctx, hg_factor_t f, hg_hodlr_t b, double* out);
hg_status hg_trace_quad(hg_ctx_t ctx, hg_factor_t fa, hg_hodlr_t b, hg_factor_t fc, hg_hodlr_t d, double* out);
/* hutchinson_trace — mle.cpp:56-75: stochastic cross-check of tr(K^-1 B) with
 * n_samples >= 2 Rademacher probes (HG_EINVAL below 2), generated on the host
 * with std::mt19937_64(seed) + std::bernoulli_distribution(0.5) in the
 * reference's order; probes are applied 64 at a time (B Z, then the solve). */
hg_status hg_hutchinson_trace(hg_ctx_t ctx, hg_factor_t f, hg_hodlr_t b, int n_samples, uint64_t seed,
                              double* estimate, double* std_error);

/* ------------------------------------------------------ covariance oracle */
/* CovarianceOracle (oracle.hpp:15-52) implemented on the device.
 * hg_oracle_dense: DenseMatrixOracle (oracle.hpp:115-143), K and p derivative
 *   matrices n x n, host pointers (copied to the device).
 * hg_oracle_matern: 1D Matérn nu = nu2/2 on sorted points, theta = (sigma2,
 *   ell) plus a fixed nugget; scan = 1 uses the O(n) exponential-polynomial
 *   recurrence, 0 the dense on-the-fly kernel.
 * hg_oracle_callback: user forward model; fn(user, j, V, ldv, s, Y, ldy,
 *   stream) writes Y = K V (j = -1) or dK/dtheta_j V with device pointers. */
typedef int (*hg_apply_fn)(void* user, int j, const double* V, int64_t ldv, int64_t s, double* Y, int64_t ldy,
                           void* stream);
hg_status hg_oracle_dense(hg_ctx_t ctx, int64_t n, const double* K, int p, const double* dK, hg_oracle_t* out);
hg_status hg_oracle_matern(hg_ctx_t ctx, int64_t n, const double* x, int nu2, double sigma2, double ell,
                           double nugget, int scan, hg_oracle_t* out);
hg_status hg_oracle_callback(hg_ctx_t ctx, int64_t n, int p, hg_apply_fn fn, void* user, hg_oracle_t* out);
/* Forward-model oracles of BASELINE.json configs 2, 3, 5 (the
 * reference's own models are FEM and out of scope). theta = (sigma2, ell, kappa).
 * hg_oracle_cokriging: joint [u; f] of -u'' + kappa^2 u = f (FD, Dirichlet) on
 *   m interior points of [0,1], f Matérn nu = 1/2; n = 2m, rows interleaved
 *   (2i = u_i, 2i+1 = f_i); nugget added on the diagonal (FP64 needs one: the
 *   joint covariance's condition number exceeds 1e15 without).
 * hg_oracle_spde2d: u = (-Lap_h + kappa^2)^-1 f on the nside x nside periodic
 *   grid, f Matérn nu = 3/2 (spectral), plus a fixed nugget (u alone is
 *   singular in FP64); n = nside^2; order[i] = grid index iy*nside + ix of
 *   row i (NULL = natural order), e.g. a KD ordering. */
hg_status hg_oracle_cokriging(hg_ctx_t ctx, int64_t m, double sigma2, double ell, double kappa, double nugget,
                              hg_oracle_t* out);
hg_status hg_oracle_spde2d(hg_ctx_t ctx, int nside, double sigma2, double ell, double kappa, double nugget,
                           const int64_t* order, hg_oracle_t* out);
/* PermutedOracle (oracle.hpp:58-111): the view K'(i,j) = K(p_i, p_j) of any
 * oracle under to_base[reordered position] = base index (host array, copied).
 * The base must outlive the view; applies advance both oracles' counters. */
hg_status hg_oracle_permuted(hg_ctx_t ctx, hg_oracle_t base, const int64_t* to_base, hg_oracle_t* out);
hg_status hg_oracle_set_parameters(hg_oracle_t o, const double* theta, int p);
hg_status hg_oracle_free(hg_oracle_t o);
/* apply (j = -1) / apply_derivative (j >= 0) — oracle.hpp:25-35 */
hg_status hg_oracle_apply(hg_ctx_t ctx, hg_oracle_t o, int j, const double* V, int64_t ldv, int64_t s, double* Y,
                          int64_t ldy, int loc);
/* apply_columns / derivative_columns / reset_counters — oracle.hpp:37-42 */
hg_status hg_oracle_counters(hg_oracle_t o, uint64_t* apply_columns, uint64_t* derivative_columns, int reset);

/* ------------------------------------------------------------ sketch build */
/* build_hodlr / build_hodlr_with_derivatives with SketchPlan(tree, k, seed)
 * generated on the host by std::mt19937_64 + std::normal_distribution in the
 * reference's fill order — sketch.cpp:10-31, 128-356. */
/* SketchPlan sampler bytes (sketch.cpp:10-31): level 0 = the leaf sampler
 * (n x max_leaf_size stacked identities), level l in [1, tau] = the n x k
 * Gaussian sampler of level l; generated on the host with the reference's
 * mt19937_64 / normal_distribution fill order, cached on the device. */
hg_status hg_sketch_sampler(hg_ctx_t ctx, int64_t n, int tau, int64_t k, uint64_t seed, int level, double* out,
                            int64_t ldo, int loc);
/* randomized_range(y, k) (sketch.cpp:37-76): rows x k block y -> q (rows x k,
 * orthonormal), r (k x k upper, diag >= 0, host), perm (k, host; y.col(perm[i])
 * -> position i), numeric rank (#|r_ii| > 64 eps |r_00|); deficient columns
 * completed with unit vectors orthogonalised twice. k <= 128. */
hg_status hg_randomized_range(hg_ctx_t ctx, const double* y, int64_t ldy, int64_t rows, int64_t k, double* q,
                              int64_t ldq, double* r, int* perm, int64_t* numeric_rank, int loc);
/* diff_qr(b, db, q, r) (sketch.cpp:78-111): derivative of b = q r under db ->
 * dq, dq_span = q dOmega (rows x k), dr (k x k, host), ill-conditioned flag
 * (max/min |r_ii| > 1e12). b itself is not needed (as in the reference). */
hg_status hg_diff_qr(hg_ctx_t ctx, const double* db, int64_t lddb, const double* q, int64_t ldq, const double* r,
                     int64_t rows, int64_t k, double* dq, int64_t lddq, double* dq_span, int64_t ldds, double* dr,
                     int* ill_conditioned, int loc);
hg_status hg_build(hg_ctx_t ctx, hg_oracle_t o, int tau, int64_t k, uint64_t seed, int with_derivatives,
                   hg_build_t* out);
hg_status hg_build_free(hg_build_t b);
/* BuildResult::h / deriv[j] (returned handles are owned by the caller) */
hg_status hg_build_h(hg_build_t b, hg_hodlr_t* out);
hg_status hg_build_deriv(hg_build_t b, int j, hg_hodlr_t* out);
int hg_build_num_warnings(hg_build_t b);
/* Rank decisions per (level, node): numeric_rank, w2, rw[0..p) — logged for
 * comparison with the CPU path (sketch.cpp:54-59, 214-221, 249-252). */
int hg_build_decisions(hg_build_t b, int p, int64_t* out);

/* -------------------------------------------------------------------- mle */
/* log_likelihood / score / fisher_information — mle.cpp:25-54. y, ybar are
 * host vectors of length n (ybar may be NULL). Fisher uses the p cached
 * ProductReps (identical arithmetic to recomputing them per pair). */
hg_status hg_log_likelihood(hg_ctx_t ctx, hg_factor_t f, const double* y, const double* ybar, double* out);
hg_status hg_score(hg_ctx_t ctx, hg_factor_t f, const hg_hodlr_t* deriv, int p, const double* y,
                   const double* ybar, double* out);
hg_status hg_fisher_information(hg_ctx_t ctx, hg_factor_t f, const hg_hodlr_t* deriv, int p, double* out);
/* One MLE iteration (acceptance.cpp:297-308): build with derivatives,
 * factorize (Left), log-likelihood, score, Fisher. times[5] = build_deriv,
 * factorize, loglik, score, fisher seconds (device events). */
hg_status hg_mle_iteration(hg_ctx_t ctx, hg_oracle_t o, int tau, int64_t k, uint64_t seed, const double* y,
                           double* loglik, double* score, double* fisher, double* times);
/* The same iteration plus the solve of nrhs right-hand sides B (n x nrhs) into
 * X, with y/B/X at `loc` (HG_HOST: copied in/out inside the call; HG_DEVICE:
 * device pointers). times[5] = build_deriv, factorize, loglik+solves, score,
 * fisher seconds (device events). */
/* fit_mle (mle.cpp:188-322; FitOptions{max_iter, rel_tol, dense}):
 * BFGS on transformed parameters (transforms[i]: 0 positive theta = exp(u),
 * 1 correlation theta = tanh(u), 2 unbounded) with a backtracking line
 * search; every evaluation is a device build + factorization with the
 * SketchPlan of `seed` fixed for the whole fit (dense != 0: the exact dense
 * device evaluation of mle.cpp:131-169 instead). Outputs FitReport: theta_hat
 * (p), fisher (p x p, NaN if not SPD), ci (p x 2: lo, hi), status ("converged",
 * "max_iter", "line_search_failed", "not_positive_definite[_at_start]"),
 * traces (up to trace_cap iterations; theta_trace p x cap), columns[2] =
 * oracle apply / derivative columns, seconds. ybar may be NULL (zero mean). */
hg_status hg_fit_mle(hg_ctx_t ctx, hg_oracle_t o, int tau, int64_t k, uint64_t seed, const double* y,
                     const double* ybar, int p, const int* transforms, const double* theta0, int max_iter,
                     double rel_tol, int dense, double* theta_hat, double* fisher, double* ci, int* ci_valid, int* iterations,
                     int* converged, char* status, int status_len, double* loglik_trace, double* grad_norm_trace,
                     double* theta_trace, int trace_cap, int* trace_len, uint64_t* columns, double* seconds);
/* dense_exact — mle.cpp:345-380 (n <= 2^13, HG_ELENGTH above): exact dense
 * log-likelihood, score and Fisher (p x p column-major) of the oracle at its
 * current parameters; y, ybar host (ybar may be NULL). */
hg_status hg_dense_exact(hg_ctx_t ctx, hg_oracle_t o, const double* y, const double* ybar, double* loglik,
                         double* score, double* fisher);
/* accuracy_metrics — mle.cpp:382-403: out = {eps_L, eps_S, eps_I, eta_g, eta_I};
 * HG_EINVAL when the exact Fisher matrix is not SPD. Host arithmetic. */
hg_status hg_accuracy_metrics(int p, double loglik, const double* score_exact, const double* fisher_exact,
                              double loglik_approx, const double* score_approx, const double* fisher_approx,
                              double* out);
hg_status hg_mle_evaluate(hg_ctx_t ctx, hg_oracle_t o, int tau, int64_t k, uint64_t seed, const double* y,
                          const double* B, int64_t nrhs, double* X, int loc, double* loglik, double* score,
                          double* fisher, double* times);

/* ------------------------------------ strong admissibility
 * Not in the reference (weak HODLR only): an eta-admissible
 * H-matrix over the KD block-cluster tree of the nside x nside periodic grid
 * (BASELINE.json configs 3 and 5). order[i] = grid index of row i (a KD
 * order, e.g. build_kd_ordering of the grid); the cluster tree is the uniform
 * ClusterTree(nside^2, tau) over it. A pair of one depth is admissible when
 * min(diam) <= eta * dist on the torus and both sides exceed k rows: rank-k
 * block U V^T; inadmissible leaf pairs are dense; symmetric (t <= s stored).
 * hg_hstrong_plan: host only, the block counts and storage of that tree.
 * hg_hstrong_build: the oracle must be translation invariant on the grid (it
 *   is probed with two unit vectors; HG_EINVAL otherwise), param = -1 -> K,
 *   j -> dK/dtheta_j; blocks compressed by a batched randomized range finder
 *   (width k, power_iters subspace iterations, Gaussian sketch from seed) on
 *   entries generated from the probed column (matrix-free).
 * hg_hstrong_trace_product: tr(A B) of two symmetric matrices of one plan. */
typedef struct hg_hstrong_s* hg_hstrong_t;
hg_status hg_hstrong_plan(const int64_t* order, int nside, int tau, double eta, int64_t k, int64_t* n_lowrank,
                          int64_t* n_dense, int64_t* lowrank_entries, int64_t* dense_entries, int64_t* stored_doubles);
hg_status hg_hstrong_build(hg_ctx_t ctx, hg_oracle_t o, int param, const int64_t* order, int nside, int tau,
                           double eta, int64_t k, int power_iters, uint64_t seed, hg_hstrong_t* out);
hg_status hg_hstrong_free(hg_hstrong_t h);
hg_status hg_hstrong_matvec(hg_ctx_t ctx, hg_hstrong_t h, const double* X, int64_t ldx, int64_t s, double* Y,
                            int64_t ldy, int loc);
hg_status hg_hstrong_trace_product(hg_ctx_t ctx, hg_hstrong_t a, hg_hstrong_t b, double* out);
hg_status hg_hstrong_blocks(hg_hstrong_t h, int64_t* n_lowrank, int64_t* n_dense, int64_t* bytes);

/* ---------------------------------------------------- kernel-level ledger */
/* Per kernel class (seg_tn, seg_nn, leaf_mm, leaf_solve, leaf_factor, cap_lu,
 * cap_solve, qr, form_q, oracle, reduce, other, hmatvec): device ms from CUDA events
 * around each launch, algorithmic flops and bytes, launch count. Off by
 * default; returns the number of classes written (<= 13). */
void hg_prof_enable(int on);
int hg_prof_read(int reset, double* ms, double* flops, double* bytes, int64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* HODLRGP_B200_H */
