// TEST INFRASTRUCTURE ONLY — parity oracle for the B200 HODLR-MLE hot path.
//
// A CPU restatement of the reference C++ library `hodlrgp`
// (/root/reference/proj, arXiv 2303.10102) restricted to the hot path:
//   cluster_tree.cpp, hodlr_matrix.cpp, sketch.cpp, factorization.cpp,
//   product_rep.cpp, mle.cpp:25-54 and oracle.hpp.
// The reference cannot be compiled here (Eigen, doctest, CLI11 and
// nlohmann-json are absent), so this file restates its
// algorithms line by line on a small column-major matrix type and a set of
// self-written dense kernels that follow Eigen 3.4's algorithms
// (ColPivHouseholderQR, HouseholderQR, LLT, PartialPivLU; JacobiSVD is
// restated as one-sided Jacobi, whose singular triplets agree to roundoff).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// call into this code, and only as the checker. The product path
// (paper_2303_10102_b200/) never links it.
#pragma once

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

using Index = std::int64_t;

// ---------------------------------------------------------------- matrices
/// Column-major dense matrix (stands in for Eigen::MatrixXd).
struct Mat {
    Index r = 0, c = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(Index rows, Index cols) : r(rows), c(cols), a(size_t(rows * cols), 0.0) {}
    double& operator()(Index i, Index j) { return a[size_t(i + j * r)]; }
    double operator()(Index i, Index j) const { return a[size_t(i + j * r)]; }
    double* data() { return a.data(); }
    const double* data() const { return a.data(); }
    double* col(Index j) { return a.data() + j * r; }
    const double* col(Index j) const { return a.data() + j * r; }
    Index rows() const { return r; }
    Index cols() const { return c; }
    bool empty() const { return c == 0; }
    static Mat zeros(Index rows, Index cols) { return Mat(rows, cols); }
    static Mat identity(Index rows, Index cols);
    Mat block(Index i0, Index j0, Index nr, Index nc) const;
    void set_block(Index i0, Index j0, const Mat& b);
    void add_block(Index i0, Index j0, const Mat& b, double s = 1.0);
    Mat middle_rows(Index i0, Index nr) const { return block(i0, 0, nr, c); }
    Mat left_cols(Index nc) const { return block(0, 0, r, nc); }
    Mat transpose() const;
    double norm() const;  // Frobenius
    double trace() const;
};

Mat operator+(const Mat& x, const Mat& y);
Mat operator-(const Mat& x, const Mat& y);
Mat operator*(double s, const Mat& x);
/// Plain product x * y.
Mat matmul(const Mat& x, const Mat& y);
/// op(x) * op(y) with transposition flags.
Mat matmul_t(const Mat& x, bool tx, const Mat& y, bool ty);
/// C = alpha op(A) op(B) + beta C on raw column-major storage.
void gemm(bool ta, bool tb, Index m, Index n, Index k, double alpha, const double* A, Index lda,
          const double* B, Index ldb, double beta, double* C, Index ldc);
double dot_sum(const Mat& x, const Mat& y);  // sum(x .* y)
/// Pairwise-summed dot product with strides.
double pdot(const double* a, const double* b, Index n, Index sa, Index sb);

/// Use an external BLAS dgemm (scipy's bundled OpenBLAS) for large GEMMs
/// when available; only affects the CPU timing baseline, never semantics.
bool enable_external_blas(const char* path, int threads);
const char* blas_backend();

// ----------------------------------------------------------- dense kernels
/// Eigen 3.4 ColPivHouseholderQR restated (max-norm pivot, first index on
/// ties, LAPACK xGEQPF norm downdating at sqrt(eps)).
struct ColPivQR {
    Mat qr;                      // R in the upper triangle, essentials below
    std::vector<double> hcoeffs; // tau_k
    std::vector<int> transpositions;
    std::vector<int> perm;       // indices(): column perm[i] of input -> position i
    void compute(const Mat& y);
    Mat householder_q_thin(Index ncols) const;  // Q * I(m, ncols)
    Mat matrix_r() const;                       // full upper-triangular R (min(m,n) x n)
};

/// Eigen HouseholderQR (unpivoted) restated.
struct HouseholderQR {
    Mat qr;
    std::vector<double> hcoeffs;
    void compute(const Mat& y);
    Mat householder_q_thin(Index ncols) const;
};

/// Eigen JacobiSVD(ComputeThinU|ComputeThinV) restated as one-sided Jacobi.
/// Singular values sorted non-increasing.
struct ThinSVD {
    Mat u, v;
    std::vector<double> s;
    void compute(const Mat& a);
};

/// Eigen LLT (lower triangle read only).
struct LLT {
    Mat l;
    bool ok = false;
    void compute(const Mat& a);
    Mat solve(const Mat& b) const;
};

/// Eigen PartialPivLU (first max-abs pivot).
struct PartialPivLU {
    Mat lu;
    std::vector<int> perm;   // row i of P*A = row perm[i] of A
    int transpositions_parity = 0;
    void compute(const Mat& a);
    Mat solve(const Mat& b) const;
    Mat solve_transpose(const Mat& b) const;  // A^{-T} b
    double det_p() const { return transpositions_parity ? -1.0 : 1.0; }
};

// ------------------------------------------------------------ cluster tree
/// cluster_tree.hpp:24-51, cluster_tree.cpp:10-32
class ClusterTree {
public:
    struct Range {
        Index lo = 0, hi = 0;
        Index size() const { return hi - lo; }
    };
    ClusterTree() = default;
    ClusterTree(Index n, int tau);
    Index size() const { return n_; }
    int depth() const { return tau_; }
    const std::vector<Range>& level(int d) const { return levels_[size_t(d)]; }
    const std::vector<Range>& leaves() const { return levels_[size_t(tau_)]; }
    Index num_leaves() const { return Index(levels_[size_t(tau_)].size()); }
    Index max_leaf_size() const;
    bool same_structure(const ClusterTree& o) const { return n_ == o.n_ && tau_ == o.tau_; }

private:
    Index n_ = 0;
    int tau_ = 0;
    std::vector<std::vector<Range>> levels_;
};

/// cluster_tree.cpp:34-38
int tree_depth(Index n, Index leaf_min, Index leaf_max);

struct KdOrdering {
    std::vector<Index> perm, inv;
    ClusterTree tree;
    Mat reordered_coords;
};
/// cluster_tree.cpp:40-90 (coords n x d, d in {1,2})
KdOrdering build_kd_ordering(const Mat& coords, Index leaf_min, Index leaf_max);

// ----------------------------------------------------------- HODLR matrix
/// hodlr_matrix.hpp:20-40, hodlr_matrix.cpp:17-66
struct LowRankBlock {
    Mat left, right;
    Index rank() const { return left.c; }
    bool empty() const { return left.c == 0; }
    Mat dense() const { return matmul_t(left, false, right, true); }
    void apply(const Mat& x, Index xr0, Mat& y, Index yr0) const;            // y += L R^T x
    void apply_transpose(const Mat& x, Index xr0, Mat& y, Index yr0) const;  // y += R L^T x
    static LowRankBlock concat(const LowRankBlock& a, const LowRankBlock& b);
    LowRankBlock compressed(double rtol) const;
};

/// hodlr_matrix.hpp:48-106
class HodlrMatrix {
public:
    HodlrMatrix() = default;
    static HodlrMatrix zero(const ClusterTree& tree, bool symmetric = true);
    static HodlrMatrix identity(const ClusterTree& tree);
    static HodlrMatrix from_dense(const ClusterTree& tree, const Mat& a, bool symmetric);
    static HodlrMatrix random_spd(const ClusterTree& tree, Index k, std::uint64_t seed);
    static HodlrMatrix random_symmetric(const ClusterTree& tree, Index k, std::uint64_t seed);

    const ClusterTree& tree() const { return tree_; }
    Index size() const { return tree_.size(); }
    int depth() const { return tree_.depth(); }
    bool symmetric() const { return symmetric_; }
    LowRankBlock& upper(int l, Index j) { return upper_[size_t(l - 1)][size_t(j)]; }
    const LowRankBlock& upper(int l, Index j) const { return upper_[size_t(l - 1)][size_t(j)]; }
    LowRankBlock lower_block(int l, Index j) const;
    LowRankBlock& lower(int l, Index j);
    Mat& leaf(Index i) { return leaves_[size_t(i)]; }
    const Mat& leaf(Index i) const { return leaves_[size_t(i)]; }
    Index num_leaves() const { return Index(leaves_.size()); }
    void make_asymmetric();

    Mat matvec(const Mat& x) const;
    Mat sub_matvec(int d, Index node, const Mat& x, bool transpose = false) const;
    double trace() const;
    Mat densify() const;
    static double trace_product(const HodlrMatrix& a, const HodlrMatrix& b);

private:
    ClusterTree tree_;
    bool symmetric_ = true;
    std::vector<std::vector<LowRankBlock>> upper_, lower_;
    std::vector<Mat> leaves_;
};

// --------------------------------------------------------- covariance oracle
/// oracle.hpp:15-52 — matrix-free K(theta) with counted applies.
class CovarianceOracle {
public:
    virtual ~CovarianceOracle() = default;
    virtual Index dim() const = 0;
    virtual Index num_params() const = 0;
    Mat apply(const Mat& v) const {
        apply_columns_ += std::uint64_t(v.c);
        return do_apply(v);
    }
    Mat apply_derivative(int j, const Mat& v) const {
        derivative_columns_ += std::uint64_t(v.c);
        return do_apply_derivative(j, v);
    }
    std::uint64_t apply_columns() const { return apply_columns_.load(); }
    std::uint64_t derivative_columns() const { return derivative_columns_.load(); }
    void reset_counters() const {
        apply_columns_ = 0;
        derivative_columns_ = 0;
    }

protected:
    virtual Mat do_apply(const Mat& v) const = 0;
    virtual Mat do_apply_derivative(int j, const Mat& v) const = 0;

private:
    mutable std::atomic<std::uint64_t> apply_columns_{0}, derivative_columns_{0};
};

/// oracle.hpp:115-143
class DenseMatrixOracle : public CovarianceOracle {
public:
    DenseMatrixOracle(Mat k, std::vector<Mat> dk = {}) : k_(std::move(k)), dk_(std::move(dk)) {}
    Index dim() const override { return k_.r; }
    Index num_params() const override { return Index(dk_.size()); }
    const Mat& dense() const { return k_; }
    const Mat& dense_derivative(int j) const { return dk_[size_t(j)]; }

protected:
    Mat do_apply(const Mat& v) const override { return matmul(k_, v); }
    Mat do_apply_derivative(int j, const Mat& v) const override {
        if (dk_.empty()) return Mat(v.r, v.c);
        return matmul(dk_[size_t(j)], v);
    }

private:
    Mat k_;
    std::vector<Mat> dk_;
};

/// 1D Matérn covariance on sorted points (BASELINE.json configs C1, C4):
///   k(d) = sigma2 * p_nu(a) * exp(-a), a = c_nu d / ell,
///   p_{1/2} = 1, p_{3/2} = 1 + a, p_{5/2} = 1 + a + a^2/3,
/// plus nugget * I; parameters theta = (sigma2, ell). Derivatives:
///   dk/dsigma2 = k_noiseless / sigma2,
///   dk/dell    = sigma2 * q_nu(a) * exp(-a) / ell with
///   q_{1/2} = a, q_{3/2} = a^2, q_{5/2} = a^2 (1 + a) / 3.
/// Both forms (dense O(n^2) per column and the O(n) exponential-polynomial
/// two-sided scan) are provided; the product implements the same formulas
/// on the GPU. The reference's forward models (FEM/SPDE) are not used by
/// any BASELINE.json config.
class Matern1dOracle : public CovarianceOracle {
public:
    /// nu2 = 2*nu in {1, 3, 5}; scan = use the O(n) recurrence.
    Matern1dOracle(std::vector<double> x, int nu2, double sigma2, double ell, double nugget,
                   bool scan);
    Index dim() const override { return Index(x_.size()); }
    Index num_params() const override { return 2; }
    void set_parameters(double sigma2, double ell) { sigma2_ = sigma2; ell_ = ell; }
    double kernel(double d, int which) const;  // which: -1 value (no nugget), 0, 1 derivs

protected:
    Mat do_apply(const Mat& v) const override { return apply_impl(-1, v); }
    Mat do_apply_derivative(int j, const Mat& v) const override { return apply_impl(j, v); }

private:
    Mat apply_impl(int which, const Mat& v) const;
    std::vector<double> x_;
    int nu2_;
    double sigma2_, ell_, nugget_;
    bool scan_;
};

// ------------------------------------------------------------------ sketch
/// sketch.hpp:17-40, sketch.cpp:10-35
class SketchPlan {
public:
    SketchPlan() = default;
    SketchPlan(const ClusterTree& tree, Index k, std::uint64_t seed);
    Index rank() const { return k_; }
    bool dimensioned_for(const ClusterTree& tree, Index k) const {
        return n_ == tree.size() && tau_ == tree.depth() && k_ == k;
    }
    const Mat& level_sampler(int l) const { return level_samplers_[size_t(l - 1)]; }
    const Mat& leaf_sampler() const { return leaf_sampler_; }

private:
    Index k_ = 0, n_ = 0;
    int tau_ = 0;
    std::vector<Mat> level_samplers_;
    Mat leaf_sampler_;
};

struct RangeResult {
    Mat q, r;
    std::vector<int> perm;
    Index numeric_rank = 0;
};
/// sketch.cpp:37-76
RangeResult randomized_range(const Mat& y, Index k);

struct DiffQrResult {
    Mat dq, dq_span, dr;
    bool ill_conditioned = false;
};
/// sketch.cpp:78-111
DiffQrResult diff_qr(const Mat& b, const Mat& db, const Mat& q, const Mat& r);

/// Rank decisions taken by the build (logged for CPU/GPU comparison).
struct BuildDecision {
    int level;
    Index node;
    Index numeric_rank;   // randomized_range (sketch.cpp:54-59)
    Index w2;             // q2 width (sketch.cpp:214-221)
    std::vector<Index> rw;  // per param (sketch.cpp:249-252)
};

struct BuildResult {
    HodlrMatrix h;
    std::vector<HodlrMatrix> deriv;
    std::vector<std::string> warnings;
    std::vector<BuildDecision> decisions;
};
/// sketch.cpp:347-356 (build_impl :128-343)
HodlrMatrix build_hodlr(const CovarianceOracle& oracle, const ClusterTree& tree, Index k,
                        const SketchPlan& plan);
BuildResult build_hodlr_with_derivatives(const CovarianceOracle& oracle, const ClusterTree& tree,
                                         Index k, const SketchPlan& plan);
BuildResult build_impl(const CovarianceOracle& oracle, const ClusterTree& tree, Index k,
                       const SketchPlan& plan, bool with_deriv);

// ----------------------------------------------------------- factorization
struct NotPositiveDefinite : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum class Orientation { Right, Left };

/// factorization.hpp:25-38, factorization.cpp:7-44
class LeafFactor {
public:
    void compute(const Mat& a, bool prefer_llt);
    Mat solve(const Mat& b) const;
    Mat multiply(const Mat& b) const { return matmul(mat_, b); }
    double logdet_positive() const;
    bool uses_llt() const { return use_llt_; }

private:
    Mat mat_;
    bool use_llt_ = false;
    LLT llt_;
    PartialPivLU lu_;
};

/// factorization.hpp:45-78
class HodlrFactorization {
public:
    struct LevelBlock {
        Mat u, v;
        PartialPivLU cap;
        double logdet_cap = 0.0;
        bool cap_positive = true;
    };
    const ClusterTree& tree() const { return tree_; }
    Orientation orientation() const { return orient_; }
    int depth() const { return int(levels_.size()); }
    Index size() const { return tree_.size(); }
    const std::vector<LevelBlock>& level(int i) const { return levels_[size_t(i - 1)]; }
    const LeafFactor& leaf(Index b) const { return leaf_factors_[size_t(b)]; }
    Index num_leaves() const { return Index(leaf_factors_.size()); }
    Mat solve(const Mat& b) const;
    double logdet() const;
    friend HodlrFactorization factorize(const HodlrMatrix& h, Orientation orient);

private:
    ClusterTree tree_;
    Orientation orient_ = Orientation::Right;
    std::vector<LeafFactor> leaf_factors_;
    std::vector<std::vector<LevelBlock>> levels_;
};

/// factorization.cpp:62-168
HodlrFactorization factorize(const HodlrMatrix& h, Orientation orient = Orientation::Right);

// ------------------------------------------------------------ trace algebra
/// product_rep.hpp:14-26
struct ProductRep {
    struct CorrBlock {
        Mat u, v;
    };
    HodlrMatrix base;
    std::vector<std::vector<CorrBlock>> corrections;
    Index size() const { return base.size(); }
    Mat densify() const;
};
/// Diagnostic switch (default off = the reference's association,
/// product_rep.cpp:74-78 + :32-45: p = -(cap^{-1} v^T)^T precomputed, then
/// rows += p (q^T rows)). On: rows -= v cap^{-T} (u^T rows) via the LU solve,
/// the association the device path uses; identical in exact arithmetic but
/// it avoids forming p when the capacitance is ill-conditioned.
void set_solve_association(bool on);
/// Diagnostic switch (default off = the reference, sketch.cpp:194-233). On:
/// each q2 is projected against q once more and its columns renormalised,
/// the device's default HG_Q2_REORTHOGONALIZED.
void set_q2_reorthogonalize(bool on);
/// Diagnostic switch (default off = the reference, sketch.cpp:331-341: every
/// derivative block compressed after the last level). On: each level's
/// blocks are compressed when committed, the device's default
/// HG_COMPRESS_AT_LEVEL.
void set_compress_at_level(bool on);
ProductRep multiply(const HodlrFactorization& f, const HodlrMatrix& b);
ProductRep solve_multiply(const HodlrFactorization& f, const HodlrMatrix& b);
double trace_product_rep(const ProductRep& p);
double trace_pair(const ProductRep& p, const ProductRep& q);
double trace_solve(const HodlrFactorization& f_left, const HodlrMatrix& b);
double trace_solve(const HodlrMatrix& a, const HodlrMatrix& b);
double trace_quad(const HodlrFactorization& fa, const HodlrMatrix& b, const HodlrFactorization& fc,
                  const HodlrMatrix& d);
double trace_quad(const HodlrMatrix& a, const HodlrMatrix& b, const HodlrMatrix& c,
                  const HodlrMatrix& d);

// --------------------------------------------------------------- mle glue
/// mle.cpp:56-75: Rademacher-probe estimate of tr(K^-1 B) (mt19937_64 +
/// bernoulli_distribution(0.5), one probe at a time, in the reference's order).
struct HutchinsonResult {
    double estimate = 0;
    double std_error = 0;
};
HutchinsonResult hutchinson_trace(const HodlrFactorization& f, const HodlrMatrix& b, int n_samples,
                                  std::uint64_t seed);
/// mle.cpp:25-54
double log_likelihood(const HodlrFactorization& f, const Mat& y, const Mat& ybar);
std::vector<double> score(const HodlrFactorization& f, const std::vector<HodlrMatrix>& deriv,
                          const Mat& y, const Mat& ybar);
/// fisher_information with the p ProductReps cached (same arithmetic as
/// mle.cpp:43-54, which recomputes solve_multiply per pair).
Mat fisher_information(const HodlrFactorization& f, const std::vector<HodlrMatrix>& deriv,
                       bool cache_reps = false);

// ------------------------------------------------------------ host RNG
/// std::mt19937_64 + std::normal_distribution<double>, row-major fill
/// (the fill order of the reference's test helpers).
Mat randn(Index r, Index c, std::uint64_t seed);

}  // namespace oracle
