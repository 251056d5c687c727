// Matrix-free covariance operators on the device (CovarianceOracle,
// oracle.hpp:15-143): K V and dK/dtheta_j V on column-major device panels,
// with the reference's relaxed-atomic column counters.
#pragma once

#include <atomic>

#include "kernels.cuh"

namespace hg {

class DOracle {
public:
    explicit DOracle(i64 n, int p) : n_(n), p_(p) {}
    virtual ~DOracle() = default;
    i64 dim() const { return n_; }
    int num_params() const { return p_; }
    virtual void set_parameters(const double* theta, int p) { (void)theta, (void)p; }
    /// oracle.hpp:25-35: j = -1 -> K V, j >= 0 -> dK/dtheta_j V.
    void apply(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy) const {
        if (s <= 0) return;
        (j < 0 ? apply_cols_ : deriv_cols_).fetch_add(std::uint64_t(s), std::memory_order_relaxed);
        do_apply(j, V, ldv, s, Y, ldy);
    }
    /// apply under a ZeroRows hint: V is zero on the depth segments of parity
    /// z.parity and, with z.out_depth >= 0, the caller reads Y only on those
    /// rows. Oracles may skip the work this makes dead; default = apply.
    void apply_masked(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy, const ZeroRows& z) const {
        if (s <= 0) return;
        (j < 0 ? apply_cols_ : deriv_cols_).fetch_add(std::uint64_t(s), std::memory_order_relaxed);
        do_apply_masked(j, V, ldv, s, Y, ldy, z);
    }
    /// dK/dtheta_j = a K + b I exactly (e.g. sigma2 of sigma2 C + nugget I):
    /// callers may form that derivative's applies from value applies of the
    /// same columns. Default: no such relation.
    virtual bool affine_derivative(int j, double* a, double* b) const {
        (void)j, (void)a, (void)b;
        return false;
    }
    /// A derivative apply formed that way still counts as one (the column
    /// counters keep the reference's meaning, oracle.hpp:37-45).
    void count_derivative_columns(int s) const { deriv_cols_.fetch_add(std::uint64_t(s), std::memory_order_relaxed); }
    std::uint64_t apply_columns() const { return apply_cols_.load(); }
    std::uint64_t derivative_columns() const { return deriv_cols_.load(); }
    void reset_counters() const {
        apply_cols_ = 0;
        deriv_cols_ = 0;
    }

protected:
    virtual void do_apply(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy) const = 0;
    virtual void do_apply_masked(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy, const ZeroRows&) const {
        do_apply(j, V, ldv, s, Y, ldy);
    }
    i64 n_;
    int p_;

private:
    mutable std::atomic<std::uint64_t> apply_cols_{0}, deriv_cols_{0};
};

/// DenseMatrixOracle (oracle.hpp:115-143), matrices resident on the device.
std::unique_ptr<DOracle> make_dense_oracle(i64 n, const double* K, int p, const double* dK);

/// 1D Matérn nu = nu2/2 on sorted points, theta = (sigma2, ell), fixed nugget.
///   k(d) = sigma2 poly_nu(a) e^{-a}, a = c_nu d / ell (c = 1, sqrt3, sqrt5).
/// scan: O(n) two-sided exponential-polynomial recurrence (chunked 3-phase
/// scan); otherwise the dense kernel evaluated on the fly inside the tiles.
std::unique_ptr<DOracle> make_matern_oracle(i64 n, const double* x, int nu2, double sigma2, double ell,
                                            double nugget, bool scan);

/// BASELINE.json C2: joint [u; f] co-kriging covariance (models.cu), n = 2m,
/// theta = (sigma2, ell, kappa), fixed nugget on the diagonal.
std::unique_ptr<DOracle> make_cokriging_oracle(i64 m, double sigma2, double ell, double kappa, double nugget);

/// BASELINE.json C3/C5: covariance of u = (-Lap_h + kappa^2)^-1 f on the N x N
/// periodic grid (models.cu), n = N^2, theta = (sigma2, ell, kappa); row i of
/// every panel is grid point order[i] (null = natural order).
std::unique_ptr<DOracle> make_spde2d_oracle(int N, double sigma2, double ell, double kappa, double nugget,
                                            const std::int64_t* order);

using ApplyFn = int (*)(void* user, int j, const double* V, std::int64_t ldv, std::int64_t s, double* Y,
                        std::int64_t ldy, void* stream);
std::unique_ptr<DOracle> make_callback_oracle(i64 n, int p, ApplyFn fn, void* user);

/// PermutedOracle (oracle.hpp:58-111) over any device oracle; to_base (host,
/// n entries) maps reordered positions to base indices. base must outlive it.
std::unique_ptr<DOracle> make_permuted_oracle(DOracle* base, const std::int64_t* to_base);

/// Plain C = alpha A B + beta C (A m x k, B k x n), via the segmented engine.
void gemm_nn(i64 m, int n, int k, const double* A, i64 lda, const double* B, i64 ldb, double* C, i64 ldc,
             double alpha, double beta);

}  // namespace hg
