// TEST INFRASTRUCTURE ONLY — dense kernels of the parity oracle.
//
// Restates the Eigen 3.4 algorithms the reference calls on its hot path
// (SURVEY.md §8c "Third-party boundary"): ColPivHouseholderQR
// (sketch.cpp:41,209), HouseholderQR + JacobiSVD (hodlr_matrix.cpp:44-56),
// LLT / PartialPivLU (factorization.hpp:36-37,50), triangular solves
// (sketch.cpp:92,106) and GEMM. Eigen is not present in this image; these
// follow its published algorithms, not its source.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>

#include "oracle.hpp"

namespace oracle {

// ------------------------------------------------------------------- Mat
Mat Mat::identity(Index rows, Index cols) {
    Mat m(rows, cols);
    for (Index i = 0; i < std::min(rows, cols); ++i) m(i, i) = 1.0;
    return m;
}

Mat Mat::block(Index i0, Index j0, Index nr, Index nc) const {
    Mat b(nr, nc);
    for (Index j = 0; j < nc; ++j)
        std::memcpy(b.col(j), col(j0 + j) + i0, static_cast<size_t>(nr) * sizeof(double));
    return b;
}

void Mat::set_block(Index i0, Index j0, const Mat& b) {
    for (Index j = 0; j < b.c; ++j)
        std::memcpy(col(j0 + j) + i0, b.col(j), static_cast<size_t>(b.r) * sizeof(double));
}

void Mat::add_block(Index i0, Index j0, const Mat& b, double s) {
    for (Index j = 0; j < b.c; ++j) {
        double* d = col(j0 + j) + i0;
        const double* src = b.col(j);
        for (Index i = 0; i < b.r; ++i) d[i] += s * src[i];
    }
}

Mat Mat::transpose() const {
    Mat t(c, r);
    for (Index j = 0; j < c; ++j)
        for (Index i = 0; i < r; ++i) t(j, i) = (*this)(i, j);
    return t;
}

double Mat::norm() const { return std::sqrt(pdot(a.data(), a.data(), Index(a.size()), 1, 1)); }

double Mat::trace() const {
    double t = 0;
    for (Index i = 0; i < std::min(r, c); ++i) t += (*this)(i, i);
    return t;
}

Mat operator+(const Mat& x, const Mat& y) {
    Mat z = x;
    for (size_t i = 0; i < z.a.size(); ++i) z.a[i] += y.a[i];
    return z;
}
Mat operator-(const Mat& x, const Mat& y) {
    Mat z = x;
    for (size_t i = 0; i < z.a.size(); ++i) z.a[i] -= y.a[i];
    return z;
}
Mat operator*(double s, const Mat& x) {
    Mat z = x;
    for (double& v : z.a) v *= s;
    return z;
}

double dot_sum(const Mat& x, const Mat& y) { return pdot(x.data(), y.data(), Index(x.a.size()), 1, 1); }

// ------------------------------------------------------------ reductions
/// Pairwise (blocked) dot product: 4 interleaved accumulators on blocks of
/// 64, halves combined recursively — the error behaviour of Eigen's
/// vectorised, cache-blocked reductions rather than a sequential sum.
double pdot(const double* a, const double* b, Index n, Index sa, Index sb) {
    if (n <= 64) {
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
        Index i = 0;
        for (; i + 4 <= n; i += 4) {
            s0 += a[i * sa] * b[i * sb];
            s1 += a[(i + 1) * sa] * b[(i + 1) * sb];
            s2 += a[(i + 2) * sa] * b[(i + 2) * sb];
            s3 += a[(i + 3) * sa] * b[(i + 3) * sb];
        }
        for (; i < n; ++i) s0 += a[i * sa] * b[i * sb];
        return (s0 + s1) + (s2 + s3);
    }
    const Index h = n / 2;
    return pdot(a, b, h, sa, sb) + pdot(a + h * sa, b + h * sb, n - h, sa, sb);
}

// ------------------------------------------------------------------ GEMM
namespace {
using dgemm_fn = void (*)(const char*, const char*, const int*, const int*, const int*,
                          const double*, const double*, const int*, const double*, const int*,
                          const double*, double*, const int*);
dgemm_fn g_dgemm = nullptr;
const char* g_backend = "builtin";
}  // namespace

bool enable_external_blas(const char* path, int threads) {
    if (!path || !*path) {  // back to the built-in loops
        g_dgemm = nullptr;
        g_backend = "builtin";
        return true;
    }
    void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) return false;
    auto f = reinterpret_cast<dgemm_fn>(dlsym(h, "scipy_dgemm_"));
    if (!f) f = reinterpret_cast<dgemm_fn>(dlsym(h, "dgemm_"));
    if (!f) return false;
    using setnt_fn = void (*)(int);
    auto s = reinterpret_cast<setnt_fn>(dlsym(h, "scipy_openblas_set_num_threads"));
    if (!s) s = reinterpret_cast<setnt_fn>(dlsym(h, "openblas_set_num_threads"));
    if (s && threads > 0) s(threads);
    g_dgemm = f;
    g_backend = "openblas";
    return true;
}

const char* blas_backend() { return g_backend; }

void gemm(bool ta, bool tb, Index m, Index n, Index k, double alpha, const double* A, Index lda,
          const double* B, Index ldb, double beta, double* C, Index ldc) {
    if (m == 0 || n == 0) return;
    if (g_dgemm && m * n * k >= 32768 && m < (Index(1) << 31) && n < (Index(1) << 31) &&
        k < (Index(1) << 31)) {
        int im = int(m), in = int(n), ik = int(k), ilda = int(std::max<Index>(lda, 1)),
            ildb = int(std::max<Index>(ldb, 1)), ildc = int(ldc);
        char cta = ta ? 'T' : 'N', ctb = tb ? 'T' : 'N';
        g_dgemm(&cta, &ctb, &im, &in, &ik, &alpha, A, &ilda, B, &ildb, &beta, C, &ildc);
        return;
    }
    // Builtin: C = beta C + alpha op(A) op(B), j-p-i loop order (contiguous i).
    for (Index j = 0; j < n; ++j) {
        double* cj = C + j * ldc;
        if (beta == 0.0)
            for (Index i = 0; i < m; ++i) cj[i] = 0.0;
        else if (beta != 1.0)
            for (Index i = 0; i < m; ++i) cj[i] *= beta;
    }
    if (k == 0) return;
    if (!ta) {
        for (Index j = 0; j < n; ++j) {
            double* cj = C + j * ldc;
            for (Index p = 0; p < k; ++p) {
                double b = alpha * (tb ? B[j + p * ldb] : B[p + j * ldb]);
                if (b == 0.0) continue;
                const double* ap = A + p * lda;
                for (Index i = 0; i < m; ++i) cj[i] += ap[i] * b;
            }
        }
    } else {
        // C(i,j) = sum_p A(p,i) op(B)(p,j): dot products over contiguous p.
        std::vector<double> bcol;
        for (Index j = 0; j < n; ++j) {
            const double* bj;
            if (tb) {
                bcol.resize(static_cast<size_t>(k));
                for (Index p = 0; p < k; ++p) bcol[static_cast<size_t>(p)] = B[j + p * ldb];
                bj = bcol.data();
            } else {
                bj = B + j * ldb;
            }
            double* cj = C + j * ldc;
            for (Index i = 0; i < m; ++i) cj[i] += alpha * pdot(A + i * lda, bj, k, 1, 1);
        }
    }
}

Mat matmul_t(const Mat& x, bool tx, const Mat& y, bool ty) {
    Index m = tx ? x.c : x.r, k = tx ? x.r : x.c, n = ty ? y.r : y.c;
    Index k2 = ty ? y.c : y.r;
    if (k != k2) throw std::invalid_argument("matmul: inner dimension mismatch");
    Mat z(m, n);
    gemm(tx, ty, m, n, k, 1.0, x.data(), x.r, y.data(), y.r, 0.0, z.data(), std::max<Index>(m, 1));
    return z;
}

Mat matmul(const Mat& x, const Mat& y) { return matmul_t(x, false, y, false); }

// ------------------------------------------------------------ Householder
namespace {

double sq_norm(const double* v, Index n) { return pdot(v, v, n, 1, 1); }

/// Eigen MatrixBase::makeHouseholderInPlace on x[0..n): returns tau, beta;
/// essential part overwrites x[1..n).
void make_householder(double* x, Index n, double& tau, double& beta) {
    double tail_sq = n == 1 ? 0.0 : sq_norm(x + 1, n - 1);
    double c0 = x[0];
    const double tol = std::numeric_limits<double>::min();
    if (tail_sq <= tol) {
        tau = 0.0;
        beta = c0;
        for (Index i = 1; i < n; ++i) x[i] = 0.0;
    } else {
        beta = std::sqrt(c0 * c0 + tail_sq);
        if (c0 >= 0.0) beta = -beta;
        for (Index i = 1; i < n; ++i) x[i] = x[i] / (c0 - beta);
        tau = (beta - c0) / beta;
    }
}

/// Eigen applyHouseholderOnTheLeft: block (rows x cols, ld) with v = [1;ess].
void apply_householder_left(double* blk, Index rows, Index cols, Index ld, const double* ess,
                            double tau) {
    if (rows == 1) {
        for (Index j = 0; j < cols; ++j) blk[j * ld] *= (1.0 - tau);
        return;
    }
    if (tau == 0.0) return;
    for (Index j = 0; j < cols; ++j) {
        double* cj = blk + j * ld;
        double t = pdot(ess, cj + 1, rows - 1, 1, 1);
        t += cj[0];
        cj[0] -= tau * t;
        for (Index i = 1; i < rows; ++i) cj[i] -= tau * ess[i - 1] * t;
    }
}

/// Q * I(m, ncols) from compact Householder storage (H_0 ... H_{s-1}).
Mat form_q(const Mat& qr, const std::vector<double>& hcoeffs, Index ncols) {
    const Index m = qr.r;
    const Index s = Index(hcoeffs.size());
    Mat q = Mat::identity(m, ncols);
    for (Index k = s - 1; k >= 0; --k) {
        // apply H_k to rows k..m-1 of q
        apply_householder_left(q.data() + k, m - k, ncols, m, qr.col(k) + k + 1,
                               hcoeffs[static_cast<size_t>(k)]);
    }
    return q;
}

}  // namespace

void ColPivQR::compute(const Mat& y) {
    const Index m = y.r, n = y.c, size = std::min(m, n);
    qr = y;
    hcoeffs.assign(static_cast<size_t>(size), 0.0);
    transpositions.assign(static_cast<size_t>(size), 0);
    std::vector<double> norms_upd(static_cast<size_t>(n)), norms_dir(static_cast<size_t>(n));
    for (Index j = 0; j < n; ++j) norms_dir[static_cast<size_t>(j)] = norms_upd[static_cast<size_t>(j)] = std::sqrt(sq_norm(qr.col(j), m));
    const double downdate_thr = std::sqrt(std::numeric_limits<double>::epsilon());
    for (Index k = 0; k < size; ++k) {
        Index best = k;
        double bv = norms_upd[static_cast<size_t>(k)];
        for (Index j = k + 1; j < n; ++j)
            if (norms_upd[static_cast<size_t>(j)] > bv) {
                bv = norms_upd[static_cast<size_t>(j)];
                best = j;
            }
        transpositions[static_cast<size_t>(k)] = int(best);
        if (best != k) {
            std::swap_ranges(qr.col(k), qr.col(k) + m, qr.col(best));
            std::swap(norms_upd[static_cast<size_t>(k)], norms_upd[static_cast<size_t>(best)]);
            std::swap(norms_dir[static_cast<size_t>(k)], norms_dir[static_cast<size_t>(best)]);
        }
        double tau, beta;
        make_householder(qr.col(k) + k, m - k, tau, beta);
        hcoeffs[static_cast<size_t>(k)] = tau;
        qr(k, k) = beta;
        apply_householder_left(qr.col(k + 1) + k, m - k, n - k - 1, m, qr.col(k) + k + 1, tau);
        for (Index j = k + 1; j < n; ++j) {
            if (norms_upd[static_cast<size_t>(j)] != 0.0) {
                double temp = std::abs(qr(k, j)) / norms_upd[static_cast<size_t>(j)];
                temp = (1.0 + temp) * (1.0 - temp);
                temp = temp < 0.0 ? 0.0 : temp;
                double ratio = norms_upd[static_cast<size_t>(j)] / norms_dir[static_cast<size_t>(j)];
                double temp2 = temp * ratio * ratio;
                if (temp2 <= downdate_thr) {
                    norms_dir[static_cast<size_t>(j)] = std::sqrt(sq_norm(qr.col(j) + k + 1, m - k - 1));
                    norms_upd[static_cast<size_t>(j)] = norms_dir[static_cast<size_t>(j)];
                } else {
                    norms_upd[static_cast<size_t>(j)] *= std::sqrt(temp);
                }
            }
        }
    }
    perm.resize(static_cast<size_t>(n));
    for (Index j = 0; j < n; ++j) perm[static_cast<size_t>(j)] = int(j);
    for (Index k = 0; k < size; ++k) std::swap(perm[static_cast<size_t>(k)], perm[static_cast<size_t>(transpositions[static_cast<size_t>(k)])]);
}

Mat ColPivQR::householder_q_thin(Index ncols) const { return form_q(qr, hcoeffs, ncols); }

Mat ColPivQR::matrix_r() const {
    Index s = std::min(qr.r, qr.c);
    Mat r(s, qr.c);
    for (Index j = 0; j < qr.c; ++j)
        for (Index i = 0; i <= std::min(j, s - 1); ++i) r(i, j) = qr(i, j);
    return r;
}

void HouseholderQR::compute(const Mat& y) {
    const Index m = y.r, n = y.c, size = std::min(m, n);
    qr = y;
    hcoeffs.assign(static_cast<size_t>(size), 0.0);
    for (Index k = 0; k < size; ++k) {
        double tau, beta;
        make_householder(qr.col(k) + k, m - k, tau, beta);
        hcoeffs[static_cast<size_t>(k)] = tau;
        qr(k, k) = beta;
        apply_householder_left(qr.col(k + 1) + k, m - k, n - k - 1, m, qr.col(k) + k + 1, tau);
    }
}

Mat HouseholderQR::householder_q_thin(Index ncols) const { return form_q(qr, hcoeffs, ncols); }

// -------------------------------------------------------------------- SVD
namespace {

/// One-sided Jacobi on the columns of u (m x n, m >= n); v accumulates.
void jacobi_columns(Mat& u, Mat& v) {
    const Index m = u.r, n = u.c;
    const double eps = std::numeric_limits<double>::epsilon();
    for (int sweep = 0; sweep < 80; ++sweep) {
        bool rotated = false;
        for (Index p = 0; p < n - 1; ++p)
            for (Index q = p + 1; q < n; ++q) {
                double* up = u.col(p);
                double* uq = u.col(q);
                double alpha = 0, beta = 0, gamma = 0;
                for (Index i = 0; i < m; ++i) {
                    alpha += up[i] * up[i];
                    beta += uq[i] * uq[i];
                    gamma += up[i] * uq[i];
                }
                if (gamma == 0.0 || std::abs(gamma) <= eps * std::sqrt(alpha * beta)) continue;
                rotated = true;
                double zeta = (beta - alpha) / (2.0 * gamma);
                double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
                for (Index i = 0; i < m; ++i) {
                    double a = up[i], b = uq[i];
                    up[i] = c * a - s * b;
                    uq[i] = s * a + c * b;
                }
                double* vp = v.col(p);
                double* vq = v.col(q);
                for (Index i = 0; i < v.r; ++i) {
                    double a = vp[i], b = vq[i];
                    vp[i] = c * a - s * b;
                    vq[i] = s * a + c * b;
                }
            }
        if (!rotated) break;
    }
}

}  // namespace

void ThinSVD::compute(const Mat& a) {
    const bool tall = a.r >= a.c;
    Mat w = tall ? a : a.transpose();
    const Index n = w.c;
    Mat vv = Mat::identity(n, n);
    jacobi_columns(w, vv);
    std::vector<double> sv(static_cast<size_t>(n));
    for (Index j = 0; j < n; ++j) sv[static_cast<size_t>(j)] = std::sqrt(sq_norm(w.col(j), w.r));
    std::vector<Index> order(static_cast<size_t>(n));
    for (Index j = 0; j < n; ++j) order[static_cast<size_t>(j)] = j;
    std::stable_sort(order.begin(), order.end(),
                     [&](Index x, Index y) { return sv[static_cast<size_t>(x)] > sv[static_cast<size_t>(y)]; });
    Mat uu(w.r, n), vs(n, n);
    s.assign(static_cast<size_t>(n), 0.0);
    for (Index j = 0; j < n; ++j) {
        Index o = order[static_cast<size_t>(j)];
        s[static_cast<size_t>(j)] = sv[static_cast<size_t>(o)];
        for (Index i = 0; i < w.r; ++i) uu(i, j) = sv[static_cast<size_t>(o)] > 0 ? w(i, o) / sv[static_cast<size_t>(o)] : 0.0;
        for (Index i = 0; i < n; ++i) vs(i, j) = vv(i, o);
    }
    if (tall) {
        u = uu;
        v = vs;
    } else {
        u = vs;
        v = uu;
    }
}

// -------------------------------------------------------------------- LLT
void LLT::compute(const Mat& a) {
    const Index n = a.r;
    l = Mat(n, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = j; i < n; ++i) l(i, j) = a(i, j);  // lower triangle only
    ok = true;
    for (Index k = 0; k < n; ++k) {
        double x = l(k, k);
        for (Index p = 0; p < k; ++p) x -= l(k, p) * l(k, p);
        if (x <= 0.0) {
            ok = false;
            return;
        }
        x = std::sqrt(x);
        l(k, k) = x;
        for (Index p = 0; p < k; ++p) {
            double lkp = l(k, p);
            if (lkp == 0.0) continue;
            const double* cp = l.col(p);
            double* ck = l.col(k);
            for (Index i = k + 1; i < n; ++i) ck[i] -= cp[i] * lkp;
        }
        for (Index i = k + 1; i < n; ++i) l(i, k) /= x;
    }
}

Mat LLT::solve(const Mat& b) const {
    const Index n = l.r;
    Mat x = b;
    for (Index c = 0; c < x.c; ++c) {
        double* xc = x.col(c);
        for (Index i = 0; i < n; ++i) {  // L y = b
            double s = xc[i];
            for (Index p = 0; p < i; ++p) s -= l(i, p) * xc[p];
            xc[i] = s / l(i, i);
        }
        for (Index i = n - 1; i >= 0; --i) {  // L^T x = y
            double s = xc[i];
            const double* li = l.col(i);
            for (Index p = i + 1; p < n; ++p) s -= li[p] * xc[p];
            xc[i] = s / l(i, i);
        }
    }
    return x;
}

// ------------------------------------------------------------ PartialPivLU
void PartialPivLU::compute(const Mat& a) {
    const Index n = a.r;
    lu = a;
    perm.resize(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) perm[static_cast<size_t>(i)] = int(i);
    int ntrans = 0;
    for (Index k = 0; k < n; ++k) {
        Index best = k;
        double bv = std::abs(lu(k, k));
        for (Index i = k + 1; i < n; ++i)
            if (std::abs(lu(i, k)) > bv) {
                bv = std::abs(lu(i, k));
                best = i;
            }
        if (best != k) {
            ++ntrans;
            for (Index j = 0; j < n; ++j) std::swap(lu(k, j), lu(best, j));
            std::swap(perm[static_cast<size_t>(k)], perm[static_cast<size_t>(best)]);
        }
        double piv = lu(k, k);
        if (piv != 0.0)
            for (Index i = k + 1; i < n; ++i) lu(i, k) /= piv;
        for (Index j = k + 1; j < n; ++j) {
            double ukj = lu(k, j);
            if (ukj == 0.0) continue;
            double* cj = lu.col(j);
            const double* ck = lu.col(k);
            for (Index i = k + 1; i < n; ++i) cj[i] -= ck[i] * ukj;
        }
    }
    transpositions_parity = ntrans % 2;
}

Mat PartialPivLU::solve(const Mat& b) const {
    const Index n = lu.r;
    Mat x(b.r, b.c);
    for (Index c = 0; c < b.c; ++c) {
        double* xc = x.col(c);
        for (Index i = 0; i < n; ++i) xc[i] = b(perm[static_cast<size_t>(i)], c);
        for (Index j = 0; j < n; ++j) {  // unit lower
            double xj = xc[j];
            const double* lj = lu.col(j);
            for (Index i = j + 1; i < n; ++i) xc[i] -= lj[i] * xj;
        }
        for (Index j = n - 1; j >= 0; --j) {  // upper
            xc[j] /= lu(j, j);
            double xj = xc[j];
            const double* uj = lu.col(j);
            for (Index i = 0; i < j; ++i) xc[i] -= uj[i] * xj;
        }
    }
    return x;
}

Mat PartialPivLU::solve_transpose(const Mat& b) const {
    // A^T = U^T L^T P  =>  x = P^T L^{-T} U^{-T} b
    const Index n = lu.r;
    Mat x(b.r, b.c);
    std::vector<double> w(static_cast<size_t>(n));
    for (Index c = 0; c < b.c; ++c) {
        for (Index i = 0; i < n; ++i) w[static_cast<size_t>(i)] = b(i, c);
        for (Index i = 0; i < n; ++i) {  // U^T y = b (lower, non-unit)
            double s = w[static_cast<size_t>(i)];
            const double* ui = lu.col(i);
            for (Index p = 0; p < i; ++p) s -= ui[p] * w[static_cast<size_t>(p)];
            w[static_cast<size_t>(i)] = s / lu(i, i);
        }
        for (Index i = n - 1; i >= 0; --i) {  // L^T z = y (upper, unit)
            double s = w[static_cast<size_t>(i)];
            const double* li = lu.col(i);
            for (Index p = i + 1; p < n; ++p) s -= li[p] * w[static_cast<size_t>(p)];
            w[static_cast<size_t>(i)] = s;
        }
        for (Index i = 0; i < n; ++i) x(perm[static_cast<size_t>(i)], c) = w[static_cast<size_t>(i)];
    }
    return x;
}

// -------------------------------------------------------------------- RNG
Mat randn(Index r, Index c, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> g(0.0, 1.0);
    Mat m(r, c);
    for (Index i = 0; i < r; ++i)
        for (Index j = 0; j < c; ++j) m(i, j) = g(rng);
    return m;
}

}  // namespace oracle
