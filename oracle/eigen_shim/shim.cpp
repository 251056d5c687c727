// TEST INFRASTRUCTURE ONLY — out-of-line parts of the Eigen-API shim
// (oracle/eigen_shim/Eigen/Dense): strided copies and reductions, the GEMM
// dispatch, and the decompositions, which delegate to the restated Eigen 3.4
// algorithms in oracle/dense.cpp.
#include <Eigen/Dense>

#include <algorithm>
#include <omp.h>

#include "../oracle.hpp"

namespace Eigen {
namespace internal {

bool overlaps(const View& a, const View& b) {
    if (!a.p || !b.p || a.r == 0 || a.c == 0 || b.r == 0 || b.c == 0) return false;
    auto span = [](const View& w, const double*& lo, const double*& hi) {
        const double* p0 = w.p;
        const double* p1 = w.p + (w.r - 1) * w.rs + (w.c - 1) * w.cs;
        lo = std::min(p0, p1);
        hi = std::max(p0, p1);
        // negative strides never occur; min/max covers transposed views
        const double* q0 = w.p + (w.r - 1) * w.rs;
        const double* q1 = w.p + (w.c - 1) * w.cs;
        lo = std::min({lo, q0, q1});
        hi = std::max({hi, q0, q1});
    };
    const double *alo, *ahi, *blo, *bhi;
    span(a, alo, ahi);
    span(b, blo, bhi);
    return !(ahi < blo || bhi < alo);
}

void copy_view(const View& s, const View& d) {
    if (s.rs == 1 && d.rs == 1) {
        for (Index j = 0; j < s.c; ++j) std::copy(s.p + j * s.cs, s.p + j * s.cs + s.r, d.p + j * d.cs);
        return;
    }
    for (Index j = 0; j < s.c; ++j)
        for (Index i = 0; i < s.r; ++i) d.at(i, j) = s.at(i, j);
}

// Reductions use the restated pairwise (Eigen-like blocked) summation.
double dot_view(const View& a, const View& b) {
    if (a.r * a.c != b.r * b.c) throw std::invalid_argument("dot: size mismatch");
    const Index n = a.r * a.c;
    auto stride = [](const View& w) { return w.c == 1 ? w.rs : w.cs; };
    if ((a.c == 1 || a.r == 1) && (b.c == 1 || b.r == 1)) return oracle::pdot(a.p, b.p, n, stride(a), stride(b));
    double s = 0;
    for (Index j = 0; j < a.c; ++j) s += oracle::pdot(a.p + j * a.cs, b.p + j * b.cs, a.r, a.rs, b.rs);
    return s;
}

double sum_view(const View& a) {
    static const double one = 1.0;
    double s = 0;
    for (Index j = 0; j < a.c; ++j) s += oracle::pdot(a.p + j * a.cs, &one, a.r, a.rs, 0);
    return s;
}

double sqnorm_view(const View& a) {
    double s = 0;
    for (Index j = 0; j < a.c; ++j) s += oracle::pdot(a.p + j * a.cs, a.p + j * a.cs, a.r, a.rs, a.rs);
    return s;
}

namespace {
/// BLAS view of a strided operand: column-major ('N', ld) or the transpose
/// of one ('T', ld). Returns false when neither stride is unit.
bool blas_form(const View& w, bool& trans, Index& ld) {
    if (w.rs == 1) {
        trans = false;
        ld = std::max<Index>(w.cs, std::max<Index>(w.r, 1));
        return true;
    }
    if (w.cs == 1) {
        trans = true;
        ld = std::max<Index>(w.rs, std::max<Index>(w.c, 1));
        return true;
    }
    if (w.c == 1) {  // strided column = transpose of a 1 x r row with ld = rs
        trans = true;
        ld = std::max<Index>(w.rs, 1);
        return true;
    }
    if (w.r == 1) {
        trans = false;
        ld = std::max<Index>(w.cs, 1);
        return true;
    }
    return false;
}
}  // namespace

void gemm_view(const View& a, const View& b, double alpha, double beta, const View& c) {
    const Index m = a.r, n = b.c, k = a.c;
    if (m == 0 || n == 0) return;
    if (c.rs != 1) throw std::logic_error("gemm_view: output must be column-major");
    MatrixXd ta, tb;
    View A = a, B = b;
    bool tra, trb;
    Index lda, ldb;
    if (!blas_form(A, tra, lda)) {
        ta = MatrixXd(Block(A));
        A = ta.view();
        blas_form(A, tra, lda);
    }
    if (!blas_form(B, trb, ldb)) {
        tb = MatrixXd(Block(B));
        B = tb.view();
        blas_form(B, trb, ldb);
    }
    const Index ldc = std::max<Index>(c.cs, std::max<Index>(m, 1));
    if (k == 0) {
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < m; ++i) c.at(i, j) = beta == 0.0 ? 0.0 : beta * c.at(i, j);
        return;
    }
    // Eigen parallelises large products over OpenMP when not already inside a
    // parallel region; split the longer output dimension across threads.
    const int nt = omp_in_parallel() ? 1 : omp_get_max_threads();
    const double work = double(m) * double(n) * double(k);
    if (nt > 1 && work > 4.0e6) {
        const bool split_n = n >= m;
        const Index len = split_n ? n : m;
        const Index chunks = std::min<Index>(nt, std::max<Index>(1, len / 16));
#pragma omp parallel for schedule(static) num_threads(int(chunks))
        for (Index t = 0; t < chunks; ++t) {
            const Index lo = len * t / chunks, hi = len * (t + 1) / chunks;
            if (hi <= lo) continue;
            if (split_n) {
                // op(B) columns lo..hi: 'N' -> B + lo*ldb; 'T' -> B + lo
                const double* Bp = trb ? B.p + lo : B.p + lo * ldb;
                oracle::gemm(tra, trb, m, hi - lo, k, alpha, A.p, lda, Bp, ldb, beta, c.p + lo * ldc, ldc);
            } else {
                const double* Ap = tra ? A.p + lo * lda : A.p + lo;
                oracle::gemm(tra, trb, hi - lo, n, k, alpha, Ap, lda, B.p, ldb, beta, c.p + lo, ldc);
            }
        }
        return;
    }
    oracle::gemm(tra, trb, m, n, k, alpha, A.p, lda, B.p, ldb, beta, c.p, ldc);
}

}  // namespace internal

// --------------------------------------------------------------- helpers
namespace {
oracle::Mat to_mat(const MatrixXd& a) {
    oracle::Mat m(a.rows(), a.cols());
    if (a.size()) std::copy(a.data(), a.data() + a.size(), m.data());
    return m;
}
MatrixXd from_mat(const oracle::Mat& m) {
    MatrixXd a(m.r, m.c);
    if (m.r * m.c) std::copy(m.data(), m.data() + m.r * m.c, a.data());
    return a;
}
}  // namespace

MatrixXd MatrixXd::Random(Index r, Index c) {
    MatrixXd m(r, c);
    for (Index j = 0; j < c; ++j)
        for (Index i = 0; i < r; ++i) m(i, j) = -1.0 + 2.0 * double(std::rand()) / double(RAND_MAX);
    return m;
}
VectorXd VectorXd::Random(Index n) { return VectorXd(MatrixXd::Random(n, 1)); }
VectorXd VectorXd::LinSpaced(Index n, double lo, double hi) {
    VectorXd v(n);
    if (n == 1) {
        v[0] = hi;
        return v;
    }
    const double step = (hi - lo) / double(n - 1);
    // Eigen's linspaced_op: lo + i*step, last element forced to hi.
    for (Index i = 0; i < n; ++i) v[i] = i == n - 1 ? hi : lo + double(i) * step;
    return v;
}

void MatrixXd::conservativeResize(Index r, Index c) {
    MatrixXd t(r, c);
    for (Index j = 0; j < std::min(c, c_); ++j)
        for (Index i = 0; i < std::min(r, r_); ++i) t(i, j) = (*this)(i, j);
    *this = std::move(t);
}

// Q * m with Q = H_0 ... H_{s-1} (v_k = [1; essential below the diagonal]).
MatrixXd HouseholderSequence::apply(const internal::View& mv) const {
    MatrixXd out(Block{mv});
    const MatrixXd& qr = *qr_;
    const Index rows = qr.rows(), s = Index(h_->size()), cols = out.cols();
    if (out.rows() != rows) throw std::invalid_argument("householderQ(): dimension mismatch");
    for (Index k = s - 1; k >= 0; --k) {
        const double tau = (*h_)[static_cast<size_t>(k)];
        const Index len = rows - k;
        if (len == 1) {
            for (Index j = 0; j < cols; ++j) out(k, j) *= (1.0 - tau);
            continue;
        }
        if (tau == 0.0) continue;
        const double* ess = qr.data() + k + 1 + k * rows;
        for (Index j = 0; j < cols; ++j) {
            double* cj = out.data() + k + j * rows;
            double t = oracle::pdot(ess, cj + 1, len - 1, 1, 1) + cj[0];
            cj[0] -= tau * t;
            for (Index i = 1; i < len; ++i) cj[i] -= tau * ess[i - 1] * t;
        }
    }
    return out;
}

namespace impl {

HouseholderQR& HouseholderQR::compute(const MatrixXd& a) {
    oracle::HouseholderQR q;
    q.compute(to_mat(a));
    qr_ = from_mat(q.qr);
    h_ = q.hcoeffs;
    return *this;
}

ColPivHouseholderQR& ColPivHouseholderQR::compute(const MatrixXd& a) {
    oracle::ColPivQR q;
    q.compute(to_mat(a));
    qr_ = from_mat(q.qr);
    h_ = q.hcoeffs;
    perm_ = PermutationMatrix(VectorXi(std::vector<int>(q.perm.begin(), q.perm.end())));
    return *this;
}

LLT& LLT::compute(const MatrixXd& a) {
    oracle::LLT l;
    l.compute(to_mat(a));
    ok_ = l.ok;
    l_ = from_mat(l.l);
    return *this;
}

MatrixXd LLT::solve_impl(const MatrixXd& b) const {
    oracle::LLT l;
    l.l = to_mat(l_);
    l.ok = ok_;
    return from_mat(l.solve(to_mat(b)));
}

PartialPivLU& PartialPivLU::compute(const MatrixXd& a) {
    oracle::PartialPivLU lu;
    lu.compute(to_mat(a));
    lu_ = from_mat(lu.lu);
    rowperm_ = lu.perm;
    parity_ = lu.transpositions_parity;
    // Eigen's permutationP(): P with (P A) = L U; indices()[i] = destination of row i.
    std::vector<int> dest(rowperm_.size());
    for (size_t i = 0; i < rowperm_.size(); ++i) dest[static_cast<size_t>(rowperm_[i])] = int(i);
    p_ = PermutationMatrix(VectorXi(dest));
    return *this;
}

double PartialPivLU::determinant() const {
    double d = parity_ ? -1.0 : 1.0;
    for (Index i = 0; i < lu_.rows(); ++i) d *= lu_(i, i);
    return d;
}

MatrixXd PartialPivLU::solve_impl(const MatrixXd& b, bool trans) const {
    oracle::PartialPivLU lu;
    lu.lu = to_mat(lu_);
    lu.perm = rowperm_;
    lu.transpositions_parity = parity_;
    return from_mat(trans ? lu.solve_transpose(to_mat(b)) : lu.solve(to_mat(b)));
}

JacobiSVD& JacobiSVD::compute(const MatrixXd& a, unsigned int) {
    oracle::ThinSVD s;
    s.compute(to_mat(a));
    u_ = from_mat(s.u);
    v_ = from_mat(s.v);
    s_ = VectorXd(Index(s.s.size()));
    for (size_t i = 0; i < s.s.size(); ++i) s_[Index(i)] = s.s[i];
    return *this;
}

// Cyclic Jacobi eigenvalue iteration (symmetric input; ascending order like
// Eigen's SelfAdjointEigenSolver).
SelfAdjointEigenSolver& SelfAdjointEigenSolver::compute(const MatrixXd& a0, int) {
    const Index n = a0.rows();
    MatrixXd a = a0, z = MatrixXd::Identity(n, n);
    info_ = Success;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0;
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < n; ++i)
                if (i != j) off += a(i, j) * a(i, j);
        if (off <= 1e-300) break;
        for (Index p = 0; p < n - 1; ++p)
            for (Index q = p + 1; q < n; ++q) {
                if (a(p, q) == 0.0) continue;
                const double th = (a(q, q) - a(p, p)) / (2.0 * a(p, q));
                const double t = (th >= 0 ? 1.0 : -1.0) / (std::abs(th) + std::sqrt(th * th + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (Index k = 0; k < n; ++k) {
                    const double akp = a(k, p), akq = a(k, q);
                    a(k, p) = c * akp - s * akq;
                    a(k, q) = s * akp + c * akq;
                }
                for (Index k = 0; k < n; ++k) {
                    const double apk = a(p, k), aqk = a(q, k);
                    a(p, k) = c * apk - s * aqk;
                    a(q, k) = s * apk + c * aqk;
                }
                for (Index k = 0; k < n; ++k) {
                    const double zkp = z(k, p), zkq = z(k, q);
                    z(k, p) = c * zkp - s * zkq;
                    z(k, q) = s * zkp + c * zkq;
                }
            }
    }
    std::vector<Index> order(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) order[static_cast<size_t>(i)] = i;
    std::stable_sort(order.begin(), order.end(), [&](Index x, Index y) { return a(x, x) < a(y, y); });
    w_ = VectorXd(n);
    z_ = MatrixXd(n, n);
    for (Index j = 0; j < n; ++j) {
        const Index o = order[static_cast<size_t>(j)];
        w_[j] = a(o, o);
        for (Index i = 0; i < n; ++i) z_(i, j) = z(i, o);
    }
    return *this;
}

}  // namespace impl
}  // namespace Eigen
