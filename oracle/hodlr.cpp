// TEST INFRASTRUCTURE ONLY — HODLR hot path of the parity oracle.
//
// Line-by-line restatement of /root/reference/proj/src/{cluster_tree,
// hodlr_matrix,sketch,factorization,product_rep,mle}.cpp on oracle::Mat.
// Each function cites the reference lines it follows.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <numeric>
#include <random>

#include "oracle.hpp"
#include "matern1d.hpp"


namespace oracle {

bool g_q2_reorthogonalize = false;
void set_q2_reorthogonalize(bool on) { g_q2_reorthogonalize = on; }
bool g_compress_at_level = false;
void set_compress_at_level(bool on) { g_compress_at_level = on; }

// ============================================================ cluster tree
// cluster_tree.cpp:10-22
ClusterTree::ClusterTree(Index n, int tau) : n_(n), tau_(tau) {
    levels_.resize(static_cast<size_t>(tau + 1));
    levels_[0] = {Range{0, n}};
    for (int d = 1; d <= tau; ++d) {
        levels_[static_cast<size_t>(d)].reserve(static_cast<size_t>(1) << d);
        for (const Range& p : levels_[static_cast<size_t>(d - 1)]) {
            Index left = (p.size() + 1) / 2;  // left child takes ceil(len/2)
            levels_[static_cast<size_t>(d)].push_back(Range{p.lo, p.lo + left});
            levels_[static_cast<size_t>(d)].push_back(Range{p.lo + left, p.hi});
        }
    }
}

// cluster_tree.cpp:24-28
Index ClusterTree::max_leaf_size() const {
    Index m = 0;
    for (const Range& r : leaves()) m = std::max(m, r.size());
    return m;
}

// cluster_tree.cpp:34-38
int tree_depth(Index n, Index leaf_min, Index leaf_max) {
    if (n <= leaf_max) return 0;
    int tau = int(std::floor(std::log2(double(n) / double(leaf_min))));
    return std::max(tau, 1);
}

// cluster_tree.cpp:40-90
KdOrdering build_kd_ordering(const Mat& c, Index leaf_min, Index leaf_max) {
    const Index n = c.r;
    const int d = int(c.c);
    if (n < 1) throw std::invalid_argument("build_kd_ordering: empty point set");
    if (d != 1 && d != 2) throw std::invalid_argument("build_kd_ordering: d must be 1 or 2");
    if (leaf_min < 1 || leaf_min > leaf_max)
        throw std::invalid_argument("build_kd_ordering: need 1 <= leaf_min <= leaf_max");
    for (double v : c.a)
        if (!std::isfinite(v)) throw std::invalid_argument("build_kd_ordering: non-finite coordinates");
    KdOrdering out;
    out.tree = ClusterTree(n, tree_depth(n, leaf_min, leaf_max));
    std::vector<Index> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), Index{0});
    for (int depth = 0; depth < out.tree.depth(); ++depth) {
        for (const auto& node : out.tree.level(depth)) {
            auto first = order.begin() + node.lo, last = order.begin() + node.hi;
            int axis = 0;
            if (d == 2) {
                double lo0 = c(*first, 0), hi0 = lo0, lo1 = c(*first, 1), hi1 = lo1;
                for (auto it = first; it != last; ++it) {
                    lo0 = std::min(lo0, c(*it, 0));
                    hi0 = std::max(hi0, c(*it, 0));
                    lo1 = std::min(lo1, c(*it, 1));
                    hi1 = std::max(hi1, c(*it, 1));
                }
                axis = (hi1 - lo1) > (hi0 - lo0) ? 1 : 0;
            }
            std::stable_sort(first, last, [&](Index a, Index b) {
                if (c(a, axis) != c(b, axis)) return c(a, axis) < c(b, axis);
                return a < b;
            });
        }
    }
    out.inv = order;
    out.perm.resize(static_cast<size_t>(n));
    for (Index pos = 0; pos < n; ++pos) out.perm[static_cast<size_t>(order[static_cast<size_t>(pos)])] = pos;
    out.reordered_coords = Mat(n, d);
    for (Index pos = 0; pos < n; ++pos)
        for (int k = 0; k < d; ++k) out.reordered_coords(pos, k) = c(order[static_cast<size_t>(pos)], k);
    return out;
}

// ============================================================ low-rank block
// hodlr_matrix.cpp:17-22: y += left (right^T x)
void LowRankBlock::apply(const Mat& x, Index xr0, Mat& y, Index yr0) const {
    if (empty()) return;
    const Index s = x.c;
    Mat t(rank(), s);
    gemm(true, false, rank(), s, right.r, 1.0, right.data(), right.r, x.data() + xr0, x.r, 0.0,
         t.data(), rank());
    gemm(false, false, left.r, s, rank(), 1.0, left.data(), left.r, t.data(), rank(), 1.0,
         y.data() + yr0, y.r);
}

// hodlr_matrix.cpp:24-29: y += right (left^T x)
void LowRankBlock::apply_transpose(const Mat& x, Index xr0, Mat& y, Index yr0) const {
    if (empty()) return;
    const Index s = x.c;
    Mat t(rank(), s);
    gemm(true, false, rank(), s, left.r, 1.0, left.data(), left.r, x.data() + xr0, x.r, 0.0,
         t.data(), rank());
    gemm(false, false, right.r, s, rank(), 1.0, right.data(), right.r, t.data(), rank(), 1.0,
         y.data() + yr0, y.r);
}

// hodlr_matrix.cpp:31-40
LowRankBlock LowRankBlock::concat(const LowRankBlock& a, const LowRankBlock& b) {
    if (a.empty()) return b;
    if (b.empty()) return a;
    LowRankBlock out;
    out.left = Mat(a.left.r, a.rank() + b.rank());
    out.left.set_block(0, 0, a.left);
    out.left.set_block(0, a.rank(), b.left);
    out.right = Mat(a.right.r, a.rank() + b.rank());
    out.right.set_block(0, 0, a.right);
    out.right.set_block(0, a.rank(), b.right);
    return out;
}

// hodlr_matrix.cpp:42-66
LowRankBlock LowRankBlock::compressed(double rtol) const {
    if (empty()) return *this;
    HouseholderQR ql, qr;
    ql.compute(left);
    qr.compute(right);
    const Index wl = std::min(left.r, left.c), wr = std::min(right.r, right.c);
    Mat tl(wl, left.c), tr(wr, right.c);
    for (Index j = 0; j < left.c; ++j)
        for (Index i = 0; i <= std::min(j, wl - 1); ++i) tl(i, j) = ql.qr(i, j);
    for (Index j = 0; j < right.c; ++j)
        for (Index i = 0; i <= std::min(j, wr - 1); ++i) tr(i, j) = qr.qr(i, j);
    ThinSVD svd;
    svd.compute(matmul_t(tl, false, tr, true));
    const Index wmin = std::min(wl, wr);
    Index r = 0;
    while (r < wmin && svd.s[static_cast<size_t>(r)] > rtol * svd.s[0]) ++r;
    Mat us(wl, r), vr(wr, r);
    for (Index j = 0; j < r; ++j) {
        for (Index i = 0; i < wl; ++i) us(i, j) = svd.u(i, j) * svd.s[static_cast<size_t>(j)];
        for (Index i = 0; i < wr; ++i) vr(i, j) = svd.v(i, j);
    }
    LowRankBlock out;
    out.left = matmul(ql.householder_q_thin(wl), us);
    out.right = matmul(qr.householder_q_thin(wr), vr);
    return out;
}

// ============================================================ HODLR matrix
// hodlr_matrix.cpp:68-81
HodlrMatrix HodlrMatrix::zero(const ClusterTree& tree, bool symmetric) {
    HodlrMatrix h;
    h.tree_ = tree;
    h.symmetric_ = symmetric;
    h.upper_.resize(static_cast<size_t>(tree.depth()));
    for (int l = 1; l <= tree.depth(); ++l) h.upper_[static_cast<size_t>(l - 1)].resize(tree.level(l - 1).size());
    if (!symmetric) h.lower_ = h.upper_;
    h.leaves_.resize(static_cast<size_t>(tree.num_leaves()));
    for (Index i = 0; i < tree.num_leaves(); ++i) {
        Index m = tree.leaves()[static_cast<size_t>(i)].size();
        h.leaves_[static_cast<size_t>(i)] = Mat(m, m);
    }
    return h;
}

// hodlr_matrix.cpp:83-88
HodlrMatrix HodlrMatrix::identity(const ClusterTree& tree) {
    HodlrMatrix h = zero(tree);
    for (auto& lf : h.leaves_) lf = Mat::identity(lf.r, lf.c);
    return h;
}

// hodlr_matrix.cpp:90-122
HodlrMatrix HodlrMatrix::from_dense(const ClusterTree& tree, const Mat& a, bool symmetric) {
    if (a.r != tree.size() || a.c != tree.size())
        throw std::invalid_argument("from_dense: size mismatch");
    HodlrMatrix h = zero(tree, symmetric);
    auto factor = [](const Mat& block) {
        ThinSVD svd;
        svd.compute(block);
        double tol = 1e-13 * std::max<double>(1.0, svd.s.empty() ? 0.0 : svd.s[0]);
        Index r = 0;
        while (r < Index(svd.s.size()) && svd.s[static_cast<size_t>(r)] > tol) ++r;
        LowRankBlock lr;
        lr.left = svd.u.left_cols(r);
        lr.right = Mat(svd.v.r, r);
        for (Index j = 0; j < r; ++j)
            for (Index i = 0; i < svd.v.r; ++i) lr.right(i, j) = svd.v(i, j) * svd.s[static_cast<size_t>(j)];
        return lr;
    };
    for (int l = 1; l <= tree.depth(); ++l) {
        const auto& kids = tree.level(l);
        for (size_t j = 0; j < tree.level(l - 1).size(); ++j) {
            auto cl = kids[2 * j], cr = kids[2 * j + 1];
            h.upper(l, Index(j)) = factor(a.block(cl.lo, cr.lo, cl.size(), cr.size()));
            if (!symmetric) h.lower(l, Index(j)) = factor(a.block(cr.lo, cl.lo, cr.size(), cl.size()));
        }
    }
    for (Index i = 0; i < tree.num_leaves(); ++i) {
        auto r = tree.leaves()[static_cast<size_t>(i)];
        h.leaves_[static_cast<size_t>(i)] = a.block(r.lo, r.lo, r.size(), r.size());
    }
    return h;
}

namespace {
// hodlr_matrix.cpp:126-160
HodlrMatrix random_with_shift(const ClusterTree& tree, Index k, std::uint64_t seed, double shift) {
    HodlrMatrix h = HodlrMatrix::zero(tree);
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    auto rnd = [&](Index r, Index c) {
        Mat m(r, c);
        for (Index i = 0; i < r; ++i)
            for (Index j = 0; j < c; ++j) m(i, j) = gauss(rng);
        return m;
    };
    auto div = [](Mat m, double s) {
        for (double& v : m.a) v = v / s;
        return m;
    };
    for (int l = 1; l <= tree.depth(); ++l) {
        const auto& kids = tree.level(l);
        for (size_t j = 0; j < tree.level(l - 1).size(); ++j) {
            Index m1 = kids[2 * j].size(), m2 = kids[2 * j + 1].size();
            Index r = std::min({k, m1, m2});
            LowRankBlock lr;
            lr.left = div(rnd(m1, r), std::sqrt(double(m1)));
            lr.right = div(rnd(m2, r), std::sqrt(double(m2)));
            h.upper(l, Index(j)) = lr;
        }
    }
    for (Index i = 0; i < tree.num_leaves(); ++i) {
        Index m = tree.leaves()[static_cast<size_t>(i)].size();
        Mat g = div(rnd(m, m), std::sqrt(double(m)));
        Mat gt = g.transpose();
        h.leaf(i) = 0.5 * (g + gt);
        if (shift > 0.0) {
            h.leaf(i) = matmul_t(g, false, g, true);
            for (Index t = 0; t < m; ++t) h.leaf(i)(t, t) += shift;
        }
    }
    return h;
}
}  // namespace

// hodlr_matrix.cpp:162-172
HodlrMatrix HodlrMatrix::random_spd(const ClusterTree& tree, Index k, std::uint64_t seed) {
    return random_with_shift(tree, k, seed, 2.0 + 2.0 * tree.depth());
}
HodlrMatrix HodlrMatrix::random_symmetric(const ClusterTree& tree, Index k, std::uint64_t seed) {
    return random_with_shift(tree, k, seed, 0.0);
}

// hodlr_matrix.cpp:174-180
LowRankBlock HodlrMatrix::lower_block(int l, Index j) const {
    if (symmetric_) {
        const LowRankBlock& u = upper_[static_cast<size_t>(l - 1)][static_cast<size_t>(j)];
        return LowRankBlock{u.right, u.left};
    }
    return lower_[static_cast<size_t>(l - 1)][static_cast<size_t>(j)];
}

// hodlr_matrix.cpp:182-185
LowRankBlock& HodlrMatrix::lower(int l, Index j) {
    if (symmetric_) throw std::logic_error("lower(): symmetric storage");
    return lower_[static_cast<size_t>(l - 1)][static_cast<size_t>(j)];
}

// hodlr_matrix.cpp:187-196
void HodlrMatrix::make_asymmetric() {
    if (!symmetric_) return;
    lower_.resize(upper_.size());
    for (size_t l = 0; l < upper_.size(); ++l) {
        lower_[l].resize(upper_[l].size());
        for (size_t j = 0; j < upper_[l].size(); ++j)
            lower_[l][j] = LowRankBlock{upper_[l][j].right, upper_[l][j].left};
    }
    symmetric_ = false;
}

// hodlr_matrix.cpp:198-222
Mat HodlrMatrix::matvec(const Mat& x) const {
    if (x.r != size()) throw std::invalid_argument("matvec: dimension mismatch");
    Mat y(x.r, x.c);
    const auto& lv = tree_.leaves();
#pragma omp parallel for schedule(static)
    for (Index i = 0; i < num_leaves(); ++i) {
        auto r = lv[static_cast<size_t>(i)];
        gemm(false, false, r.size(), x.c, r.size(), 1.0, leaves_[static_cast<size_t>(i)].data(), r.size(),
             x.data() + r.lo, x.r, 1.0, y.data() + r.lo, y.r);
    }
    for (int l = 1; l <= depth(); ++l) {
        const auto& kids = tree_.level(l);
        const Index nodes = Index(tree_.level(l - 1).size());
#pragma omp parallel for schedule(static)
        for (Index j = 0; j < nodes; ++j) {
            auto cl = kids[static_cast<size_t>(2 * j)], cr = kids[static_cast<size_t>(2 * j + 1)];
            upper(l, j).apply(x, cr.lo, y, cl.lo);
            lower_block(l, j).apply(x, cl.lo, y, cr.lo);
        }
    }
    return y;
}

// hodlr_matrix.cpp:228-265
Mat HodlrMatrix::sub_matvec(int d, Index node, const Mat& x, bool transpose) const {
    auto range = tree_.level(d)[static_cast<size_t>(node)];
    if (x.r != range.size()) throw std::invalid_argument("sub_matvec: dimension mismatch");
    Mat y(x.r, x.c);
    Index leaves_per = num_leaves() >> d;
    for (Index i = node * leaves_per; i < (node + 1) * leaves_per; ++i) {
        auto r = tree_.leaves()[static_cast<size_t>(i)];
        Index off = r.lo - range.lo;
        gemm(transpose, false, r.size(), x.c, r.size(), 1.0, leaves_[static_cast<size_t>(i)].data(), r.size(),
             x.data() + off, x.r, 1.0, y.data() + off, y.r);
    }
    for (int l = d + 1; l <= depth(); ++l) {
        Index per = (Index{1} << (l - 1)) >> d;
        const auto& kids = tree_.level(l);
        for (Index j = node * per; j < (node + 1) * per; ++j) {
            auto cl = kids[static_cast<size_t>(2 * j)], cr = kids[static_cast<size_t>(2 * j + 1)];
            Index ol = cl.lo - range.lo, orr = cr.lo - range.lo;
            const LowRankBlock up = upper(l, j);
            const LowRankBlock lo = lower_block(l, j);
            if (transpose) {
                up.apply_transpose(x, ol, y, orr);
                lo.apply_transpose(x, orr, y, ol);
            } else {
                up.apply(x, orr, y, ol);
                lo.apply(x, ol, y, orr);
            }
        }
    }
    return y;
}

// hodlr_matrix.cpp:267-271
double HodlrMatrix::trace() const {
    double t = 0;
    for (const auto& lf : leaves_) t += lf.trace();
    return t;
}

// hodlr_matrix.cpp:273-292
Mat HodlrMatrix::densify() const {
    if (size() > (Index{1} << 14)) throw std::length_error("densify: matrix too large");
    Mat a(size(), size());
    for (Index i = 0; i < num_leaves(); ++i) {
        auto r = tree_.leaves()[static_cast<size_t>(i)];
        a.set_block(r.lo, r.lo, leaves_[static_cast<size_t>(i)]);
    }
    for (int l = 1; l <= depth(); ++l) {
        const auto& kids = tree_.level(l);
        for (size_t j = 0; j < tree_.level(l - 1).size(); ++j) {
            auto cl = kids[2 * j], cr = kids[2 * j + 1];
            if (!upper(l, Index(j)).empty()) a.set_block(cl.lo, cr.lo, upper(l, Index(j)).dense());
            LowRankBlock lo = lower_block(l, Index(j));
            if (!lo.empty()) a.set_block(cr.lo, cl.lo, lo.dense());
        }
    }
    return a;
}

// hodlr_matrix.cpp:294-318
double HodlrMatrix::trace_product(const HodlrMatrix& a, const HodlrMatrix& b) {
    if (!a.tree().same_structure(b.tree())) throw std::invalid_argument("trace_product: tree mismatch");
    double t = 0;
    for (Index i = 0; i < a.num_leaves(); ++i) {
        const Mat& x = a.leaf(i);
        const Mat& y = b.leaf(i);
        double s = 0;
        for (Index c = 0; c < x.c; ++c) s += pdot(&x.a[static_cast<size_t>(c)], y.col(c), x.r, x.r, 1);
        t += s;
    }
    for (int l = 1; l <= a.depth(); ++l) {
        for (size_t j = 0; j < a.tree().level(l - 1).size(); ++j) {
            const LowRankBlock au = a.upper(l, Index(j)), al = a.lower_block(l, Index(j));
            const LowRankBlock bu = b.upper(l, Index(j)), bl = b.lower_block(l, Index(j));
            if (!au.empty() && !bl.empty())
                t += matmul(matmul_t(bl.right, true, au.left, false),
                            matmul_t(au.right, true, bl.left, false))
                         .trace();
            if (!al.empty() && !bu.empty())
                t += matmul(matmul_t(bu.right, true, al.left, false),
                            matmul_t(al.right, true, bu.left, false))
                         .trace();
        }
    }
    return t;
}

// ========================================================= Matérn oracle
Matern1dOracle::Matern1dOracle(std::vector<double> x, int nu2, double sigma2, double ell,
                               double nugget, bool scan)
    : x_(std::move(x)), nu2_(nu2), sigma2_(sigma2), ell_(ell), nugget_(nugget), scan_(scan) {
    if (nu2 != 1 && nu2 != 3 && nu2 != 5) throw std::invalid_argument("Matern1d: nu in {1/2,3/2,5/2}");
    for (size_t i = 1; i < x_.size(); ++i)
        if (x_[i] < x_[i - 1]) throw std::invalid_argument("Matern1d: points must be sorted");
}

double Matern1dOracle::kernel(double d, int which) const {
    return matern1d::kernel(nu2_, which, sigma2_, ell_, d);
}

Mat Matern1dOracle::apply_impl(int which, const Mat& v) const {
    const Index n = dim();
    if (v.r != n) throw std::invalid_argument("Matern1d: dimension mismatch");
    Mat y(n, v.c);
    if (!scan_) {  // dense kernel matrix times V through the GEMM
        Mat kd(n, n);
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < n; ++i) kd(i, j) = kernel(std::abs(x_[size_t(i)] - x_[size_t(j)]), which);
        y = matmul(kd, v);
        if (which < 0 && nugget_ != 0.0)
            for (Index c = 0; c < v.c; ++c)
                for (Index i = 0; i < n; ++i) y(i, c) += nugget_ * v(i, c);
        return y;
    }
    matern1d::apply(x_.data(), n, nu2_, sigma2_, ell_, nugget_, which, true, v.data(), v.r, v.c, y.data(), n);
    return y;
}

// ================================================================= sketch
// sketch.cpp:10-31
SketchPlan::SketchPlan(const ClusterTree& tree, Index k, std::uint64_t seed)
    : k_(k), n_(tree.size()), tau_(tree.depth()) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    level_samplers_.resize(static_cast<size_t>(tau_));
    for (int l = 1; l <= tau_; ++l) {
        Mat& s = level_samplers_[static_cast<size_t>(l - 1)];
        s = Mat(n_, k);
        const auto& kids = tree.level(l);
        for (size_t j = 0; j < tree.level(l - 1).size(); ++j) {
            auto cr = kids[2 * j + 1];
            for (Index i = cr.lo; i < cr.hi; ++i)
                for (Index c = 0; c < k; ++c) s(i, c) = gauss(rng);
        }
    }
    const Index m = tree.max_leaf_size();
    leaf_sampler_ = Mat(n_, m);
    for (Index b = 0; b < tree.num_leaves(); ++b) {
        auto r = tree.leaves()[static_cast<size_t>(b)];
        for (Index i = 0; i < r.size(); ++i) leaf_sampler_(r.lo + i, i) = 1.0;
    }
}

// sketch.cpp:37-76
RangeResult randomized_range(const Mat& y, Index k) {
    const Index m = y.r;
    if (y.c != k) throw std::invalid_argument("randomized_range: expected k columns");
    if (m < k) throw std::invalid_argument("randomized_range: m < k");
    ColPivQR qr;
    qr.compute(y);
    RangeResult out;
    out.q = qr.householder_q_thin(k);
    out.r = Mat(k, k);
    for (Index j = 0; j < k; ++j)
        for (Index i = 0; i <= j; ++i) out.r(i, j) = qr.qr(i, j);
    out.perm = qr.perm;
    for (Index i = 0; i < k; ++i) {
        if (out.r(i, i) < 0) {
            for (Index t = 0; t < m; ++t) out.q(t, i) = -out.q(t, i);
            for (Index t = 0; t < k; ++t) out.r(i, t) = -out.r(i, t);
        }
    }
    const double d0 = std::abs(out.r(0, 0));
    out.numeric_rank = 0;
    while (out.numeric_rank < k &&
           std::abs(out.r(out.numeric_rank, out.numeric_rank)) >
               64 * std::numeric_limits<double>::epsilon() * d0)
        ++out.numeric_rank;
    if (out.numeric_rank < k) {
        for (Index i = out.numeric_rank; i < k; ++i)
            for (Index t = 0; t < k; ++t) out.r(i, t) = 0.0;
        Index filled = out.numeric_rank;
        std::vector<double> v(static_cast<size_t>(m)), g(static_cast<size_t>(k));
        for (Index e = 0; e < m && filled < k; ++e) {
            std::fill(v.begin(), v.end(), 0.0);
            v[static_cast<size_t>(e)] = 1.0;
            for (int pass = 0; pass < 2; ++pass) {
                for (Index c = 0; c < filled; ++c) {
                    double s = 0;
                    const double* qc = out.q.col(c);
                    for (Index t = 0; t < m; ++t) s += qc[t] * v[static_cast<size_t>(t)];
                    g[static_cast<size_t>(c)] = s;
                }
                for (Index c = 0; c < filled; ++c) {
                    const double* qc = out.q.col(c);
                    for (Index t = 0; t < m; ++t) v[static_cast<size_t>(t)] -= qc[t] * g[static_cast<size_t>(c)];
                }
            }
            double nv = 0;
            for (double x : v) nv += x * x;
            nv = std::sqrt(nv);
            if (nv < 0.5) continue;
            for (Index t = 0; t < m; ++t) out.q(t, filled) = v[static_cast<size_t>(t)] / nv;
            ++filled;
        }
    }
    return out;
}

namespace {
/// X <- X R^{-1}, R upper triangular (Eigen solveInPlace<OnTheRight>).
void solve_upper_right(Mat& x, const Mat& r) {
    const Index k = r.r;
    for (Index j = 0; j < k; ++j) {
        double* xj = x.col(j);
        for (Index i = 0; i < j; ++i) {
            double rij = r(i, j);
            if (rij == 0.0) continue;
            const double* xi = x.col(i);
            for (Index t = 0; t < x.r; ++t) xj[t] -= xi[t] * rij;
        }
        for (Index t = 0; t < x.r; ++t) xj[t] /= r(j, j);
    }
}
}  // namespace

// sketch.cpp:78-111
DiffQrResult diff_qr(const Mat& b, const Mat& db, const Mat& q, const Mat& r) {
    (void)b;
    const Index k = r.r;
    DiffQrResult out;
    double dmax = 0, dmin = std::numeric_limits<double>::infinity();
    for (Index i = 0; i < k; ++i) {
        dmax = std::max(dmax, std::abs(r(i, i)));
        dmin = std::min(dmin, std::abs(r(i, i)));
    }
    out.ill_conditioned = !(dmin > 0) || dmax / dmin > 1e12;
    Mat qtdb = matmul_t(q, true, db, false);
    Mat y = qtdb;
    solve_upper_right(y, r);
    Mat domega(k, k);
    for (Index i = 1; i < k; ++i)
        for (Index j = 0; j < i; ++j) {
            domega(i, j) = y(i, j);
            domega(j, i) = -y(i, j);
        }
    out.dr = matmul(y - domega, r);
    for (Index j = 0; j < k; ++j)
        for (Index i = j + 1; i < k; ++i) out.dr(i, j) = 0.0;
    Mat resid = db - matmul(q, qtdb);
    solve_upper_right(resid, r);
    out.dq_span = matmul(q, domega);
    out.dq = out.dq_span + resid;
    return out;
}

namespace {
// sketch.cpp:115-126
void check_rank_fits(const ClusterTree& tree, Index k) {
    for (int l = 1; l <= tree.depth(); ++l) {
        const auto& kids = tree.level(l);
        for (size_t j = 0; j < tree.level(l - 1).size(); ++j) {
            Index m = std::min(kids[2 * j].size(), kids[2 * j + 1].size());
            if (k > m)
                throw std::invalid_argument("build_hodlr: rank " + std::to_string(k) +
                                            " exceeds block dimension at level " + std::to_string(l));
        }
    }
}
}  // namespace

// sketch.cpp:128-343
BuildResult build_impl(const CovarianceOracle& oracle, const ClusterTree& tree, Index k,
                       const SketchPlan& plan, bool with_deriv) {
    if (oracle.dim() != tree.size()) throw std::invalid_argument("build_hodlr: oracle dimension mismatch");
    if (!plan.dimensioned_for(tree, k))
        throw std::invalid_argument("build_hodlr: sketch plan not dimensioned for tree");
    check_rank_fits(tree, k);
    const Index n = tree.size();
    const int tau = tree.depth();
    const Index p = with_deriv ? oracle.num_params() : 0;
    BuildResult out;
    out.h = HodlrMatrix::zero(tree);
    out.deriv.assign(static_cast<size_t>(p), HodlrMatrix::zero(tree));

    for (int l = 1; l <= tau; ++l) {
        const auto& kids = tree.level(l);
        const Index nodes = Index(tree.level(l - 1).size());
        const Mat& rs = plan.level_sampler(l);
        Mat y = oracle.apply(rs) - out.h.matvec(rs);
        std::vector<Mat> dy(static_cast<size_t>(p));
        for (Index j = 0; j < p; ++j)
            dy[static_cast<size_t>(j)] = oracle.apply_derivative(int(j), rs) - out.deriv[static_cast<size_t>(j)].matvec(rs);

        std::vector<RangeResult> cap(static_cast<size_t>(nodes));
        std::vector<char> full_width(static_cast<size_t>(nodes), 0);
#pragma omp parallel for schedule(static)
        for (Index j = 0; j < nodes; ++j) {
            auto cl = kids[static_cast<size_t>(2 * j)];
            if (cl.size() == k) {
                cap[static_cast<size_t>(j)].q = Mat::identity(k, k);
                cap[static_cast<size_t>(j)].r = Mat(k, k);
                cap[static_cast<size_t>(j)].perm.resize(static_cast<size_t>(k));
                for (Index i = 0; i < k; ++i) cap[static_cast<size_t>(j)].perm[static_cast<size_t>(i)] = int(i);
                cap[static_cast<size_t>(j)].numeric_rank = k;
                full_width[static_cast<size_t>(j)] = 1;
            } else {
                cap[static_cast<size_t>(j)] = randomized_range(y.middle_rows(cl.lo, cl.size()), k);
            }
        }

        Mat s(n, k);
        for (Index j = 0; j < nodes; ++j) s.set_block(kids[static_cast<size_t>(2 * j)].lo, 0, cap[static_cast<size_t>(j)].q);
        Mat z = oracle.apply(s) - out.h.matvec(s);

        std::vector<Mat> q2(static_cast<size_t>(nodes));
        std::vector<Index> w2s(static_cast<size_t>(nodes), 0);
        Mat s2;
        Index w2max = 0;
        if (p > 0) {
            s2 = Mat(n, k * p);
#pragma omp parallel for schedule(static)
            for (Index j = 0; j < nodes; ++j) {
                if (full_width[static_cast<size_t>(j)]) continue;
                auto cl = kids[static_cast<size_t>(2 * j)];
                Mat resid(cl.size(), k * p);
                double presc = 0;
                for (Index param = 0; param < p; ++param) {
                    Mat blk = dy[static_cast<size_t>(param)].middle_rows(cl.lo, cl.size());
                    resid.set_block(0, param * k, blk);
                    presc = std::max(presc, blk.norm());
                }
                const Mat& q = cap[static_cast<size_t>(j)].q;
                for (int pass = 0; pass < 2; ++pass) resid = resid - matmul(q, matmul_t(q, true, resid, false));
                ColPivQR qr2;
                qr2.compute(resid);
                const double d0 = std::abs(qr2.qr(0, 0));
                const double floor_ = std::max(1e-10 * d0, 1e-12 * presc);
                const Index w2cap = std::min(resid.c, cl.size() - k);
                Index w2 = 0;
                while (w2 < w2cap && std::abs(qr2.qr(w2, w2)) > floor_) ++w2;
                w2s[static_cast<size_t>(j)] = w2;
                if (w2 > 0) q2[static_cast<size_t>(j)] = qr2.householder_q_thin(w2);
                if (w2 > 0 && g_q2_reorthogonalize) {  // device HG_Q2_REORTHOGONALIZED
                    Mat& b = q2[static_cast<size_t>(j)];
                    b = b - matmul(q, matmul_t(q, true, b, false));
                    for (Index c = 0; c < b.c; ++c) {
                        double nn = 0;
                        for (Index r = 0; r < b.r; ++r) nn += b(r, c) * b(r, c);
                        const double inv = nn > 0 ? 1.0 / std::sqrt(nn) : 0.0;
                        for (Index r = 0; r < b.r; ++r) b(r, c) *= inv;
                    }
                }
            }
            for (Index j = 0; j < nodes; ++j) {
                const Mat& b = q2[static_cast<size_t>(j)];
                if (b.c == 0) continue;
                s2.set_block(kids[static_cast<size_t>(2 * j)].lo, 0, b);
                w2max = std::max(w2max, b.c);
            }
        }

        std::vector<std::vector<Mat>> dqc(static_cast<size_t>(p)), dt(static_cast<size_t>(p)), dt2(static_cast<size_t>(p));
        std::vector<std::vector<Index>> rws(static_cast<size_t>(p), std::vector<Index>(static_cast<size_t>(nodes), 0));
        for (Index param = 0; param < p; ++param) {
            dqc[static_cast<size_t>(param)].resize(static_cast<size_t>(nodes));
            for (Index j = 0; j < nodes; ++j) {
                auto cl = kids[static_cast<size_t>(2 * j)];
                const RangeResult& c = cap[static_cast<size_t>(j)];
                const Index rr = c.numeric_rank;
                dqc[static_cast<size_t>(param)][static_cast<size_t>(j)] = Mat(cl.size(), k);
                if (rr == 0 || full_width[static_cast<size_t>(j)]) continue;
                Index rw = 0;
                while (rw < rr && std::abs(c.r(rw, rw)) > 1e-6 * std::abs(c.r(0, 0))) ++rw;
                rws[static_cast<size_t>(param)][static_cast<size_t>(j)] = rw;
                if (rw == 0) continue;
                Mat bp(cl.size(), rw), dbp(cl.size(), rw);
                for (Index i = 0; i < rw; ++i) {
                    Index pc = c.perm[static_cast<size_t>(i)];
                    for (Index t = 0; t < cl.size(); ++t) {
                        bp(t, i) = y(cl.lo + t, pc);
                        dbp(t, i) = dy[static_cast<size_t>(param)](cl.lo + t, pc);
                    }
                }
                DiffQrResult d = diff_qr(bp, dbp, c.q.left_cols(rw), c.r.block(0, 0, rw, rw));
                dqc[static_cast<size_t>(param)][static_cast<size_t>(j)].set_block(0, 0, d.dq_span);
                if (d.ill_conditioned)
                    out.warnings.push_back("ill-conditioned QR at level " + std::to_string(l) +
                                           " param " + std::to_string(param));
            }
            Mat ds(n, k);
            for (Index j = 0; j < nodes; ++j) ds.set_block(kids[static_cast<size_t>(2 * j)].lo, 0, dqc[static_cast<size_t>(param)][static_cast<size_t>(j)]);
            Mat dz = oracle.apply_derivative(int(param), s) - out.deriv[static_cast<size_t>(param)].matvec(s) +
                     oracle.apply(ds) - out.h.matvec(ds);
            dt[static_cast<size_t>(param)].resize(static_cast<size_t>(nodes));
            for (Index j = 0; j < nodes; ++j) {
                auto cr = kids[static_cast<size_t>(2 * j + 1)];
                dt[static_cast<size_t>(param)][static_cast<size_t>(j)] = dz.middle_rows(cr.lo, cr.size());
            }
            if (w2max > 0) {
                Mat probe2 = s2.left_cols(w2max);
                Mat dz2 = oracle.apply_derivative(int(param), probe2) - out.deriv[static_cast<size_t>(param)].matvec(probe2);
                dt2[static_cast<size_t>(param)].resize(static_cast<size_t>(nodes));
                for (Index j = 0; j < nodes; ++j) {
                    auto cr = kids[static_cast<size_t>(2 * j + 1)];
                    Index w2 = q2[static_cast<size_t>(j)].c;
                    if (w2 > 0) dt2[static_cast<size_t>(param)][static_cast<size_t>(j)] = dz2.block(cr.lo, 0, cr.size(), w2);
                }
            }
        }

        for (Index j = 0; j < nodes; ++j) {
            auto cr = kids[static_cast<size_t>(2 * j + 1)];
            Mat t = z.middle_rows(cr.lo, cr.size());
            out.h.upper(l, j) = LowRankBlock{cap[static_cast<size_t>(j)].q, t};
            for (Index param = 0; param < p; ++param) {
                LowRankBlock d = LowRankBlock::concat(LowRankBlock{dqc[static_cast<size_t>(param)][static_cast<size_t>(j)], t},
                                                      LowRankBlock{cap[static_cast<size_t>(j)].q, dt[static_cast<size_t>(param)][static_cast<size_t>(j)]});
                const Mat& b = q2[static_cast<size_t>(j)];
                if (b.c > 0) d = LowRankBlock::concat(d, LowRankBlock{b, dt2[static_cast<size_t>(param)][static_cast<size_t>(j)]});
                // device HG_COMPRESS_AT_LEVEL: compress at commit, so finer
                // levels peel against the compressed block
                out.deriv[static_cast<size_t>(param)].upper(l, j) = g_compress_at_level ? d.compressed(1e-13) : d;
            }
            BuildDecision dec;
            dec.level = l;
            dec.node = j;
            dec.numeric_rank = cap[static_cast<size_t>(j)].numeric_rank;
            dec.w2 = w2s[static_cast<size_t>(j)];
            for (Index param = 0; param < p; ++param) dec.rw.push_back(rws[static_cast<size_t>(param)][static_cast<size_t>(j)]);
            out.decisions.push_back(dec);
        }
    }

    const Mat& sl = plan.leaf_sampler();
    Mat y = oracle.apply(sl) - out.h.matvec(sl);
    for (Index b = 0; b < tree.num_leaves(); ++b) {
        auto r = tree.leaves()[static_cast<size_t>(b)];
        out.h.leaf(b) = y.block(r.lo, 0, r.size(), r.size());
    }
    for (Index param = 0; param < p; ++param) {
        Mat dyl = oracle.apply_derivative(int(param), sl) - out.deriv[static_cast<size_t>(param)].matvec(sl);
        for (Index b = 0; b < tree.num_leaves(); ++b) {
            auto r = tree.leaves()[static_cast<size_t>(b)];
            out.deriv[static_cast<size_t>(param)].leaf(b) = dyl.block(r.lo, 0, r.size(), r.size());
        }
    }
    for (Index param = 0; param < p && !g_compress_at_level; ++param)
        for (int l = 1; l <= tau; ++l) {
            const Index nodes = Index(tree.level(l - 1).size());
#pragma omp parallel for schedule(static)
            for (Index j = 0; j < nodes; ++j)
                out.deriv[static_cast<size_t>(param)].upper(l, j) = out.deriv[static_cast<size_t>(param)].upper(l, j).compressed(1e-13);
        }
    return out;
}

HodlrMatrix build_hodlr(const CovarianceOracle& oracle, const ClusterTree& tree, Index k,
                        const SketchPlan& plan) {
    return build_impl(oracle, tree, k, plan, false).h;
}

BuildResult build_hodlr_with_derivatives(const CovarianceOracle& oracle, const ClusterTree& tree,
                                         Index k, const SketchPlan& plan) {
    return build_impl(oracle, tree, k, plan, true);
}

// =========================================================== factorization
// factorization.cpp:7-18
void LeafFactor::compute(const Mat& a, bool prefer_llt) {
    mat_ = a;
    use_llt_ = false;
    if (prefer_llt) {
        llt_.compute(a);
        if (llt_.ok) {
            use_llt_ = true;
            return;
        }
    }
    lu_.compute(a);
}

// factorization.cpp:20-22
Mat LeafFactor::solve(const Mat& b) const { return use_llt_ ? llt_.solve(b) : lu_.solve(b); }

// factorization.cpp:28-44
double LeafFactor::logdet_positive() const {
    if (use_llt_) {
        double ld = 0;
        for (Index i = 0; i < mat_.r; ++i) ld += std::log(llt_.l(i, i));
        return 2.0 * ld;
    }
    double ld = 0, sign = lu_.det_p();
    for (Index i = 0; i < lu_.lu.r; ++i) {
        double d = lu_.lu(i, i);
        if (d < 0) sign = -sign;
        ld += std::log(std::abs(d));
    }
    if (sign <= 0) throw NotPositiveDefinite("leaf block has non-positive determinant");
    return ld;
}

namespace {
// factorization.cpp:48-58
double lu_log_abs_det(const PartialPivLU& lu, bool& positive) {
    double ld = 0, sign = lu.det_p();
    for (Index i = 0; i < lu.lu.r; ++i) {
        double d = lu.lu(i, i);
        if (d < 0) sign = -sign;
        ld += std::log(std::abs(d));
    }
    positive = sign > 0;
    return ld;
}
}  // namespace

// factorization.cpp:62-168
HodlrFactorization factorize(const HodlrMatrix& h, Orientation orient) {
    const ClusterTree& tree = h.tree();
    const int tau = h.depth();
    HodlrFactorization f;
    f.tree_ = tree;
    f.orient_ = orient;
    f.leaf_factors_.resize(static_cast<size_t>(h.num_leaves()));
#pragma omp parallel for schedule(static)
    for (Index b = 0; b < h.num_leaves(); ++b) f.leaf_factors_[static_cast<size_t>(b)].compute(h.leaf(b), h.symmetric());

    struct Work {
        Mat wbar, xbar, w, x;
    };
    std::vector<std::vector<Work>> work(static_cast<size_t>(tau));
    for (int l = 1; l <= tau; ++l) {
        const Index nodes = Index(tree.level(l - 1).size());
        work[static_cast<size_t>(l - 1)].resize(static_cast<size_t>(nodes));
        for (Index j = 0; j < nodes; ++j) {
            const LowRankBlock& blk = h.upper(l, j);
            Work& wk = work[static_cast<size_t>(l - 1)][static_cast<size_t>(j)];
            if (blk.empty()) {
                auto cl = tree.level(l)[static_cast<size_t>(2 * j)], cr = tree.level(l)[static_cast<size_t>(2 * j + 1)];
                wk.w = wk.wbar = Mat(cl.size(), 0);
                wk.x = wk.xbar = Mat(cr.size(), 0);
            } else {
                wk.w = wk.wbar = blk.left;
                wk.x = wk.xbar = blk.right;
            }
        }
    }
    auto leaf_solve_rows = [&](Mat& m, Index row_lo) {
        Index row_hi = row_lo + m.r;
        for (Index b = 0; b < h.num_leaves(); ++b) {
            auto r = tree.leaves()[static_cast<size_t>(b)];
            if (r.hi <= row_lo || r.lo >= row_hi) continue;
            m.set_block(r.lo - row_lo, 0, f.leaf_factors_[static_cast<size_t>(b)].solve(m.middle_rows(r.lo - row_lo, r.size())));
        }
    };
    for (int l = 1; l <= tau; ++l) {
        const auto& kids = tree.level(l);
        const Index nodes = Index(tree.level(l - 1).size());
#pragma omp parallel for schedule(static)
        for (Index j = 0; j < nodes; ++j) {
            leaf_solve_rows(work[static_cast<size_t>(l - 1)][static_cast<size_t>(j)].wbar, kids[static_cast<size_t>(2 * j)].lo);
            leaf_solve_rows(work[static_cast<size_t>(l - 1)][static_cast<size_t>(j)].xbar, kids[static_cast<size_t>(2 * j + 1)].lo);
        }
    }
    f.levels_.resize(static_cast<size_t>(tau));
    for (int i = tau; i >= 1; --i) {
        const auto& nodes = tree.level(i - 1);
        auto& lev = f.levels_[static_cast<size_t>(i - 1)];
        lev.resize(nodes.size());
        for (size_t j = 0; j < nodes.size(); ++j) {
            const Work& wk = work[static_cast<size_t>(i - 1)][j];
            const Index m1 = wk.wbar.r, m2 = wk.xbar.r, r = wk.w.c;
            auto& blk = lev[j];
            blk.u = Mat(m1 + m2, 2 * r);
            blk.u.set_block(0, 0, wk.wbar);
            blk.u.set_block(m1, r, wk.xbar);
            blk.v = Mat(m1 + m2, 2 * r);
            blk.v.set_block(0, r, wk.w);
            blk.v.set_block(m1, 0, wk.x);
            Mat cap = Mat::identity(2 * r, 2 * r) + matmul_t(blk.v, true, blk.u, false);
            blk.cap.compute(cap);
            blk.logdet_cap = lu_log_abs_det(blk.cap, blk.cap_positive);
        }
        for (int l = 1; l < i; ++l) {
            const int shift = (i - 1) - l;
            const Index ncoarse = Index(tree.level(l - 1).size());
#pragma omp parallel for schedule(static)
            for (Index j = 0; j < ncoarse; ++j) {
                auto apply_inv = [&](Mat& m, Index child_node) {
                    Index first = child_node << shift, count = Index{1} << shift;
                    Index row_lo = tree.level(i - 1)[static_cast<size_t>(first)].lo;
                    for (Index b = first; b < first + count; ++b) {
                        const auto& blk = lev[static_cast<size_t>(b)];
                        auto rng = tree.level(i - 1)[static_cast<size_t>(b)];
                        if (blk.u.c == 0) continue;
                        Mat rows = m.middle_rows(rng.lo - row_lo, rng.size());
                        Mat upd = matmul(blk.u, blk.cap.solve(matmul_t(blk.v, true, rows, false)));
                        m.add_block(rng.lo - row_lo, 0, upd, -1.0);
                    }
                };
                apply_inv(work[static_cast<size_t>(l - 1)][static_cast<size_t>(j)].wbar, 2 * j);
                apply_inv(work[static_cast<size_t>(l - 1)][static_cast<size_t>(j)].xbar, 2 * j + 1);
            }
        }
    }
    return f;
}

// factorization.cpp:170-208
Mat HodlrFactorization::solve(const Mat& b) const {
    if (b.r != size()) throw std::invalid_argument("solve: dimension mismatch");
    Mat y = b;
    auto leaf_solve_all = [&]() {
#pragma omp parallel for schedule(static)
        for (Index i = 0; i < num_leaves(); ++i) {
            auto r = tree_.leaves()[static_cast<size_t>(i)];
            y.set_block(r.lo, 0, leaf_factors_[static_cast<size_t>(i)].solve(y.middle_rows(r.lo, r.size())));
        }
    };
    auto apply_level_inverse = [&](int i, bool transposed) {
        const auto& nodes = tree_.level(i - 1);
        const auto& lev = levels_[static_cast<size_t>(i - 1)];
#pragma omp parallel for schedule(static)
        for (Index j = 0; j < Index(nodes.size()); ++j) {
            const LevelBlock& blk = lev[static_cast<size_t>(j)];
            if (blk.u.c == 0) continue;
            Mat rows = y.middle_rows(nodes[static_cast<size_t>(j)].lo, nodes[static_cast<size_t>(j)].size());
            Mat upd;
            if (!transposed)
                upd = matmul(blk.u, blk.cap.solve(matmul_t(blk.v, true, rows, false)));
            else
                upd = matmul(blk.v, blk.cap.solve_transpose(matmul_t(blk.u, true, rows, false)));
            y.add_block(nodes[static_cast<size_t>(j)].lo, 0, upd, -1.0);
        }
    };
    if (orient_ == Orientation::Right) {
        leaf_solve_all();
        for (int i = depth(); i >= 1; --i) apply_level_inverse(i, false);
    } else {
        for (int i = 1; i <= depth(); ++i) apply_level_inverse(i, true);
        leaf_solve_all();
    }
    return y;
}

// factorization.cpp:214-224
double HodlrFactorization::logdet() const {
    double ld = 0;
    for (const auto& lf : leaf_factors_) ld += lf.logdet_positive();
    for (const auto& lev : levels_)
        for (const auto& blk : lev) {
            if (!blk.cap_positive) throw NotPositiveDefinite("capacitance has non-positive determinant");
            ld += blk.logdet_cap;
        }
    return ld;
}

// ============================================================ trace algebra
// product_rep.cpp:9-22
Mat ProductRep::densify() const {
    Mat a = base.densify();
    const ClusterTree& tree = base.tree();
    for (size_t i = 0; i < corrections.size(); ++i) {
        const auto& nodes = tree.level(int(i));
        for (size_t j = 0; j < corrections[i].size(); ++j) {
            const CorrBlock& c = corrections[i][j];
            if (c.u.c == 0) continue;
            a.add_block(nodes[j].lo, nodes[j].lo, matmul_t(c.u, false, c.v, true));
        }
    }
    return a;
}

bool g_solve_association = false;
void set_solve_association(bool on) { g_solve_association = on; }

namespace {
struct LevelFactor {
    std::vector<Mat> p, q;
    const std::vector<HodlrFactorization::LevelBlock>* blocks = nullptr;
};

// product_rep.cpp:32-45
void apply_blocks_to_rows(const ClusterTree& tree, const LevelFactor& lf, int df, Mat& m, int d,
                          Index node) {
    const int shift = df - d;
    const Index first = node << shift, count = Index{1} << shift;
    const Index row0 = tree.level(d)[static_cast<size_t>(node)].lo;
    for (Index b = first; b < first + count; ++b) {
        if (lf.p[static_cast<size_t>(b)].c == 0) continue;
        auto rng = tree.level(df)[static_cast<size_t>(b)];
        Mat rows = m.middle_rows(rng.lo - row0, rng.size());
        if (lf.blocks && g_solve_association) {
            const auto& blk = (*lf.blocks)[static_cast<size_t>(b)];
            Mat t = blk.cap.solve_transpose(matmul_t(blk.u, true, rows, false));
            m.add_block(rng.lo - row0, 0, matmul(blk.v, t), -1.0);
            continue;
        }
        m.add_block(rng.lo - row0, 0, matmul(lf.p[static_cast<size_t>(b)], matmul_t(lf.q[static_cast<size_t>(b)], true, rows, false)));
    }
}

// product_rep.cpp:47-155
ProductRep pipeline(const HodlrFactorization& f, const HodlrMatrix& b, bool inverse) {
    if (!f.tree().same_structure(b.tree()))
        throw std::invalid_argument("product pipeline: tree structure mismatch");
    if (!inverse && f.orientation() != Orientation::Right)
        throw std::invalid_argument("multiply: factorization must be Right-oriented");
    if (inverse && f.orientation() != Orientation::Left)
        throw std::invalid_argument("solve_multiply: factorization must be Left-oriented");
    const ClusterTree& tree = f.tree();
    const int tau = f.depth();
    ProductRep rep;
    rep.base = b;
    rep.base.make_asymmetric();
    rep.corrections.resize(static_cast<size_t>(tau));
    for (int i = 1; i <= tau; ++i) {
        const auto& nodes = tree.level(i - 1);
        const auto& lev = f.level(i);
        LevelFactor lf;
        if (inverse) lf.blocks = &lev;
        lf.p.resize(nodes.size());
        lf.q.resize(nodes.size());
        for (size_t j = 0; j < nodes.size(); ++j) {
            const auto& blk = lev[j];
            if (blk.u.c == 0) {
                lf.p[j] = Mat(nodes[j].size(), 0);
                lf.q[j] = Mat(nodes[j].size(), 0);
            } else if (inverse) {
                lf.p[j] = -1.0 * blk.cap.solve(blk.v.transpose()).transpose();
                lf.q[j] = blk.u;
            } else {
                lf.p[j] = blk.u;
                lf.q[j] = blk.v;
            }
        }
        for (int m = 1; m < i; ++m)
            for (size_t j = 0; j < rep.corrections[static_cast<size_t>(m - 1)].size(); ++j) {
                auto& c = rep.corrections[static_cast<size_t>(m - 1)][j];
                if (c.u.c == 0) continue;
                apply_blocks_to_rows(tree, lf, i - 1, c.u, m - 1, Index(j));
            }
        for (int m = 1; m < i; ++m) {
            const Index coarse = Index(tree.level(m - 1).size());
            for (Index j = 0; j < coarse; ++j) {
                LowRankBlock& up = rep.base.upper(m, j);
                if (!up.empty()) apply_blocks_to_rows(tree, lf, i - 1, up.left, m, 2 * j);
                LowRankBlock& lo = rep.base.lower(m, j);
                if (!lo.empty()) apply_blocks_to_rows(tree, lf, i - 1, lo.left, m, 2 * j + 1);
            }
        }
        rep.corrections[static_cast<size_t>(i - 1)].resize(nodes.size());
        for (size_t j = 0; j < nodes.size(); ++j) {
            auto& c = rep.corrections[static_cast<size_t>(i - 1)][j];
            if (lf.p[j].c == 0) {
                c.u = Mat(nodes[j].size(), 0);
                c.v = Mat(nodes[j].size(), 0);
                continue;
            }
            c.u = lf.p[j];
            c.v = rep.base.sub_matvec(i - 1, Index(j), lf.q[j], true);
        }
    }
    auto apply_leaf_rows = [&](Mat& m, int d, Index node) {
        const int shift = tau - d;
        const Index first = node << shift, count = Index{1} << shift;
        const Index row0 = tree.level(d)[static_cast<size_t>(node)].lo;
        for (Index lb = first; lb < first + count; ++lb) {
            auto rng = tree.leaves()[static_cast<size_t>(lb)];
            Mat rows = m.middle_rows(rng.lo - row0, rng.size());
            m.set_block(rng.lo - row0, 0, inverse ? f.leaf(lb).solve(rows) : f.leaf(lb).multiply(rows));
        }
    };
    for (int i = 1; i <= tau; ++i)
        for (size_t j = 0; j < rep.corrections[static_cast<size_t>(i - 1)].size(); ++j) {
            auto& c = rep.corrections[static_cast<size_t>(i - 1)][j];
            if (c.u.c != 0) apply_leaf_rows(c.u, i - 1, Index(j));
        }
    for (int m = 1; m <= tau; ++m) {
        const Index coarse = Index(tree.level(m - 1).size());
        for (Index j = 0; j < coarse; ++j) {
            LowRankBlock& up = rep.base.upper(m, j);
            if (!up.empty()) apply_leaf_rows(up.left, m, 2 * j);
            LowRankBlock& lo = rep.base.lower(m, j);
            if (!lo.empty()) apply_leaf_rows(lo.left, m, 2 * j + 1);
        }
    }
    for (Index lb = 0; lb < rep.base.num_leaves(); ++lb)
        rep.base.leaf(lb) = inverse ? f.leaf(lb).solve(rep.base.leaf(lb)) : f.leaf(lb).multiply(rep.base.leaf(lb));
    return rep;
}

// product_rep.cpp:159-176
double pair_term(const ClusterTree& tree, const std::vector<ProductRep::CorrBlock>& coarse, int ci,
                 const std::vector<ProductRep::CorrBlock>& fine, int fi) {
    const int dc = ci - 1, df = fi - 1, shift = df - dc;
    double s = 0;
    for (size_t b = 0; b < fine.size(); ++b) {
        const auto& fb = fine[b];
        if (fb.u.c == 0) continue;
        const Index big = Index(b) >> shift;
        const auto& cb = coarse[static_cast<size_t>(big)];
        if (cb.u.c == 0) continue;
        const Index off = tree.level(df)[b].lo - tree.level(dc)[static_cast<size_t>(big)].lo;
        const Index sz = tree.level(df)[b].size();
        Mat g1 = matmul_t(cb.v.middle_rows(off, sz), true, fb.u, false);
        Mat g2 = matmul_t(fb.v, true, cb.u.middle_rows(off, sz), false);
        double t = 0;
        for (Index c = 0; c < g1.c; ++c)
            for (Index r = 0; r < g1.r; ++r) t += g1(r, c) * g2(c, r);
        s += t;
    }
    return s;
}
}  // namespace

ProductRep multiply(const HodlrFactorization& f, const HodlrMatrix& b) { return pipeline(f, b, false); }
ProductRep solve_multiply(const HodlrFactorization& f, const HodlrMatrix& b) { return pipeline(f, b, true); }

// product_rep.cpp:188-194
double trace_product_rep(const ProductRep& p) {
    double t = p.base.trace();
    for (const auto& lev : p.corrections)
        for (const auto& c : lev)
            if (c.u.c != 0) t += dot_sum(c.u, c.v);
    return t;
}

// product_rep.cpp:196-202
double trace_solve(const HodlrFactorization& f_left, const HodlrMatrix& b) {
    return trace_product_rep(solve_multiply(f_left, b));
}
double trace_solve(const HodlrMatrix& a, const HodlrMatrix& b) {
    return trace_solve(factorize(a, Orientation::Left), b);
}

// product_rep.cpp:204-235
double trace_pair(const ProductRep& pb, const ProductRep& pd) {
    const ClusterTree& tree = pb.base.tree();
    const int tau = pb.base.depth();
    double t = HodlrMatrix::trace_product(pb.base, pd.base);
    auto cross = [&](const HodlrMatrix& h, const std::vector<std::vector<ProductRep::CorrBlock>>& corr) {
        double s = 0;
        for (int i = 1; i <= tau; ++i)
            for (size_t j = 0; j < corr[static_cast<size_t>(i - 1)].size(); ++j) {
                const auto& c = corr[static_cast<size_t>(i - 1)][j];
                if (c.u.c == 0) continue;
                Mat hu = h.sub_matvec(i - 1, Index(j), c.u);
                s += dot_sum(c.v, hu);
            }
        return s;
    };
    t += cross(pb.base, pd.corrections);
    t += cross(pd.base, pb.corrections);
    for (int i = 1; i <= tau; ++i)
        for (int j = 1; j <= tau; ++j) {
            if (i <= j)
                t += pair_term(tree, pb.corrections[static_cast<size_t>(i - 1)], i, pd.corrections[static_cast<size_t>(j - 1)], j);
            else
                t += pair_term(tree, pd.corrections[static_cast<size_t>(j - 1)], j, pb.corrections[static_cast<size_t>(i - 1)], i);
        }
    return t;
}

// product_rep.cpp:237-245
double trace_quad(const HodlrFactorization& fa, const HodlrMatrix& b, const HodlrFactorization& fc,
                  const HodlrMatrix& d) {
    return trace_pair(solve_multiply(fa, b), solve_multiply(fc, d));
}
double trace_quad(const HodlrMatrix& a, const HodlrMatrix& b, const HodlrMatrix& c, const HodlrMatrix& d) {
    return trace_quad(factorize(a, Orientation::Left), b, factorize(c, Orientation::Left), d);
}

// =================================================================== mle
namespace {
constexpr double kLog2Pi = 1.8378770664093454836;
Mat residual(const Mat& y, const Mat& ybar) {
    if (ybar.r == 0) return y;
    if (ybar.r != y.r) throw std::invalid_argument("mean length mismatch");
    return y - ybar;
}
}  // namespace

// mle.cpp:25-30
double log_likelihood(const HodlrFactorization& f, const Mat& y, const Mat& ybar) {
    Mat r = residual(y, ybar);
    if (r.r != f.size()) throw std::invalid_argument("log_likelihood: length mismatch");
    return -0.5 * double(f.size()) * kLog2Pi - 0.5 * f.logdet() - 0.5 * dot_sum(r, f.solve(r));
}

// mle.cpp:32-41
std::vector<double> score(const HodlrFactorization& f, const std::vector<HodlrMatrix>& deriv,
                          const Mat& y, const Mat& ybar) {
    Mat r = residual(y, ybar);
    Mat w = f.solve(r);
    std::vector<double> s(deriv.size());
    for (size_t j = 0; j < deriv.size(); ++j)
        s[j] = -0.5 * trace_solve(f, deriv[j]) + 0.5 * dot_sum(w, deriv[j].matvec(w));
    return s;
}

// mle.cpp:56-75
HutchinsonResult hutchinson_trace(const HodlrFactorization& f, const HodlrMatrix& b, int n_samples,
                                  std::uint64_t seed) {
    if (n_samples < 2) throw std::invalid_argument("hutchinson_trace: need >= 2 samples");
    std::mt19937_64 rng(seed);
    std::bernoulli_distribution coin(0.5);
    const Index n = f.size();
    double sum = 0, sumsq = 0;
    for (int s = 0; s < n_samples; ++s) {
        Mat z(n, 1);
        for (Index i = 0; i < n; ++i) z(i, 0) = coin(rng) ? 1.0 : -1.0;
        const double v = dot_sum(z, f.solve(b.matvec(z)));
        sum += v;
        sumsq += v * v;
    }
    HutchinsonResult out;
    out.estimate = sum / n_samples;
    const double var = (sumsq - sum * sum / n_samples) / (n_samples - 1);
    out.std_error = std::sqrt(std::max(var, 0.0) / n_samples);
    return out;
}

// mle.cpp:43-54
Mat fisher_information(const HodlrFactorization& f, const std::vector<HodlrMatrix>& deriv, bool cache) {
    const Index p = Index(deriv.size());
    Mat info(p, p);
    std::vector<ProductRep> reps;
    if (cache)
        for (const auto& d : deriv) reps.push_back(solve_multiply(f, d));
    for (Index i = 0; i < p; ++i)
        for (Index j = i; j < p; ++j) {
            double t = cache ? 0.5 * trace_pair(reps[static_cast<size_t>(i)], reps[static_cast<size_t>(j)])
                             : 0.5 * trace_quad(f, deriv[static_cast<size_t>(i)], f, deriv[static_cast<size_t>(j)]);
            info(i, j) = t;
            info(j, i) = t;
        }
    Mat out(p, p);
    for (Index i = 0; i < p; ++i)
        for (Index j = 0; j < p; ++j) out(i, j) = 0.5 * (info(i, j) + info(j, i));
    return out;
}

}  // namespace oracle
