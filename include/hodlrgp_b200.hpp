// hodlrgp_b200.hpp — C++ drop-in for the reference's hot-path API
// (/root/reference/proj/include/hodlrgp/*.hpp) over the C ABI of
// include/hodlrgp_b200.h. Header-only RAII layer: every numerical call runs
// on the GPU through libhodlrgp_b200.so; matrices cross the boundary as
// Eigen::MatrixXd / VectorXd exactly as in the reference signatures (the
// reference's callers already depend on Eigen).
//
// Names, argument meaning and exceptions follow the reference:
//   cluster_tree.hpp:24-71  ClusterTree, tree_depth, build_kd_ordering
//   hodlr_matrix.hpp:48-106 HodlrMatrix (zero, identity, random_spd,
//                           random_symmetric, matvec, sub_matvec, trace,
//                           densify, trace_product, make_asymmetric)
//   oracle.hpp:15-143       CovarianceOracle (device oracles + a host-model
//                           adapter), PermutedOracle, DenseMatrixOracle
//   sketch.hpp:17-85        SketchPlan, build_hodlr, build_hodlr_with_derivatives,
//                           BuildResult
//   factorization.hpp:14-82 NotPositiveDefinite, Orientation, factorize,
//                           HodlrFactorization::{solve, logdet}
//   product_rep.hpp:14-55   ProductRep, multiply, solve_multiply,
//                           trace_product_rep, trace_pair, trace_solve (2),
//                           trace_quad (2)
//   mle.hpp:16-26           log_likelihood, score, fisher_information
// Status codes map back to the reference exception types (HG_NOT_SPD ->
// NotPositiveDefinite, HG_EINVAL -> std::invalid_argument, HG_ELENGTH ->
// std::length_error, HG_ELOGIC -> std::logic_error, else std::runtime_error).
//
// Objects are handles with value semantics (copying a HodlrMatrix deep-copies
// its device storage, like the reference's value types). Everything runs on
// one context (device 0 and its own stream unless set_default_context() is
// called first). Define HODLRGP_B200_AS_HODLRGP to make these names visible
// as hodlrgp::... for unchanged caller code.
#pragma once

#include <Eigen/Dense>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hodlrgp_b200.h"

namespace hodlrgp_b200 {

using Index = std::int64_t;

// ------------------------------------------------------------- errors
struct NotPositiveDefinite : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(hg_status s) {
    if (s == HG_OK) return;
    const std::string msg = hg_last_error();
    switch (s) {
        case HG_NOT_SPD: throw NotPositiveDefinite(msg);
        case HG_EINVAL: throw std::invalid_argument(msg);
        case HG_ELENGTH: throw std::length_error(msg);
        case HG_ELOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

// ------------------------------------------------------------ context
class Context {
public:
    explicit Context(int device = 0, void* stream = nullptr) {
        hg_ctx_t c = nullptr;
        check(hg_ctx_create(device, stream, &c));
        c_.reset(c, [](hg_ctx_t x) { hg_ctx_destroy(x); });
    }
    hg_ctx_t get() const { return c_.get(); }
    void synchronize() const { check(hg_ctx_synchronize(get())); }
    void set_option(int option, int value) const { check(hg_ctx_set_option(get(), option, value)); }

private:
    std::shared_ptr<hg_ctx_s> c_;
};

inline std::shared_ptr<Context>& default_context_slot() {
    static thread_local std::shared_ptr<Context> c;
    return c;
}
inline const Context& default_context() {
    auto& c = default_context_slot();
    if (!c) c = std::make_shared<Context>(0);
    return *c;
}
inline void set_default_context(std::shared_ptr<Context> c) { default_context_slot() = std::move(c); }
inline hg_ctx_t ctx() { return default_context().get(); }

// ------------------------------------------------------- cluster tree
/// cluster_tree.hpp:24-51 — uniform binary tree, left child ceil(len/2).
class ClusterTree {
public:
    struct Range {
        Index lo = 0;
        Index hi = 0;
        Index size() const { return hi - lo; }
    };
    ClusterTree() = default;
    ClusterTree(Index n, int tau) : n_(n), tau_(tau) {
        std::vector<int64_t> lohi(2 * ((std::size_t(1) << (tau + 1)) - 1));
        check(hg_tree_ranges(n, tau, lohi.data()));
        levels_.resize(static_cast<std::size_t>(tau + 1));
        std::size_t o = 0;
        for (int d = 0; d <= tau; ++d)
            for (Index j = 0; j < (Index{1} << d); ++j, o += 2) levels_[static_cast<std::size_t>(d)].push_back({lohi[o], lohi[o + 1]});
    }
    Index size() const { return n_; }
    int depth() const { return tau_; }
    const std::vector<Range>& level(int d) const { return levels_[static_cast<std::size_t>(d)]; }
    const std::vector<Range>& leaves() const { return levels_[static_cast<std::size_t>(tau_)]; }
    Index num_leaves() const { return Index(leaves().size()); }
    Index max_leaf_size() const {
        Index m = 0;
        for (const Range& r : leaves()) m = std::max(m, r.size());
        return m;
    }
    bool same_structure(const ClusterTree& o) const { return n_ == o.n_ && tau_ == o.tau_; }

private:
    Index n_ = 0;
    int tau_ = 0;
    std::vector<std::vector<Range>> levels_;
};

/// cluster_tree.cpp:34-38
inline int tree_depth(Index n, Index leaf_min, Index leaf_max) { return hg_tree_depth(n, leaf_min, leaf_max); }

struct PointSet {
    Eigen::MatrixXd coords;  // n x d, d in {1, 2}
    Index size() const { return coords.rows(); }
    int dim() const { return static_cast<int>(coords.cols()); }
};

struct KdOrdering {
    std::vector<Index> perm;  // perm[original] = reordered position
    std::vector<Index> inv;   // inv[reordered] = original index
    ClusterTree tree;
    Eigen::MatrixXd reordered_coords;
};

/// cluster_tree.cpp:40-90
inline KdOrdering build_kd_ordering(const PointSet& points, Index leaf_min, Index leaf_max) {
    const Index n = points.size();
    const int d = points.dim();
    Eigen::MatrixXd c = points.coords;
    std::vector<int64_t> perm(static_cast<std::size_t>(n)), inv(static_cast<std::size_t>(n));
    int tau = 0;
    check(hg_kd_ordering(n, d, c.data(), leaf_min, leaf_max, perm.data(), inv.data(), &tau));
    KdOrdering out;
    out.perm.assign(perm.begin(), perm.end());
    out.inv.assign(inv.begin(), inv.end());
    out.tree = ClusterTree(n, tau);
    out.reordered_coords = Eigen::MatrixXd(n, d);
    for (Index pos = 0; pos < n; ++pos)
        for (int a = 0; a < d; ++a) out.reordered_coords(pos, a) = c(out.inv[static_cast<std::size_t>(pos)], a);
    return out;
}

// -------------------------------------------------------------- HODLR
enum class Orientation { Right = HG_RIGHT, Left = HG_LEFT };

class HodlrMatrix {
public:
    HodlrMatrix() = default;
    /// Adopt a handle from the C ABI (hg_build_h, hg_hodlr_import, ...).
    explicit HodlrMatrix(hg_hodlr_t h) : h_(h, [](hg_hodlr_t x) { hg_hodlr_free(x); }) { refresh(); }
    HodlrMatrix(const HodlrMatrix& o) {
        if (o.h_) {
            hg_hodlr_t c = nullptr;
            check(hg_hodlr_copy(ctx(), o.h_.get(), &c));
            *this = HodlrMatrix(c);
        }
    }
    HodlrMatrix(HodlrMatrix&&) = default;
    HodlrMatrix& operator=(const HodlrMatrix& o) {
        if (this != &o) *this = HodlrMatrix(o);
        return *this;
    }
    HodlrMatrix& operator=(HodlrMatrix&&) = default;

    /// hodlr_matrix.cpp:68-88, :162-172
    static HodlrMatrix zero(const ClusterTree& t, bool symmetric = true) {
        hg_hodlr_t h = nullptr;
        check(hg_hodlr_zero(ctx(), t.size(), t.depth(), symmetric ? 1 : 0, &h));
        return HodlrMatrix(h);
    }
    static HodlrMatrix identity(const ClusterTree& t) {
        hg_hodlr_t h = nullptr;
        check(hg_hodlr_identity(ctx(), t.size(), t.depth(), &h));
        return HodlrMatrix(h);
    }
    static HodlrMatrix random_spd(const ClusterTree& t, Index k, std::uint64_t seed) {
        hg_hodlr_t h = nullptr;
        check(hg_hodlr_random(ctx(), t.size(), t.depth(), k, seed, 1, &h));
        return HodlrMatrix(h);
    }
    static HodlrMatrix random_symmetric(const ClusterTree& t, Index k, std::uint64_t seed) {
        hg_hodlr_t h = nullptr;
        check(hg_hodlr_random(ctx(), t.size(), t.depth(), k, seed, 0, &h));
        return HodlrMatrix(h);
    }

    const ClusterTree& tree() const { return tree_; }
    Index size() const { return tree_.size(); }
    int depth() const { return tree_.depth(); }
    bool symmetric() const { return sym_; }
    hg_hodlr_t handle() const { return h_.get(); }

    void make_asymmetric() {
        check(hg_hodlr_make_asymmetric(ctx(), h_.get()));
        sym_ = false;
    }

    /// hodlr_matrix.cpp:198-226
    Eigen::MatrixXd matvec(const Eigen::MatrixXd& x) const {
        if (x.rows() != size()) throw std::invalid_argument("matvec: dimension mismatch");
        Eigen::MatrixXd xc = x, y(x.rows(), x.cols());
        check(hg_hodlr_matvec(ctx(), h_.get(), xc.data(), xc.rows(), xc.cols(), y.data(), y.rows(), HG_HOST));
        return y;
    }
    Eigen::VectorXd matvec(const Eigen::VectorXd& x) const {
        return Eigen::VectorXd(matvec(Eigen::MatrixXd(x)));
    }
    /// hodlr_matrix.cpp:228-265
    Eigen::MatrixXd sub_matvec(int d, Index node, const Eigen::MatrixXd& x, bool transpose = false) const {
        Eigen::MatrixXd xc = x, y(x.rows(), x.cols());
        check(hg_hodlr_sub_matvec(ctx(), h_.get(), d, node, xc.data(), xc.rows(), xc.cols(), transpose ? 1 : 0,
                                  y.data(), y.rows(), HG_HOST));
        return y;
    }
    double trace() const {
        double t = 0;
        check(hg_hodlr_trace(ctx(), h_.get(), &t));
        return t;
    }
    /// hodlr_matrix.cpp:273-292 (guard 2^14)
    Eigen::MatrixXd densify() const {
        if (size() > (Index{1} << 14)) throw std::length_error("densify: matrix too large");
        Eigen::MatrixXd a = Eigen::MatrixXd::Identity(size(), size());
        return matvec(a);
    }
    /// hodlr_matrix.cpp:294-318
    static double trace_product(const HodlrMatrix& a, const HodlrMatrix& b) {
        double t = 0;
        check(hg_trace_product(ctx(), a.h_.get(), b.h_.get(), &t));
        return t;
    }

private:
    void refresh() {
        int64_t n = 0;
        int tau = 0, sym = 0;
        check(hg_hodlr_info(h_.get(), &n, &tau, &sym, nullptr));
        tree_ = ClusterTree(n, tau);
        sym_ = sym != 0;
    }
    std::shared_ptr<hg_hodlr_s> h_;
    ClusterTree tree_;
    bool sym_ = true;
};

// ------------------------------------------------------ factorization
class HodlrFactorization {
public:
    HodlrFactorization() = default;
    explicit HodlrFactorization(hg_factor_t f, const ClusterTree& t, Orientation o)
        : f_(f, [](hg_factor_t x) { hg_factor_free(x); }), tree_(t), orient_(o) {}
    const ClusterTree& tree() const { return tree_; }
    Orientation orientation() const { return orient_; }
    int depth() const { return tree_.depth(); }
    Index size() const { return tree_.size(); }
    hg_factor_t handle() const { return f_.get(); }
    /// factorization.cpp:170-212
    Eigen::MatrixXd solve(const Eigen::MatrixXd& b) const {
        if (b.rows() != size()) throw std::invalid_argument("solve: dimension mismatch");
        Eigen::MatrixXd bc = b, x(b.rows(), b.cols());
        check(hg_factor_solve(ctx(), f_.get(), bc.data(), bc.rows(), bc.cols(), x.data(), x.rows(), HG_HOST));
        return x;
    }
    Eigen::VectorXd solve(const Eigen::VectorXd& b) const { return Eigen::VectorXd(solve(Eigen::MatrixXd(b))); }
    /// factorization.cpp:214-224 (throws NotPositiveDefinite)
    double logdet() const {
        double ld = 0;
        check(hg_factor_logdet(ctx(), f_.get(), &ld));
        return ld;
    }

private:
    std::shared_ptr<hg_factor_s> f_;
    ClusterTree tree_;
    Orientation orient_ = Orientation::Right;
};

/// factorization.cpp:62-168
inline HodlrFactorization factorize(const HodlrMatrix& h, Orientation orient = Orientation::Right) {
    hg_factor_t f = nullptr;
    check(hg_factorize(ctx(), h.handle(), static_cast<int>(orient), &f));
    return HodlrFactorization(f, h.tree(), orient);
}

// -------------------------------------------------------- trace algebra
class ProductRep {
public:
    ProductRep() = default;
    ProductRep(hg_prodrep_t p, Index n) : p_(p, [](hg_prodrep_t x) { hg_prodrep_free(x); }), n_(n) {}
    Index size() const { return n_; }
    hg_prodrep_t handle() const { return p_.get(); }
    /// product_rep.cpp:9-22 (guard 2^14)
    Eigen::MatrixXd densify() const {
        Eigen::MatrixXd a(n_, n_);
        check(hg_prodrep_densify(ctx(), p_.get(), a.data()));
        return a;
    }

private:
    std::shared_ptr<hg_prodrep_s> p_;
    Index n_ = 0;
};

/// product_rep.cpp:180-186
inline ProductRep multiply(const HodlrFactorization& f, const HodlrMatrix& b) {
    hg_prodrep_t p = nullptr;
    check(hg_multiply(ctx(), f.handle(), b.handle(), &p));
    return ProductRep(p, b.size());
}
inline ProductRep solve_multiply(const HodlrFactorization& f, const HodlrMatrix& b) {
    hg_prodrep_t p = nullptr;
    check(hg_solve_multiply(ctx(), f.handle(), b.handle(), &p));
    return ProductRep(p, b.size());
}
/// product_rep.cpp:188-245
inline double trace_product_rep(const ProductRep& p) {
    double t = 0;
    check(hg_trace_product_rep(ctx(), p.handle(), &t));
    return t;
}
inline double trace_pair(const ProductRep& p, const ProductRep& q) {
    double t = 0;
    check(hg_trace_pair(ctx(), p.handle(), q.handle(), &t));
    return t;
}
inline double trace_solve(const HodlrFactorization& f_left, const HodlrMatrix& b) {
    double t = 0;
    check(hg_trace_solve(ctx(), f_left.handle(), b.handle(), &t));
    return t;
}
inline double trace_solve(const HodlrMatrix& a, const HodlrMatrix& b) {
    return trace_solve(factorize(a, Orientation::Left), b);
}
/// mle.hpp:28-34
struct HutchinsonResult {
    double estimate = 0;
    double std_error = 0;
};
inline HutchinsonResult hutchinson_trace(const HodlrFactorization& f, const HodlrMatrix& b, int n_samples,
                                         std::uint64_t seed) {
    HutchinsonResult r;
    check(hg_hutchinson_trace(ctx(), f.handle(), b.handle(), n_samples, seed, &r.estimate, &r.std_error));
    return r;
}
inline double trace_quad(const HodlrFactorization& fa, const HodlrMatrix& b, const HodlrFactorization& fc,
                         const HodlrMatrix& d) {
    double t = 0;
    check(hg_trace_quad(ctx(), fa.handle(), b.handle(), fc.handle(), d.handle(), &t));
    return t;
}
inline double trace_quad(const HodlrMatrix& a, const HodlrMatrix& b, const HodlrMatrix& c, const HodlrMatrix& d) {
    return trace_quad(factorize(a, Orientation::Left), b, factorize(c, Orientation::Left), d);
}

// ------------------------------------------------------------ oracles
/// oracle.hpp:15-52. Concrete forward models run on the device; a host model
/// (the reference's subclassing style) plugs in through HostCovarianceOracle.
class CovarianceOracle {
public:
    virtual ~CovarianceOracle() = default;
    Index dim() const { return n_; }
    Index num_params() const { return p_; }
    Eigen::VectorXd parameters() const { return theta_; }
    virtual void set_parameters(const Eigen::VectorXd& theta) {
        theta_ = theta;
        Eigen::VectorXd t = theta;
        check(hg_oracle_set_parameters(o_.get(), t.data(), static_cast<int>(t.size())));
    }
    /// K V (oracle.hpp:25-29)
    Eigen::MatrixXd apply(const Eigen::MatrixXd& v) const { return run(-1, v); }
    /// dK/dtheta_j V (oracle.hpp:31-35)
    Eigen::MatrixXd apply_derivative(int j, const Eigen::MatrixXd& v) const { return run(j, v); }
    std::uint64_t apply_columns() const { return counters(false).first; }
    std::uint64_t derivative_columns() const { return counters(false).second; }
    void reset_counters() const { counters(true); }
    hg_oracle_t handle() const { return o_.get(); }

protected:
    CovarianceOracle() = default;
    void adopt(hg_oracle_t o, Index n, Index p) {
        o_.reset(o, [](hg_oracle_t x) { hg_oracle_free(x); });
        n_ = n;
        p_ = p;
    }
    Eigen::VectorXd theta_;

private:
    Eigen::MatrixXd run(int j, const Eigen::MatrixXd& v) const {
        Eigen::MatrixXd vc = v, y(v.rows(), v.cols());
        check(hg_oracle_apply(ctx(), o_.get(), j, vc.data(), vc.rows(), vc.cols(), y.data(), y.rows(), HG_HOST));
        return y;
    }
    std::pair<std::uint64_t, std::uint64_t> counters(bool reset) const {
        uint64_t a = 0, d = 0;
        check(hg_oracle_counters(o_.get(), &a, &d, reset ? 1 : 0));
        return {a, d};
    }
    std::shared_ptr<hg_oracle_s> o_;
    Index n_ = 0, p_ = 0;
};

/// oracle.hpp:115-143, matrices resident on the device.
class DenseMatrixOracle : public CovarianceOracle {
public:
    DenseMatrixOracle(Eigen::MatrixXd k, std::vector<Eigen::MatrixXd> dk = {},
                      Eigen::VectorXd theta = Eigen::VectorXd()) {
        const Index n = k.rows();
        Eigen::MatrixXd all(n, n * std::max<Index>(Index(dk.size()), 1));
        for (std::size_t j = 0; j < dk.size(); ++j) all.middleCols(Index(j) * n, n) = dk[j];
        hg_oracle_t o = nullptr;
        check(hg_oracle_dense(ctx(), n, k.data(), static_cast<int>(dk.size()), all.data(), &o));
        adopt(o, n, Index(dk.size()));
        theta_ = theta;
    }
    void set_parameters(const Eigen::VectorXd& theta) override { theta_ = theta; }
};

/// 1D Matérn nu = nu2/2 on sorted points (BASELINE C1/C4), theta = (sigma2, ell).
class MaternOracle : public CovarianceOracle {
public:
    MaternOracle(const Eigen::VectorXd& x, int nu2, double sigma2, double ell, double nugget, bool scan = true) {
        Eigen::VectorXd xc = x;
        hg_oracle_t o = nullptr;
        check(hg_oracle_matern(ctx(), xc.size(), xc.data(), nu2, sigma2, ell, nugget, scan ? 1 : 0, &o));
        adopt(o, xc.size(), 2);
        theta_ = Eigen::VectorXd(2);
        theta_ << sigma2, ell;
    }
};

/// oracle.hpp:58-111 over any oracle above (kept alive by the view).
class PermutedOracle : public CovarianceOracle {
public:
    PermutedOracle(std::shared_ptr<const CovarianceOracle> base, std::vector<Index> to_base)
        : base_(std::move(base)), p_(std::move(to_base)) {
        if (Index(p_.size()) != base_->dim()) throw std::invalid_argument("PermutedOracle: permutation size mismatch");
        std::vector<int64_t> p(p_.begin(), p_.end());
        hg_oracle_t o = nullptr;
        check(hg_oracle_permuted(ctx(), base_->handle(), p.data(), &o));
        adopt(o, base_->dim(), base_->num_params());
        theta_ = base_->parameters();
    }
    /// x in reordered layout -> base layout (oracle.hpp:74-79)
    Eigen::VectorXd scatter(const Eigen::VectorXd& x) const {
        Eigen::VectorXd out(x.size());
        for (Index i = 0; i < x.size(); ++i) out[p_[static_cast<std::size_t>(i)]] = x[i];
        return out;
    }
    /// x in base layout -> reordered layout (oracle.hpp:81-86)
    Eigen::VectorXd gather(const Eigen::VectorXd& x) const {
        Eigen::VectorXd out(x.size());
        for (Index i = 0; i < x.size(); ++i) out[i] = x[p_[static_cast<std::size_t>(i)]];
        return out;
    }

private:
    std::shared_ptr<const CovarianceOracle> base_;
    std::vector<Index> p_;
};

/// A device forward model written against the raw callback (device pointers,
/// the context's CUDA stream): the fast way to plug a new physics model in.
class DeviceCallbackOracle : public CovarianceOracle {
public:
    DeviceCallbackOracle(Index n, Index p, hg_apply_fn fn, void* user) {
        hg_oracle_t o = nullptr;
        check(hg_oracle_callback(ctx(), n, static_cast<int>(p), fn, user, &o));
        adopt(o, n, p);
    }
};

// --------------------------------------------------------- construction
/// sketch.hpp:17-40 — the sampler is regenerated bit-identically from the
/// seed on the host (sketch.cpp:10-31) and cached on the device by the build.
class SketchPlan {
public:
    SketchPlan() = default;
    SketchPlan(const ClusterTree& tree, Index k, std::uint64_t seed) : seed_(seed), k_(k), tree_(tree) {}
    std::uint64_t seed() const { return seed_; }
    Index rank() const { return k_; }
    bool dimensioned_for(const ClusterTree& tree, Index k) const { return tree_.same_structure(tree) && k_ == k; }

private:
    std::uint64_t seed_ = 0;
    Index k_ = 0;
    ClusterTree tree_;
};

struct BuildResult {
    HodlrMatrix h;
    std::vector<HodlrMatrix> deriv;
    std::vector<std::string> warnings;
};

inline BuildResult build_impl(const CovarianceOracle& oracle, const ClusterTree& tree, Index k, const SketchPlan& plan,
                              bool with_deriv) {
    if (oracle.dim() != tree.size()) throw std::invalid_argument("build_hodlr: oracle dimension mismatch");
    if (!plan.dimensioned_for(tree, k)) throw std::invalid_argument("build_hodlr: sketch plan not dimensioned for tree");
    hg_build_t b = nullptr;
    check(hg_build(ctx(), oracle.handle(), tree.depth(), k, plan.seed(), with_deriv ? 1 : 0, &b));
    std::unique_ptr<hg_build_s, hg_status (*)(hg_build_t)> guard(b, &hg_build_free);
    BuildResult out;
    hg_hodlr_t h = nullptr;
    check(hg_build_h(b, &h));
    out.h = HodlrMatrix(h);
    if (with_deriv)
        for (Index j = 0; j < oracle.num_params(); ++j) {
            hg_hodlr_t d = nullptr;
            check(hg_build_deriv(b, static_cast<int>(j), &d));
            out.deriv.emplace_back(d);
        }
    for (int w = 0; w < hg_build_num_warnings(b); ++w) out.warnings.push_back("ill-conditioned QR");
    return out;
}

/// sketch.cpp:347-350
inline HodlrMatrix build_hodlr(const CovarianceOracle& oracle, const ClusterTree& tree, Index k,
                               const SketchPlan& plan) {
    return build_impl(oracle, tree, k, plan, false).h;
}
/// sketch.cpp:352-356
inline BuildResult build_hodlr_with_derivatives(const CovarianceOracle& oracle, const ClusterTree& tree, Index k,
                                                const SketchPlan& plan) {
    return build_impl(oracle, tree, k, plan, true);
}

// ------------------------------------------------------------------ mle
namespace detail {
inline std::vector<hg_hodlr_t> handles(const std::vector<HodlrMatrix>& d) {
    std::vector<hg_hodlr_t> h;
    for (const auto& m : d) h.push_back(m.handle());
    return h;
}
}  // namespace detail

/// mle.cpp:25-30
inline double log_likelihood(const HodlrFactorization& f, const Eigen::VectorXd& y, const Eigen::VectorXd& ybar) {
    if (ybar.size() != 0 && ybar.size() != y.size()) throw std::invalid_argument("mean length mismatch");
    Eigen::VectorXd yc = y, yb = ybar;
    double out = 0;
    check(hg_log_likelihood(ctx(), f.handle(), yc.data(), ybar.size() ? yb.data() : nullptr, &out));
    return out;
}
/// mle.cpp:32-41
inline Eigen::VectorXd score(const HodlrFactorization& f, const std::vector<HodlrMatrix>& deriv,
                             const Eigen::VectorXd& y, const Eigen::VectorXd& ybar) {
    if (ybar.size() != 0 && ybar.size() != y.size()) throw std::invalid_argument("mean length mismatch");
    Eigen::VectorXd yc = y, yb = ybar, out(Index(deriv.size()));
    auto h = detail::handles(deriv);
    check(hg_score(ctx(), f.handle(), h.data(), static_cast<int>(h.size()), yc.data(),
                   ybar.size() ? yb.data() : nullptr, out.data()));
    return out;
}
/// mle.cpp:43-54
inline Eigen::MatrixXd fisher_information(const HodlrFactorization& f, const std::vector<HodlrMatrix>& deriv) {
    const Index p = Index(deriv.size());
    Eigen::MatrixXd out(p, p);
    auto h = detail::handles(deriv);
    check(hg_fisher_information(ctx(), f.handle(), h.data(), static_cast<int>(p), out.data()));
    return out;
}

}  // namespace hodlrgp_b200

#ifdef HODLRGP_B200_AS_HODLRGP
namespace hodlrgp {
using namespace ::hodlrgp_b200;
}
#endif
