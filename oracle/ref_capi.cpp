// TEST INFRASTRUCTURE ONLY — the same C ABI as oracle/capi.cpp (the `or_*`
// entry points pyoracle binds), implemented over the REFERENCE's own code:
// /root/reference/proj/src/{cluster_tree,hodlr_matrix,sketch,factorization,
// product_rep,mle}.cpp compiled unmodified against the Eigen-API shim
// (oracle/eigen_shim) by oracle/ref.mk into oracle/_ref/libhodlrgp_ref.so.
// This lets every parity test and the CPU baseline run on the reference
// implementation itself instead of a restatement.
//
// Differences from oracle/capi.cpp, all because the reference exposes no such
// hook: or_set_solve_association / or_set_q2_reorthogonalize / or_set_compress_at_level are ignored (the reference has only its own
// association, product_rep.cpp:74-78), or_build_decisions reports 0 nodes and
// or_factor_leaf_llt is unavailable (LeafFactor::use_llt_ is private).
#include <chrono>
#include <random>
#include <cstring>
#include <memory>
#include <string>

#include "hodlrgp/cluster_tree.hpp"
#include "hodlrgp/factorization.hpp"
#include "hodlrgp/hodlr_matrix.hpp"
#include "hodlrgp/mle.hpp"
#include "hodlrgp/oracle.hpp"
#include "hodlrgp/product_rep.hpp"
#include "hodlrgp/sketch.hpp"
#include "matern1d.hpp"

namespace oracle {  // restated helpers from oracle/dense.cpp (BLAS switch, RNG)
bool enable_external_blas(const char* path, int threads);
const char* blas_backend();
}  // namespace oracle

using namespace hodlrgp;
using Eigen::MatrixXd;
using Eigen::VectorXd;

#define OR_API extern "C" __attribute__((visibility("default")))

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const NotPositiveDefinite& e) {
        g_err = e.what();
        return 1;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 2;
    } catch (const std::length_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

MatrixXd from_ptr(const double* p, Index r, Index c) {
    MatrixXd m(r, c);
    if (r > 0 && c > 0) std::memcpy(m.data(), p, static_cast<size_t>(r * c) * sizeof(double));
    return m;
}
template <class E>
void to_ptr(const E& e, double* p) {
    MatrixXd m(e);
    if (m.size() > 0) std::memcpy(p, m.data(), static_cast<size_t>(m.size()) * sizeof(double));
}

struct OHodlr {
    HodlrMatrix h;
};
struct OFactor {
    HodlrFactorization f;
};
struct ORep {
    ProductRep p;
};
struct OOracle {
    std::unique_ptr<CovarianceOracle> o;
};
struct OBuild {
    BuildResult r;
};

/// Same forward model as the restated oracle (oracle/matern1d.hpp).
class Matern1dRefOracle : public CovarianceOracle {
public:
    Matern1dRefOracle(std::vector<double> x, int nu2, double sigma2, double ell, double nugget, bool scan)
        : x_(std::move(x)), nu2_(nu2), sigma2_(sigma2), ell_(ell), nugget_(nugget), scan_(scan) {
        if (nu2 != 1 && nu2 != 3 && nu2 != 5) throw std::invalid_argument("Matern1d: nu in {1/2,3/2,5/2}");
        for (size_t i = 1; i < x_.size(); ++i)
            if (x_[i] < x_[i - 1]) throw std::invalid_argument("Matern1d: points must be sorted");
    }
    Index dim() const override { return Index(x_.size()); }
    Index num_params() const override { return 2; }
    VectorXd parameters() const override {
        VectorXd t(2);
        t << sigma2_, ell_;
        return t;
    }
    void set_parameters(const VectorXd& t) override {
        sigma2_ = t[0];
        ell_ = t[1];
    }

protected:
    MatrixXd do_apply(const Eigen::Ref<const MatrixXd>& v) const override { return run(-1, v); }
    MatrixXd do_apply_derivative(int j, const Eigen::Ref<const MatrixXd>& v) const override { return run(j, v); }

private:
    MatrixXd run(int which, const Eigen::Ref<const MatrixXd>& v) const {
        MatrixXd vc(v), y(v.rows(), v.cols());
        matern1d::apply(x_.data(), dim(), nu2_, sigma2_, ell_, nugget_, which, scan_, vc.data(), vc.rows(),
                        vc.cols(), y.data(), y.rows());
        return y;
    }
    std::vector<double> x_;
    int nu2_;
    double sigma2_, ell_, nugget_;
    bool scan_;
};

void level_caps(const HodlrMatrix& h, int* R) {
    for (int l = 1; l <= h.depth(); ++l) {
        Index r = 0;
        for (size_t j = 0; j < h.tree().level(l - 1).size(); ++j) {
            r = std::max(r, h.upper(l, Index(j)).rank());
            r = std::max(r, h.lower_block(l, Index(j)).rank());
        }
        R[l - 1] = int(r);
    }
}

/// fisher_information (mle.cpp:43-54) with the p ProductReps of
/// solve_multiply(f, D_j) formed once and reused for every pair; the same
/// reference functions, called fewer times (cache = 0 calls the reference's
/// fisher_information itself).
MatrixXd fisher_cached(const HodlrFactorization& f, const std::vector<HodlrMatrix>& d) {
    const Index p = Index(d.size());
    std::vector<ProductRep> reps;
    for (const auto& dj : d) reps.push_back(solve_multiply(f, dj));
    MatrixXd info(p, p);
    for (Index i = 0; i < p; ++i)
        for (Index j = i; j < p; ++j) {
            const double t = 0.5 * trace_pair(reps[size_t(i)], reps[size_t(j)]);
            info(i, j) = t;
            info(j, i) = t;
        }
    return 0.5 * (info + info.transpose());
}

std::vector<HodlrMatrix> derivs_of(void** derivs, int p) {
    std::vector<HodlrMatrix> d;
    for (int j = 0; j < p; ++j) d.push_back(static_cast<OHodlr*>(derivs[j])->h);
    return d;
}
}  // namespace

OR_API const char* or_last_error() { return g_err.c_str(); }
OR_API int or_enable_blas(const char* path, int threads) { return oracle::enable_external_blas(path, threads) ? 1 : 0; }
OR_API const char* or_blas_backend() { return oracle::blas_backend(); }
OR_API void or_set_solve_association(int) {}
OR_API void or_set_q2_reorthogonalize(int) {}
OR_API void or_set_compress_at_level(int) {}
OR_API int or_is_reference() { return 1; }

// ------------------------------------------------------------------ tree
OR_API int or_tree_depth(std::int64_t n, std::int64_t lmin, std::int64_t lmax) { return tree_depth(n, lmin, lmax); }

OR_API int or_tree_ranges(std::int64_t n, int tau, std::int64_t* lo_hi) {
    return guard([&] {
        ClusterTree t(n, tau);
        size_t o = 0;
        for (int d = 0; d <= tau; ++d)
            for (const auto& r : t.level(d)) {
                lo_hi[o++] = r.lo;
                lo_hi[o++] = r.hi;
            }
    });
}

OR_API int or_kd_ordering(std::int64_t n, int d, const double* coords, std::int64_t lmin, std::int64_t lmax,
                          std::int64_t* perm, std::int64_t* inv, int* tau) {
    return guard([&] {
        KdOrdering kd = build_kd_ordering(PointSet{from_ptr(coords, n, d)}, lmin, lmax);
        for (Index i = 0; i < n; ++i) {
            perm[i] = kd.perm[static_cast<size_t>(i)];
            inv[i] = kd.inv[static_cast<size_t>(i)];
        }
        *tau = kd.tree.depth();
    });
}

// ----------------------------------------------------------------- HODLR
OR_API void* or_hodlr_random(std::int64_t n, int tau, std::int64_t k, std::uint64_t seed, int spd) {
    auto* o = new OHodlr;
    ClusterTree t(n, tau);
    o->h = spd ? HodlrMatrix::random_spd(t, k, seed) : HodlrMatrix::random_symmetric(t, k, seed);
    return o;
}

OR_API void* or_hodlr_from_dense(std::int64_t n, int tau, const double* a, int sym) {
    auto* o = new OHodlr;
    if (guard([&] { o->h = HodlrMatrix::from_dense(ClusterTree(n, tau), from_ptr(a, n, n), sym != 0); })) {
        delete o;
        return nullptr;
    }
    return o;
}

OR_API void* or_hodlr_identity(std::int64_t n, int tau) {
    auto* o = new OHodlr;
    o->h = HodlrMatrix::identity(ClusterTree(n, tau));
    return o;
}

OR_API void or_hodlr_free(void* h) { delete static_cast<OHodlr*>(h); }
OR_API void* or_hodlr_copy(void* h) { return new OHodlr(*static_cast<OHodlr*>(h)); }

OR_API int or_hodlr_info(void* hp, std::int64_t* n, int* tau, int* sym, int* R) {
    auto& h = static_cast<OHodlr*>(hp)->h;
    *n = h.size();
    *tau = h.depth();
    *sym = h.symmetric() ? 1 : 0;
    if (R) level_caps(h, R);
    return 0;
}

/// Panel exchange format of oracle/capi.cpp (per level U_l, V_l n x R_l, then leaves).
OR_API int or_hodlr_export(void* hp, double* flat, int* ranks_up, int* ranks_lo) {
    return guard([&] {
        auto& h = static_cast<OHodlr*>(hp)->h;
        const auto& tree = h.tree();
        const Index n = h.size();
        std::vector<int> R(static_cast<size_t>(h.depth()));
        level_caps(h, R.data());
        size_t off = 0, nodeoff = 0;
        for (int l = 1; l <= h.depth(); ++l) {
            const Index Rl = R[static_cast<size_t>(l - 1)];
            double* U = flat + off;
            double* V = flat + off + static_cast<size_t>(n * Rl);
            std::memset(U, 0, static_cast<size_t>(2 * n * Rl) * sizeof(double));
            const auto& kids = tree.level(l);
            for (size_t j = 0; j < tree.level(l - 1).size(); ++j) {
                auto cl = kids[2 * j], cr = kids[2 * j + 1];
                const LowRankBlock& up = h.upper(l, Index(j));
                const LowRankBlock lo = h.lower_block(l, Index(j));
                for (Index c = 0; c < up.rank(); ++c) {
                    for (Index i = 0; i < cl.size(); ++i) U[cl.lo + i + c * n] = up.left(i, c);
                    for (Index i = 0; i < cr.size(); ++i) V[cr.lo + i + c * n] = up.right(i, c);
                }
                for (Index c = 0; c < lo.rank(); ++c) {
                    for (Index i = 0; i < cr.size(); ++i) U[cr.lo + i + c * n] = lo.left(i, c);
                    for (Index i = 0; i < cl.size(); ++i) V[cl.lo + i + c * n] = lo.right(i, c);
                }
                ranks_up[nodeoff] = int(up.rank());
                ranks_lo[nodeoff] = int(lo.rank());
                ++nodeoff;
            }
            off += static_cast<size_t>(2 * n * Rl);
        }
        for (Index b = 0; b < h.num_leaves(); ++b) {
            to_ptr(h.leaf(b), flat + off);
            off += static_cast<size_t>(h.leaf(b).size());
        }
    });
}

OR_API void* or_hodlr_import(std::int64_t n, int tau, int sym, const int* R, const double* flat,
                             const int* ranks_up, const int* ranks_lo) {
    auto* o = new OHodlr;
    int rc = guard([&] {
        ClusterTree tree(n, tau);
        o->h = HodlrMatrix::zero(tree, sym != 0);
        size_t off = 0, nodeoff = 0;
        for (int l = 1; l <= tau; ++l) {
            const Index Rl = R[l - 1];
            const double* U = flat + off;
            const double* V = flat + off + static_cast<size_t>(n * Rl);
            const auto& kids = tree.level(l);
            for (size_t j = 0; j < tree.level(l - 1).size(); ++j) {
                auto cl = kids[2 * j], cr = kids[2 * j + 1];
                const Index ru = ranks_up[nodeoff], rl = ranks_lo[nodeoff];
                LowRankBlock up;
                up.left = MatrixXd(cl.size(), ru);
                up.right = MatrixXd(cr.size(), ru);
                for (Index c = 0; c < ru; ++c) {
                    for (Index i = 0; i < cl.size(); ++i) up.left(i, c) = U[cl.lo + i + c * n];
                    for (Index i = 0; i < cr.size(); ++i) up.right(i, c) = V[cr.lo + i + c * n];
                }
                o->h.upper(l, Index(j)) = up;
                if (!sym) {
                    LowRankBlock lo;
                    lo.left = MatrixXd(cr.size(), rl);
                    lo.right = MatrixXd(cl.size(), rl);
                    for (Index c = 0; c < rl; ++c) {
                        for (Index i = 0; i < cr.size(); ++i) lo.left(i, c) = U[cr.lo + i + c * n];
                        for (Index i = 0; i < cl.size(); ++i) lo.right(i, c) = V[cl.lo + i + c * n];
                    }
                    o->h.lower(l, Index(j)) = lo;
                }
                ++nodeoff;
            }
            off += static_cast<size_t>(2 * n * Rl);
        }
        for (Index b = 0; b < tree.num_leaves(); ++b) {
            const Index m = tree.leaves()[static_cast<size_t>(b)].size();
            o->h.leaf(b) = from_ptr(flat + off, m, m);
            off += static_cast<size_t>(m * m);
        }
    });
    if (rc) {
        delete o;
        return nullptr;
    }
    return o;
}

OR_API int or_hodlr_densify(void* h, double* out) {
    return guard([&] { to_ptr(static_cast<OHodlr*>(h)->h.densify(), out); });
}

OR_API int or_hodlr_matvec(void* hp, const double* x, std::int64_t s, double* y) {
    return guard([&] {
        auto& h = static_cast<OHodlr*>(hp)->h;
        to_ptr(h.matvec(from_ptr(x, h.size(), s)), y);
    });
}

OR_API int or_hodlr_sub_matvec(void* hp, int d, std::int64_t node, const double* x, std::int64_t rows,
                               std::int64_t s, int transpose, double* y) {
    return guard([&] {
        auto& h = static_cast<OHodlr*>(hp)->h;
        to_ptr(h.sub_matvec(d, node, from_ptr(x, rows, s), transpose != 0), y);
    });
}

OR_API double or_hodlr_trace(void* h) { return static_cast<OHodlr*>(h)->h.trace(); }

OR_API int or_trace_product(void* a, void* b, double* out) {
    return guard([&] { *out = HodlrMatrix::trace_product(static_cast<OHodlr*>(a)->h, static_cast<OHodlr*>(b)->h); });
}

OR_API void or_hodlr_make_asymmetric(void* h) { static_cast<OHodlr*>(h)->h.make_asymmetric(); }

// --------------------------------------------------------- factorization
OR_API void* or_factorize(void* hp, int orient) {
    auto* o = new OFactor;
    if (guard([&] {
            o->f = factorize(static_cast<OHodlr*>(hp)->h, orient ? Orientation::Left : Orientation::Right);
        })) {
        delete o;
        return nullptr;
    }
    return o;
}

OR_API void or_factor_free(void* f) { delete static_cast<OFactor*>(f); }

OR_API int or_factor_solve(void* fp, const double* b, std::int64_t s, double* x) {
    return guard([&] {
        auto& f = static_cast<OFactor*>(fp)->f;
        to_ptr(f.solve(from_ptr(b, f.size(), s)), x);
    });
}

OR_API int or_factor_logdet(void* fp, double* out) {
    return guard([&] { *out = static_cast<OFactor*>(fp)->f.logdet(); });
}

OR_API int or_factor_leaf_llt(void*, int*) {
    g_err = "reference LeafFactor does not expose its LLT/LU choice";
    return 4;
}

// ------------------------------------------------------------ product rep
OR_API void* or_solve_multiply(void* fp, void* bp) {
    auto* o = new ORep;
    if (guard([&] { o->p = solve_multiply(static_cast<OFactor*>(fp)->f, static_cast<OHodlr*>(bp)->h); })) {
        delete o;
        return nullptr;
    }
    return o;
}

OR_API void* or_multiply(void* fp, void* bp) {
    auto* o = new ORep;
    if (guard([&] { o->p = multiply(static_cast<OFactor*>(fp)->f, static_cast<OHodlr*>(bp)->h); })) {
        delete o;
        return nullptr;
    }
    return o;
}

OR_API void or_prodrep_free(void* p) { delete static_cast<ORep*>(p); }

OR_API int or_prodrep_densify(void* p, double* out) {
    return guard([&] { to_ptr(static_cast<ORep*>(p)->p.densify(), out); });
}

OR_API double or_trace_product_rep(void* p) { return trace_product_rep(static_cast<ORep*>(p)->p); }
OR_API double or_trace_pair(void* p, void* q) {
    return trace_pair(static_cast<ORep*>(p)->p, static_cast<ORep*>(q)->p);
}

OR_API int or_hutchinson_trace(void* fp, void* bp, int n_samples, std::uint64_t seed, double* out2) {
    return guard([&] {
        const HutchinsonResult r = hutchinson_trace(static_cast<OFactor*>(fp)->f, static_cast<OHodlr*>(bp)->h, n_samples, seed);
        out2[0] = r.estimate;
        out2[1] = r.std_error;
    });
}
OR_API int or_trace_solve(void* fp, void* bp, double* out) {
    return guard([&] { *out = trace_solve(static_cast<OFactor*>(fp)->f, static_cast<OHodlr*>(bp)->h); });
}

OR_API int or_trace_quad(void* fa, void* b, void* fc, void* d, double* out) {
    return guard([&] {
        *out = trace_quad(static_cast<OFactor*>(fa)->f, static_cast<OHodlr*>(b)->h, static_cast<OFactor*>(fc)->f,
                          static_cast<OHodlr*>(d)->h);
    });
}

// ----------------------------------------------------------------- sketch
OR_API int or_sketch_sampler(std::int64_t n, int tau, std::int64_t k, std::uint64_t seed, int l, double* out) {
    return guard([&] {
        SketchPlan plan(ClusterTree(n, tau), k, seed);
        to_ptr(l == 0 ? plan.leaf_sampler() : plan.level_sampler(l), out);
    });
}

OR_API int or_randomized_range(const double* y, std::int64_t m, std::int64_t k, double* q, double* r, int* perm,
                               std::int64_t* nrank) {
    return guard([&] {
        RangeResult rr = randomized_range(from_ptr(y, m, k), k);
        to_ptr(rr.q, q);
        to_ptr(rr.r, r);
        for (Index i = 0; i < k; ++i) perm[i] = rr.perm[i];
        *nrank = rr.numeric_rank;
    });
}

OR_API int or_diff_qr(const double* db, const double* q, const double* r, std::int64_t m, std::int64_t k,
                      double* dq, double* dq_span, double* dr, int* ill) {
    return guard([&] {
        MatrixXd dbm = from_ptr(db, m, k);
        DiffQrResult d = diff_qr(dbm, dbm, from_ptr(q, m, k), from_ptr(r, k, k));
        to_ptr(d.dq, dq);
        to_ptr(d.dq_span, dq_span);
        to_ptr(d.dr, dr);
        *ill = d.ill_conditioned ? 1 : 0;
    });
}

// ---------------------------------------------------------------- oracles
OR_API void* or_oracle_dense(std::int64_t n, const double* k, int p, const double* dks) {
    auto* o = new OOracle;
    std::vector<MatrixXd> dk;
    for (int j = 0; j < p; ++j) dk.push_back(from_ptr(dks + static_cast<size_t>(j) * static_cast<size_t>(n * n), n, n));
    o->o = std::make_unique<DenseMatrixOracle>(from_ptr(k, n, n), std::move(dk));
    return o;
}

OR_API void* or_oracle_matern(std::int64_t n, const double* x, int nu2, double sigma2, double ell, double nugget,
                              int scan) {
    auto* o = new OOracle;
    if (guard([&] {
            o->o = std::make_unique<Matern1dRefOracle>(std::vector<double>(x, x + n), nu2, sigma2, ell, nugget,
                                                       scan != 0);
        })) {
        delete o;
        return nullptr;
    }
    return o;
}

OR_API void or_oracle_free(void* o) { delete static_cast<OOracle*>(o); }

OR_API int or_oracle_apply(void* op, int which, const double* v, std::int64_t s, double* y) {
    return guard([&] {
        auto& o = *static_cast<OOracle*>(op)->o;
        MatrixXd vm = from_ptr(v, o.dim(), s);
        to_ptr(which < 0 ? o.apply(vm) : o.apply_derivative(which, vm), y);
    });
}

OR_API int or_oracle_counters(void* op, std::uint64_t* apply_cols, std::uint64_t* deriv_cols, int reset) {
    auto& o = *static_cast<OOracle*>(op)->o;
    *apply_cols = o.apply_columns();
    *deriv_cols = o.derivative_columns();
    if (reset) o.reset_counters();
    return 0;
}

// ------------------------------------------------------------------ build
OR_API void* or_build(void* op, int tau, std::int64_t k, std::uint64_t seed, int with_deriv) {
    auto* o = new OBuild;
    if (guard([&] {
            auto& orc = *static_cast<OOracle*>(op)->o;
            ClusterTree tree(orc.dim(), tau);
            SketchPlan plan(tree, k, seed);
            if (with_deriv)
                o->r = build_hodlr_with_derivatives(orc, tree, k, plan);
            else
                o->r.h = build_hodlr(orc, tree, k, plan);
        })) {
        delete o;
        return nullptr;
    }
    return o;
}

OR_API void or_build_free(void* b) { delete static_cast<OBuild*>(b); }
OR_API void* or_build_h(void* b) { return new OHodlr{static_cast<OBuild*>(b)->r.h}; }
OR_API void* or_build_deriv(void* b, int j) {
    return new OHodlr{static_cast<OBuild*>(b)->r.deriv[static_cast<size_t>(j)]};
}
OR_API int or_build_num_warnings(void* b) { return int(static_cast<OBuild*>(b)->r.warnings.size()); }
OR_API int or_build_decisions(void*, int, std::int64_t*) { return 0; }

// -------------------------------------------------------------------- mle
OR_API int or_log_likelihood(void* fp, const double* y, const double* ybar, double* out) {
    return guard([&] {
        auto& f = static_cast<OFactor*>(fp)->f;
        *out = log_likelihood(f, VectorXd(from_ptr(y, f.size(), 1)),
                              ybar ? VectorXd(from_ptr(ybar, f.size(), 1)) : VectorXd());
    });
}

OR_API int or_score(void* fp, void** derivs, int p, const double* y, const double* ybar, double* out) {
    return guard([&] {
        auto& f = static_cast<OFactor*>(fp)->f;
        VectorXd s = score(f, derivs_of(derivs, p), VectorXd(from_ptr(y, f.size(), 1)),
                           ybar ? VectorXd(from_ptr(ybar, f.size(), 1)) : VectorXd());
        for (int j = 0; j < p; ++j) out[j] = s[j];
    });
}

OR_API int or_fisher(void* fp, void** derivs, int p, int cache, double* out) {
    return guard([&] {
        auto& f = static_cast<OFactor*>(fp)->f;
        const auto d = derivs_of(derivs, p);
        to_ptr(cache ? fisher_cached(f, d) : fisher_information(f, d), out);
    });
}

/// One MLE iteration (acceptance.cpp:297-308) through the reference's own
/// functions, timed under the reference bench's stage names
/// (tools/hodlr_gp.cpp:425-450): build_deriv, factorize, loglik, score, fisher.
OR_API int or_mle_iteration(void* op, int tau, std::int64_t k, std::uint64_t seed, const double* y, int cache,
                            double* loglik, double* score_out, double* fisher_out, double* times) {
    return guard([&] {
        using clk = std::chrono::steady_clock;
        auto& orc = *static_cast<OOracle*>(op)->o;
        ClusterTree tree(orc.dim(), tau);
        SketchPlan plan(tree, k, seed);
        auto t0 = clk::now();
        BuildResult br = build_hodlr_with_derivatives(orc, tree, k, plan);
        auto t1 = clk::now();
        HodlrFactorization f = factorize(br.h, Orientation::Left);
        auto t2 = clk::now();
        VectorXd ym(from_ptr(y, tree.size(), 1));
        *loglik = log_likelihood(f, ym, VectorXd());
        auto t3 = clk::now();
        VectorXd s = score(f, br.deriv, ym, VectorXd());
        for (Index j = 0; j < s.size(); ++j) score_out[j] = s[j];
        auto t4 = clk::now();
        to_ptr(cache ? fisher_cached(f, br.deriv) : fisher_information(f, br.deriv), fisher_out);
        auto t5 = clk::now();
        auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
        times[0] = sec(t0, t1);
        times[1] = sec(t1, t2);
        times[2] = sec(t2, t3);
        times[3] = sec(t3, t4);
        times[4] = sec(t4, t5);
    });
}

OR_API void or_randn(std::int64_t r, std::int64_t c, std::uint64_t seed, double* out) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> g(0.0, 1.0);
    for (Index i = 0; i < r; ++i)
        for (Index j = 0; j < c; ++j) out[i + j * r] = g(rng);
}
