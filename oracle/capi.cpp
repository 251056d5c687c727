// TEST INFRASTRUCTURE ONLY — C ABI over the parity oracle, for the pytest
// suite (ctypes) and bench.py's cpu_baseline leg. Never linked by the product.
//
// Error codes mirror the product ABI (include/hodlrgp_b200.h):
//   0 ok, 1 NotPositiveDefinite, 2 invalid_argument, 3 length_error,
//   4 logic_error, 9 other.
#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include "oracle.hpp"

using namespace oracle;

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

Mat from_ptr(const double* p, Index r, Index c) {
    Mat m(r, c);
    if (r > 0 && c > 0) std::memcpy(m.data(), p, static_cast<size_t>(r * c) * sizeof(double));
    return m;
}
void to_ptr(const Mat& m, double* p) {
    if (m.r > 0 && m.c > 0) std::memcpy(p, m.data(), static_cast<size_t>(m.r * m.c) * sizeof(double));
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

/// Panel exchange format (shared with the product ABI): per level l the
/// left-factor panel U_l and right-factor panel V_l, each n x R_l col-major:
/// U rows of the left child hold upper.left, rows of the right child hold
/// lower.left; V rows of the right child hold upper.right, rows of the left
/// child hold lower.right. Columns beyond a block's rank are zero. Leaves
/// follow, concatenated col-major m_b x m_b.
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
}  // namespace

extern "C" {

const char* or_last_error() { return g_err.c_str(); }
int or_enable_blas(const char* path, int threads) { return enable_external_blas(path, threads) ? 1 : 0; }
const char* or_blas_backend() { return blas_backend(); }
void or_set_solve_association(int on) { set_solve_association(on != 0); }
void or_set_q2_reorthogonalize(int on) { set_q2_reorthogonalize(on != 0); }
void or_set_compress_at_level(int on) { set_compress_at_level(on != 0); }

// ------------------------------------------------------------------ tree
int or_tree_depth(std::int64_t n, std::int64_t lmin, std::int64_t lmax) { return tree_depth(n, lmin, lmax); }

/// lo_hi: 2 * (2^(tau+1) - 1) int64, depth-major.
int or_tree_ranges(std::int64_t n, int tau, std::int64_t* lo_hi) {
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

int or_kd_ordering(std::int64_t n, int d, const double* coords, std::int64_t lmin, std::int64_t lmax,
                   std::int64_t* perm, std::int64_t* inv, int* tau) {
    return guard([&] {
        KdOrdering kd = build_kd_ordering(from_ptr(coords, n, d), lmin, lmax);
        for (Index i = 0; i < n; ++i) {
            perm[i] = kd.perm[static_cast<size_t>(i)];
            inv[i] = kd.inv[static_cast<size_t>(i)];
        }
        *tau = kd.tree.depth();
    });
}

// ----------------------------------------------------------------- HODLR
void* or_hodlr_random(std::int64_t n, int tau, std::int64_t k, std::uint64_t seed, int spd) {
    auto* o = new OHodlr;
    ClusterTree t(n, tau);
    o->h = spd ? HodlrMatrix::random_spd(t, k, seed) : HodlrMatrix::random_symmetric(t, k, seed);
    return o;
}

void* or_hodlr_from_dense(std::int64_t n, int tau, const double* a, int sym) {
    auto* o = new OHodlr;
    if (guard([&] { o->h = HodlrMatrix::from_dense(ClusterTree(n, tau), from_ptr(a, n, n), sym != 0); })) {
        delete o;
        return nullptr;
    }
    return o;
}

void* or_hodlr_identity(std::int64_t n, int tau) {
    auto* o = new OHodlr;
    o->h = HodlrMatrix::identity(ClusterTree(n, tau));
    return o;
}

void or_hodlr_free(void* h) { delete static_cast<OHodlr*>(h); }

void* or_hodlr_copy(void* h) { return new OHodlr(*static_cast<OHodlr*>(h)); }

int or_hodlr_info(void* hp, std::int64_t* n, int* tau, int* sym, int* R) {
    auto& h = static_cast<OHodlr*>(hp)->h;
    *n = h.size();
    *tau = h.depth();
    *sym = h.symmetric() ? 1 : 0;
    if (R) level_caps(h, R);
    return 0;
}

/// flat: sum_l 2 n R_l doubles then sum_b m_b^2; ranks_up/lo: 2^tau - 1 ints.
int or_hodlr_export(void* hp, double* flat, int* ranks_up, int* ranks_lo) {
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
                const LowRankBlock up = h.upper(l, Index(j));
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
            off += static_cast<size_t>(h.leaf(b).r * h.leaf(b).c);
        }
    });
}

void* or_hodlr_import(std::int64_t n, int tau, int sym, const int* R, const double* flat,
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
                Index ru = ranks_up[nodeoff], rl = ranks_lo[nodeoff];
                LowRankBlock up;
                up.left = Mat(cl.size(), ru);
                up.right = Mat(cr.size(), ru);
                for (Index c = 0; c < ru; ++c) {
                    for (Index i = 0; i < cl.size(); ++i) up.left(i, c) = U[cl.lo + i + c * n];
                    for (Index i = 0; i < cr.size(); ++i) up.right(i, c) = V[cr.lo + i + c * n];
                }
                o->h.upper(l, Index(j)) = up;
                if (!sym) {
                    LowRankBlock lo;
                    lo.left = Mat(cr.size(), rl);
                    lo.right = Mat(cl.size(), rl);
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
            Index m = tree.leaves()[static_cast<size_t>(b)].size();
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

int or_hodlr_densify(void* h, double* out) {
    return guard([&] { to_ptr(static_cast<OHodlr*>(h)->h.densify(), out); });
}

int or_hodlr_matvec(void* hp, const double* x, std::int64_t s, double* y) {
    return guard([&] {
        auto& h = static_cast<OHodlr*>(hp)->h;
        to_ptr(h.matvec(from_ptr(x, h.size(), s)), y);
    });
}

int or_hodlr_sub_matvec(void* hp, int d, std::int64_t node, const double* x, std::int64_t rows,
                        std::int64_t s, int transpose, double* y) {
    return guard([&] {
        auto& h = static_cast<OHodlr*>(hp)->h;
        to_ptr(h.sub_matvec(d, node, from_ptr(x, rows, s), transpose != 0), y);
    });
}

double or_hodlr_trace(void* h) { return static_cast<OHodlr*>(h)->h.trace(); }

int or_trace_product(void* a, void* b, double* out) {
    return guard([&] { *out = HodlrMatrix::trace_product(static_cast<OHodlr*>(a)->h, static_cast<OHodlr*>(b)->h); });
}

void or_hodlr_make_asymmetric(void* h) { static_cast<OHodlr*>(h)->h.make_asymmetric(); }

// --------------------------------------------------------- factorization
void* or_factorize(void* hp, int orient) {
    auto* o = new OFactor;
    if (guard([&] { o->f = factorize(static_cast<OHodlr*>(hp)->h, orient ? Orientation::Left : Orientation::Right); })) {
        delete o;
        return nullptr;
    }
    return o;
}

void or_factor_free(void* f) { delete static_cast<OFactor*>(f); }

int or_factor_solve(void* fp, const double* b, std::int64_t s, double* x) {
    return guard([&] {
        auto& f = static_cast<OFactor*>(fp)->f;
        to_ptr(f.solve(from_ptr(b, f.size(), s)), x);
    });
}

int or_factor_logdet(void* fp, double* out) {
    return guard([&] { *out = static_cast<OFactor*>(fp)->f.logdet(); });
}

/// Leaf decisions: 1 where the leaf used LLT, 0 where it fell back to LU.
int or_factor_leaf_llt(void* fp, int* out) {
    auto& f = static_cast<OFactor*>(fp)->f;
    for (Index b = 0; b < f.num_leaves(); ++b) out[b] = f.leaf(b).uses_llt() ? 1 : 0;
    return 0;
}

// ------------------------------------------------------------ product rep
void* or_solve_multiply(void* fp, void* bp) {
    auto* o = new ORep;
    if (guard([&] { o->p = solve_multiply(static_cast<OFactor*>(fp)->f, static_cast<OHodlr*>(bp)->h); })) {
        delete o;
        return nullptr;
    }
    return o;
}

void* or_multiply(void* fp, void* bp) {
    auto* o = new ORep;
    if (guard([&] { o->p = multiply(static_cast<OFactor*>(fp)->f, static_cast<OHodlr*>(bp)->h); })) {
        delete o;
        return nullptr;
    }
    return o;
}

void or_prodrep_free(void* p) { delete static_cast<ORep*>(p); }

int or_prodrep_densify(void* p, double* out) {
    return guard([&] { to_ptr(static_cast<ORep*>(p)->p.densify(), out); });
}

double or_trace_product_rep(void* p) { return trace_product_rep(static_cast<ORep*>(p)->p); }
double or_trace_pair(void* p, void* q) { return trace_pair(static_cast<ORep*>(p)->p, static_cast<ORep*>(q)->p); }

int or_hutchinson_trace(void* fp, void* bp, int n_samples, std::uint64_t seed, double* out2) {
    return guard([&] {
        const HutchinsonResult r = hutchinson_trace(static_cast<OFactor*>(fp)->f, static_cast<OHodlr*>(bp)->h, n_samples, seed);
        out2[0] = r.estimate;
        out2[1] = r.std_error;
    });
}
int or_trace_solve(void* fp, void* bp, double* out) {
    return guard([&] { *out = trace_solve(static_cast<OFactor*>(fp)->f, static_cast<OHodlr*>(bp)->h); });
}

int or_trace_quad(void* fa, void* b, void* fc, void* d, double* out) {
    return guard([&] {
        *out = trace_quad(static_cast<OFactor*>(fa)->f, static_cast<OHodlr*>(b)->h,
                          static_cast<OFactor*>(fc)->f, static_cast<OHodlr*>(d)->h);
    });
}

// ----------------------------------------------------------------- sketch
int or_sketch_sampler(std::int64_t n, int tau, std::int64_t k, std::uint64_t seed, int l, double* out) {
    return guard([&] {
        SketchPlan plan(ClusterTree(n, tau), k, seed);
        to_ptr(l == 0 ? plan.leaf_sampler() : plan.level_sampler(l), out);
    });
}

int or_randomized_range(const double* y, std::int64_t m, std::int64_t k, double* q, double* r, int* perm,
                        std::int64_t* nrank) {
    return guard([&] {
        RangeResult rr = randomized_range(from_ptr(y, m, k), k);
        to_ptr(rr.q, q);
        to_ptr(rr.r, r);
        for (Index i = 0; i < k; ++i) perm[i] = rr.perm[static_cast<size_t>(i)];
        *nrank = rr.numeric_rank;
    });
}

int or_diff_qr(const double* db, const double* q, const double* r, std::int64_t m, std::int64_t k, double* dq,
               double* dq_span, double* dr, int* ill) {
    return guard([&] {
        Mat dbm = from_ptr(db, m, k);
        DiffQrResult d = diff_qr(dbm, dbm, from_ptr(q, m, k), from_ptr(r, k, k));
        to_ptr(d.dq, dq);
        to_ptr(d.dq_span, dq_span);
        to_ptr(d.dr, dr);
        *ill = d.ill_conditioned ? 1 : 0;
    });
}

// ---------------------------------------------------------------- oracles
void* or_oracle_dense(std::int64_t n, const double* k, int p, const double* dks) {
    auto* o = new OOracle;
    std::vector<Mat> dk;
    for (int j = 0; j < p; ++j) dk.push_back(from_ptr(dks + static_cast<size_t>(j) * static_cast<size_t>(n * n), n, n));
    o->o = std::make_unique<DenseMatrixOracle>(from_ptr(k, n, n), std::move(dk));
    return o;
}

void* or_oracle_matern(std::int64_t n, const double* x, int nu2, double sigma2, double ell, double nugget,
                       int scan) {
    auto* o = new OOracle;
    if (guard([&] {
            o->o = std::make_unique<Matern1dOracle>(std::vector<double>(x, x + n), nu2, sigma2, ell, nugget,
                                                    scan != 0);
        })) {
        delete o;
        return nullptr;
    }
    return o;
}

void or_oracle_free(void* o) { delete static_cast<OOracle*>(o); }

int or_oracle_apply(void* op, int which, const double* v, std::int64_t s, double* y) {
    return guard([&] {
        auto& o = *static_cast<OOracle*>(op)->o;
        Mat vm = from_ptr(v, o.dim(), s);
        to_ptr(which < 0 ? o.apply(vm) : o.apply_derivative(which, vm), y);
    });
}

int or_oracle_counters(void* op, std::uint64_t* apply_cols, std::uint64_t* deriv_cols, int reset) {
    auto& o = *static_cast<OOracle*>(op)->o;
    *apply_cols = o.apply_columns();
    *deriv_cols = o.derivative_columns();
    if (reset) o.reset_counters();
    return 0;
}

// ------------------------------------------------------------------ build
void* or_build(void* op, int tau, std::int64_t k, std::uint64_t seed, int with_deriv) {
    auto* o = new OBuild;
    if (guard([&] {
            auto& orc = *static_cast<OOracle*>(op)->o;
            ClusterTree tree(orc.dim(), tau);
            SketchPlan plan(tree, k, seed);
            o->r = build_impl(orc, tree, k, plan, with_deriv != 0);
        })) {
        delete o;
        return nullptr;
    }
    return o;
}

void or_build_free(void* b) { delete static_cast<OBuild*>(b); }

void* or_build_h(void* b) { return new OHodlr{static_cast<OBuild*>(b)->r.h}; }
void* or_build_deriv(void* b, int j) { return new OHodlr{static_cast<OBuild*>(b)->r.deriv[static_cast<size_t>(j)]}; }
int or_build_num_warnings(void* b) { return int(static_cast<OBuild*>(b)->r.warnings.size()); }

/// Per (level, node): numeric_rank, w2, then rw for each param.
int or_build_decisions(void* bp, int p, std::int64_t* out) {
    auto& r = static_cast<OBuild*>(bp)->r;
    size_t o = 0;
    for (const auto& d : r.decisions) {
        out[o++] = d.numeric_rank;
        out[o++] = d.w2;
        for (int j = 0; j < p; ++j) out[o++] = j < int(d.rw.size()) ? d.rw[static_cast<size_t>(j)] : 0;
    }
    return int(r.decisions.size());
}

// -------------------------------------------------------------------- mle
int or_log_likelihood(void* fp, const double* y, const double* ybar, double* out) {
    return guard([&] {
        auto& f = static_cast<OFactor*>(fp)->f;
        *out = log_likelihood(f, from_ptr(y, f.size(), 1), ybar ? from_ptr(ybar, f.size(), 1) : Mat());
    });
}

int or_score(void* fp, void** derivs, int p, const double* y, const double* ybar, double* out) {
    return guard([&] {
        auto& f = static_cast<OFactor*>(fp)->f;
        std::vector<HodlrMatrix> d;
        for (int j = 0; j < p; ++j) d.push_back(static_cast<OHodlr*>(derivs[j])->h);
        auto s = score(f, d, from_ptr(y, f.size(), 1), ybar ? from_ptr(ybar, f.size(), 1) : Mat());
        for (int j = 0; j < p; ++j) out[j] = s[static_cast<size_t>(j)];
    });
}

int or_fisher(void* fp, void** derivs, int p, int cache, double* out) {
    return guard([&] {
        auto& f = static_cast<OFactor*>(fp)->f;
        std::vector<HodlrMatrix> d;
        for (int j = 0; j < p; ++j) d.push_back(static_cast<OHodlr*>(derivs[j])->h);
        to_ptr(fisher_information(f, d, cache != 0), out);
    });
}

/// One full MLE iteration (acceptance.cpp:297-308) with the
/// reference bench's stage names (tools/hodlr_gp.cpp:425-450). times[]:
/// build_deriv, factorize, loglik, score, fisher (seconds).
int or_mle_iteration(void* op, int tau, std::int64_t k, std::uint64_t seed, const double* y, int cache,
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
        Mat ym = from_ptr(y, tree.size(), 1);
        *loglik = log_likelihood(f, ym, Mat());
        auto t3 = clk::now();
        auto s = score(f, br.deriv, ym, Mat());
        for (size_t j = 0; j < s.size(); ++j) score_out[j] = s[j];
        auto t4 = clk::now();
        to_ptr(fisher_information(f, br.deriv, cache != 0), fisher_out);
        auto t5 = clk::now();
        auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
        times[0] = sec(t0, t1);
        times[1] = sec(t1, t2);
        times[2] = sec(t2, t3);
        times[3] = sec(t3, t4);
        times[4] = sec(t4, t5);
    });
}

/// Deterministic N(0,1) fill, row-major over an r x c col-major output.
void or_randn(std::int64_t r, std::int64_t c, std::uint64_t seed, double* out) { to_ptr(randn(r, c, seed), out); }

}  // extern "C"
