// extern "C" boundary (include/hodlrgp_b200.h) over the device hot path.
#include <cuda_runtime.h>

#include <chrono>
#include <functional>
#include <string>

#include "../../include/hodlrgp_b200.h"
#include "api.cuh"
#include "io.cuh"

using namespace hg;

struct hg_ctx_s {
    Ctx c;
};
struct hg_hodlr_s {
    DHodlr h;
};
struct hg_factor_s {
    DFactor f;
};
struct hg_prodrep_s {
    DProductRep p;
};
struct hg_oracle_s {
    std::unique_ptr<DOracle> o;
};
static_assert(sizeof(hg_apply_fn) == sizeof(ApplyFn), "callback ABI");
struct hg_build_s {
    DBuildResult r;
};

namespace {

thread_local std::string g_err;

struct Scope {
    Ctx* prev;
    explicit Scope(hg_ctx_t ctx) : prev(&current()) {
        if (ctx) {
            cudaSetDevice(ctx->c.device);
            set_current(&ctx->c);
        }
    }
    ~Scope() { set_current(prev); }
};

template <class F>
hg_status guard(hg_ctx_t ctx, F&& f) {
    try {
        Scope s(ctx);
        f();
        return HG_OK;
    } catch (const NotPositiveDefinite& e) {
        g_err = e.what();
        return HG_NOT_SPD;
    } catch (const CudaError& e) {
        g_err = e.what();
        return HG_ECUDA;
    } catch (const IoError& e) {
        g_err = e.what();
        return HG_EIO;
    } catch (const std::bad_alloc& e) {
        g_err = e.what();
        return HG_ENOMEM;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return HG_EINVAL;
    } catch (const std::length_error& e) {
        g_err = e.what();
        return HG_ELENGTH;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return HG_ELOGIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return HG_EOTHER;
    }
}

/// Stage a host or device n x s block on the device.
struct Staged {
    DVec buf;
    const double* ptr;
    i64 ld;
    Staged(const double* p, i64 ldp, i64 rows, i64 s, int loc) {
        if (loc == HG_DEVICE) {
            ptr = p;
            ld = ldp;
            return;
        }
        buf.alloc(static_cast<size_t>(rows) * static_cast<size_t>(s));
        if (rows * s)
            HG_CUDA(cudaMemcpy2DAsync(buf.get(), static_cast<size_t>(rows) * sizeof(double), p, static_cast<size_t>(ldp) * sizeof(double),
                                      static_cast<size_t>(rows) * sizeof(double), static_cast<size_t>(s), cudaMemcpyHostToDevice,
                                      current().stream));
        ptr = buf.get();
        ld = rows;
    }
};

struct Output {
    DVec buf;
    double* dptr;
    i64 ld;
    double* host;
    i64 ldh, rows, s;
    Output(double* p, i64 ldp, i64 r, i64 cols, int loc) : host(nullptr), ldh(ldp), rows(r), s(cols) {
        if (loc == HG_DEVICE) {
            dptr = p;
            ld = ldp;
            return;
        }
        buf.alloc(static_cast<size_t>(r) * static_cast<size_t>(cols));
        dptr = buf.get();
        ld = r;
        host = p;
    }
    void finish() {
        if (host && rows * s)
            HG_CUDA(cudaMemcpy2DAsync(host, static_cast<size_t>(ldh) * sizeof(double), dptr, static_cast<size_t>(rows) * sizeof(double),
                                      static_cast<size_t>(rows) * sizeof(double), static_cast<size_t>(s), cudaMemcpyDeviceToHost,
                                      current().stream));
        sync();
    }
};

double scalar_result(const std::function<void(double*)>& f) {
    DVec d(1);
    f(d.get());
    return read_scalar(d.get());
}

}  // namespace

namespace hg {
hg_status capi_guard(hg_ctx_t ctx, const std::function<void()>& f) { return guard(ctx, f); }
}  // namespace hg

extern "C" {

const char* hg_last_error(void) { return g_err.c_str(); }

hg_status hg_ctx_create(int device, void* stream, hg_ctx_t* out) {
    auto* c = new hg_ctx_s;
    hg_status st = guard(nullptr, [&] {
        HG_CUDA(cudaSetDevice(device));
        c->c.device = device;
        if (stream) {
            c->c.stream = static_cast<cudaStream_t>(stream);
        } else {
            HG_CUDA(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
            c->c.own_stream = true;
        }
        dev_stream_adopt(c->c.stream);
        HG_CUDA(cudaDeviceGetAttribute(&c->c.num_sms, cudaDevAttrMultiProcessorCount, device));
        // Keep freed blocks in the stream-ordered pool (no trimming between calls).
        cudaMemPool_t pool;
        HG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        std::uint64_t thr = ~std::uint64_t(0);
        HG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    });
    if (st != HG_OK) {
        delete c;
        return st;
    }
    *out = c;
    return HG_OK;
}

hg_status hg_ctx_destroy(hg_ctx_t ctx) {
    return guard(ctx, [&] {
        HG_CUDA(cudaStreamSynchronize(ctx->c.stream));
        if (ctx->c.own_stream) {
            dev_stream_retire(ctx->c.stream);
            cudaStreamSynchronize(ctx->c.stream);
            cudaStreamDestroy(ctx->c.stream);
        }
        set_current(nullptr);
        delete ctx;
    });
}

hg_status hg_ctx_synchronize(hg_ctx_t ctx) { return guard(ctx, [&] { sync(); }); }
uint64_t hg_ctx_launches(hg_ctx_t ctx) { return ctx->c.launches; }
void* hg_ctx_stream(hg_ctx_t ctx) { return ctx->c.stream; }

hg_status hg_ctx_set_option(hg_ctx_t ctx, int option, int value) {
    return guard(nullptr, [&] {
        if (!ctx) throw std::invalid_argument("hg_ctx_set_option: null context");
        if (option == HG_OPT_PRODUCT_ASSOCIATION && (value == HG_ASSOC_SOLVE || value == HG_ASSOC_REFERENCE))
            ctx->c.product_assoc = value;
        else if (option == HG_OPT_COMPRESSION && (value == HG_COMPRESS_PIVOTED_QR || value == HG_COMPRESS_JACOBI_SVD))
            ctx->c.compression = value;
        else if (option == HG_OPT_Q2_BASIS && (value == HG_Q2_REORTHOGONALIZED || value == HG_Q2_REFERENCE))
            ctx->c.q2_basis = value;
        else if (option == HG_OPT_COMPRESS_AT && (value == HG_COMPRESS_AT_LEVEL || value == HG_COMPRESS_AT_END))
            ctx->c.compress_at = value;
        else if (option == HG_OPT_SKETCH_RNG && (value == HG_SKETCH_RNG_REFERENCE || value == HG_SKETCH_RNG_DEVICE))
            ctx->c.sketch_rng = value;
        else
            throw std::invalid_argument("hg_ctx_set_option: unknown option or value");
    });
}

int hg_ctx_get_option(hg_ctx_t ctx, int option) {
    if (!ctx) return -1;
    if (option == HG_OPT_PRODUCT_ASSOCIATION) return ctx->c.product_assoc;
    if (option == HG_OPT_COMPRESSION) return ctx->c.compression;
    if (option == HG_OPT_Q2_BASIS) return ctx->c.q2_basis;
    if (option == HG_OPT_COMPRESS_AT) return ctx->c.compress_at;
    if (option == HG_OPT_SKETCH_RNG) return ctx->c.sketch_rng;
    return -1;
}

// ------------------------------------------------------------------- tree
int hg_tree_depth(int64_t n, int64_t leaf_min, int64_t leaf_max) { return tree_depth(n, leaf_min, leaf_max); }

hg_status hg_tree_ranges(int64_t n, int tau, int64_t* lo_hi) {
    return guard(nullptr, [&] {
        ClusterTree t(n, tau);
        size_t o = 0;
        for (int d = 0; d <= tau; ++d)
            for (const auto& r : t.level(d)) {
                lo_hi[o++] = r.lo;
                lo_hi[o++] = r.hi;
            }
    });
}

hg_status hg_kd_ordering(int64_t n, int d, const double* coords, int64_t leaf_min, int64_t leaf_max, int64_t* perm,
                         int64_t* inv, int* tau) {
    return guard(nullptr, [&] {
        KdOrdering kd = build_kd_ordering(coords, n, d, leaf_min, leaf_max);
        for (int64_t i = 0; i < n; ++i) {
            perm[i] = kd.perm[static_cast<size_t>(i)];
            inv[i] = kd.inv[static_cast<size_t>(i)];
        }
        *tau = kd.tree.depth();
    });
}

// ------------------------------------------------------------------ hodlr
hg_status hg_hodlr_zero(hg_ctx_t ctx, int64_t n, int tau, int symmetric, hg_hodlr_t* out) {
    return guard(ctx, [&] { *out = new hg_hodlr_s{DHodlr::zero(get_tree(n, tau), symmetric != 0)}; });
}

hg_status hg_hodlr_identity(hg_ctx_t ctx, int64_t n, int tau, hg_hodlr_t* out) {
    return guard(ctx, [&] { *out = new hg_hodlr_s{DHodlr::identity(get_tree(n, tau))}; });
}

hg_status hg_hodlr_random(hg_ctx_t ctx, int64_t n, int tau, int64_t k, uint64_t seed, int spd, hg_hodlr_t* out) {
    return guard(ctx, [&] { *out = new hg_hodlr_s{DHodlr::random(get_tree(n, tau), k, seed, spd != 0)}; });
}

hg_status hg_hodlr_import(hg_ctx_t ctx, int64_t n, int tau, int symmetric, const int* R, const double* flat,
                          const int* ranks_up, const int* ranks_lo, hg_hodlr_t* out) {
    return guard(ctx, [&] {
        *out = new hg_hodlr_s{DHodlr::import_panels(get_tree(n, tau), symmetric != 0, R, flat, ranks_up, ranks_lo)};
    });
}

hg_status hg_hodlr_info(hg_hodlr_t h, int64_t* n, int* tau, int* symmetric, int* R) {
    return guard(nullptr, [&] {
        *n = h->h.n();
        *tau = h->h.tau();
        *symmetric = h->h.sym ? 1 : 0;
        if (R)
            for (int l = 1; l <= h->h.tau(); ++l) R[l - 1] = h->h.Rl(l);
    });
}

int64_t hg_hodlr_export_size(hg_hodlr_t h) { return int64_t(h->h.export_size()); }

hg_status hg_hodlr_export(hg_ctx_t ctx, hg_hodlr_t h, double* flat, int* ranks_up, int* ranks_lo) {
    return guard(ctx, [&] { h->h.export_panels(flat, ranks_up, ranks_lo); });
}

hg_status hg_write_hodlr_debug(hg_ctx_t ctx, const char* dir, const char* name, hg_hodlr_t h) {
    return guard(ctx, [&] {
        if (!dir || !name || !h) throw std::invalid_argument("write_hodlr_debug: null argument");
        write_hodlr_debug(dir, name, h->h);
    });
}

hg_status hg_read_hodlr_debug(hg_ctx_t ctx, const char* dir, const char* name, hg_hodlr_t* out) {
    return guard(ctx, [&] {
        if (!dir || !name || !out) throw std::invalid_argument("read_hodlr_debug: null argument");
        *out = new hg_hodlr_s{read_hodlr_debug(dir, name)};
    });
}

hg_status hg_hodlr_copy(hg_ctx_t ctx, hg_hodlr_t h, hg_hodlr_t* out) {
    return guard(ctx, [&] { *out = new hg_hodlr_s{hodlr_deep_copy(h->h)}; });
}

hg_status hg_hodlr_free(hg_hodlr_t h) {
    delete h;
    return HG_OK;
}

hg_status hg_hodlr_make_asymmetric(hg_ctx_t ctx, hg_hodlr_t h) {
    return guard(ctx, [&] { h->h.make_asymmetric(); });
}

hg_status hg_hodlr_matvec(hg_ctx_t ctx, hg_hodlr_t h, const double* X, int64_t ldx, int64_t s, double* Y,
                          int64_t ldy, int loc) {
    return guard(ctx, [&] {
        const i64 n = h->h.n();
        if (ldx < n || ldy < n) throw std::invalid_argument("matvec: dimension mismatch");
        Staged x(X, ldx, n, s, loc);
        Output y(Y, ldy, n, s, loc);
        hodlr_apply(h->h, x.ptr, x.ld, int(s), y.dptr, y.ld, 1, h->h.tau(), true, false, 0.0);
        y.finish();
    });
}

hg_status hg_hodlr_sub_matvec(hg_ctx_t ctx, hg_hodlr_t h, int d, int64_t node, const double* X, int64_t ldx,
                              int64_t s, int transpose, double* Y, int64_t ldy, int loc) {
    return guard(ctx, [&] {
        const auto& tree = h->h.tree->host;
        if (d < 0 || d > tree.depth() || node < 0 || node >= i64(tree.level(d).size()))
            throw std::invalid_argument("sub_matvec: node out of range");
        const Range r = tree.level(d)[static_cast<size_t>(node)];
        const i64 n = h->h.n();
        Staged x(X, ldx, r.size(), s, loc);
        DVec full(static_cast<size_t>(n) * static_cast<size_t>(s)), yf(static_cast<size_t>(n) * static_cast<size_t>(s));
        full.zero();
        HG_CUDA(cudaMemcpy2DAsync(full.get() + r.lo, static_cast<size_t>(n) * sizeof(double), x.ptr, static_cast<size_t>(x.ld) * sizeof(double),
                                  static_cast<size_t>(r.size()) * sizeof(double), static_cast<size_t>(s), cudaMemcpyDeviceToDevice,
                                  current().stream));
        hodlr_apply(h->h, full.get(), n, int(s), yf.get(), n, d + 1, h->h.tau(), true, transpose != 0, 0.0);
        Output y(Y, ldy, r.size(), s, loc);
        HG_CUDA(cudaMemcpy2DAsync(y.dptr, static_cast<size_t>(y.ld) * sizeof(double), yf.get() + r.lo, static_cast<size_t>(n) * sizeof(double),
                                  static_cast<size_t>(r.size()) * sizeof(double), static_cast<size_t>(s), cudaMemcpyDeviceToDevice,
                                  current().stream));
        y.finish();
    });
}

hg_status hg_hodlr_trace(hg_ctx_t ctx, hg_hodlr_t h, double* out) {
    return guard(ctx, [&] { *out = scalar_result([&](double* d) { hodlr_trace(h->h, d, false); }); });
}

hg_status hg_trace_product(hg_ctx_t ctx, hg_hodlr_t a, hg_hodlr_t b, double* out) {
    return guard(ctx, [&] { *out = scalar_result([&](double* d) { hodlr_trace_product(a->h, b->h, d, false); }); });
}

// ---------------------------------------------------------- factorization
hg_status hg_factorize(hg_ctx_t ctx, hg_hodlr_t h, int orientation, hg_factor_t* out) {
    return guard(ctx, [&] {
        if (orientation != HG_RIGHT && orientation != HG_LEFT) throw std::invalid_argument("factorize: orientation");
        *out = new hg_factor_s{factorize(h->h, orientation)};
    });
}

hg_status hg_factor_free(hg_factor_t f) {
    delete f;
    return HG_OK;
}

hg_status hg_factor_solve(hg_ctx_t ctx, hg_factor_t f, const double* B, int64_t ldb, int64_t s, double* X,
                          int64_t ldx, int loc) {
    return guard(ctx, [&] {
        const i64 n = f->f.n();
        if (ldb < n || ldx < n) throw std::invalid_argument("solve: dimension mismatch");
        Output y(X, ldx, n, s, loc);
        if (!(loc == HG_DEVICE && B == X && ldb == ldx))
            HG_CUDA(cudaMemcpy2DAsync(y.dptr, static_cast<size_t>(y.ld) * sizeof(double), B, static_cast<size_t>(ldb) * sizeof(double),
                                      static_cast<size_t>(n) * sizeof(double), static_cast<size_t>(s),
                                      loc == HG_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                      current().stream));
        factor_solve(f->f, y.dptr, y.ld, int(s));
        y.finish();
    });
}

hg_status hg_factor_logdet(hg_ctx_t ctx, hg_factor_t f, double* out) {
    return guard(ctx, [&] { *out = factor_logdet(f->f); });
}

hg_status hg_factor_leaf_llt(hg_ctx_t ctx, hg_factor_t f, int* out) {
    return guard(ctx, [&] {
        auto k = leaf_kinds(f->f);
        for (size_t i = 0; i < k.size(); ++i) out[i] = k[i];
    });
}

// ---------------------------------------------------------- trace algebra
hg_status hg_multiply(hg_ctx_t ctx, hg_factor_t f, hg_hodlr_t b, hg_prodrep_t* out) {
    return guard(ctx, [&] { *out = new hg_prodrep_s{pipeline(f->f, b->h, false)}; });
}

hg_status hg_solve_multiply(hg_ctx_t ctx, hg_factor_t f, hg_hodlr_t b, hg_prodrep_t* out) {
    return guard(ctx, [&] { *out = new hg_prodrep_s{pipeline(f->f, b->h, true)}; });
}

hg_status hg_prodrep_free(hg_prodrep_t p) {
    delete p;
    return HG_OK;
}

hg_status hg_prodrep_densify(hg_ctx_t ctx, hg_prodrep_t p, double* out) {
    return guard(ctx, [&] {
        auto a = prodrep_densify(p->p);
        std::memcpy(out, a.data(), a.size() * sizeof(double));
    });
}

hg_status hg_trace_product_rep(hg_ctx_t ctx, hg_prodrep_t p, double* out) {
    return guard(ctx, [&] { *out = scalar_result([&](double* d) { trace_product_rep(p->p, d, false); }); });
}

hg_status hg_trace_pair(hg_ctx_t ctx, hg_prodrep_t p, hg_prodrep_t q, double* out) {
    return guard(ctx, [&] {
        if (!p->p.base.tree->host.same_structure(q->p.base.tree->host))
            throw std::invalid_argument("trace_pair: tree mismatch");
        *out = scalar_result([&](double* d) { trace_pair(p->p, q->p, d, false); });
    });
}

hg_status hg_trace_solve(hg_ctx_t ctx, hg_factor_t f, hg_hodlr_t b, double* out) {
    return guard(ctx, [&] {
        DProductRep r = pipeline(f->f, b->h, true);
        *out = scalar_result([&](double* d) { trace_product_rep(r, d, false); });
    });
}

hg_status hg_hutchinson_trace(hg_ctx_t ctx, hg_factor_t f, hg_hodlr_t b, int n_samples, uint64_t seed,
                              double* estimate, double* std_error) {
    return guard(ctx, [&] {
        const auto r = hutchinson_trace(f->f, b->h, n_samples, seed);
        *estimate = r.first;
        *std_error = r.second;
    });
}

hg_status hg_trace_quad(hg_ctx_t ctx, hg_factor_t fa, hg_hodlr_t b, hg_factor_t fc, hg_hodlr_t d, double* out) {
    return guard(ctx, [&] {
        DProductRep p = pipeline(fa->f, b->h, true);
        DProductRep q = pipeline(fc->f, d->h, true);
        *out = scalar_result([&](double* x) { trace_pair(p, q, x, false); });
    });
}

}  // extern "C"

extern "C" {

// ------------------------------------------------------------------ oracle
hg_status hg_oracle_dense(hg_ctx_t ctx, int64_t n, const double* K, int p, const double* dK, hg_oracle_t* out) {
    return guard(ctx, [&] { *out = new hg_oracle_s{make_dense_oracle(n, K, p, dK)}; });
}

hg_status hg_oracle_matern(hg_ctx_t ctx, int64_t n, const double* x, int nu2, double sigma2, double ell,
                           double nugget, int scan, hg_oracle_t* out) {
    return guard(ctx, [&] { *out = new hg_oracle_s{make_matern_oracle(n, x, nu2, sigma2, ell, nugget, scan != 0)}; });
}

hg_status hg_oracle_cokriging(hg_ctx_t ctx, int64_t m, double sigma2, double ell, double kappa, double nugget,
                              hg_oracle_t* out) {
    return guard(ctx, [&] { *out = new hg_oracle_s{make_cokriging_oracle(m, sigma2, ell, kappa, nugget)}; });
}

hg_status hg_oracle_spde2d(hg_ctx_t ctx, int nside, double sigma2, double ell, double kappa, double nugget,
                           const int64_t* order, hg_oracle_t* out) {
    return guard(ctx, [&] { *out = new hg_oracle_s{make_spde2d_oracle(nside, sigma2, ell, kappa, nugget, order)}; });
}

hg_status hg_oracle_callback(hg_ctx_t ctx, int64_t n, int p, hg_apply_fn fn, void* user, hg_oracle_t* out) {
    return guard(ctx, [&] { *out = new hg_oracle_s{make_callback_oracle(n, p, reinterpret_cast<ApplyFn>(fn), user)}; });
}

hg_status hg_oracle_permuted(hg_ctx_t ctx, hg_oracle_t base, const int64_t* to_base, hg_oracle_t* out) {
    return guard(ctx, [&] {
        if (!base) throw std::invalid_argument("hg_oracle_permuted: null base oracle");
        *out = new hg_oracle_s{make_permuted_oracle(base->o.get(), to_base)};
    });
}

hg_status hg_oracle_set_parameters(hg_oracle_t o, const double* theta, int p) {
    return guard(nullptr, [&] { o->o->set_parameters(theta, p); });
}

hg_status hg_oracle_free(hg_oracle_t o) {
    delete o;
    return HG_OK;
}

hg_status hg_oracle_apply(hg_ctx_t ctx, hg_oracle_t o, int j, const double* V, int64_t ldv, int64_t s, double* Y,
                          int64_t ldy, int loc) {
    return guard(ctx, [&] {
        const i64 n = o->o->dim();
        if (ldv < n || ldy < n) throw std::invalid_argument("oracle apply: dimension mismatch");
        Staged v(V, ldv, n, s, loc);
        Output y(Y, ldy, n, s, loc);
        o->o->apply(j, v.ptr, v.ld, int(s), y.dptr, y.ld);
        y.finish();
    });
}

hg_status hg_oracle_counters(hg_oracle_t o, uint64_t* apply_columns, uint64_t* derivative_columns, int reset) {
    *apply_columns = o->o->apply_columns();
    *derivative_columns = o->o->derivative_columns();
    if (reset) o->o->reset_counters();
    return HG_OK;
}

// ------------------------------------------------------------------- build
hg_status hg_build(hg_ctx_t ctx, hg_oracle_t o, int tau, int64_t k, uint64_t seed, int with_derivatives,
                   hg_build_t* out) {
    return guard(ctx, [&] {
        DTreeP tree = get_tree(o->o->dim(), tau);
        DSketchPlanP plan = get_plan(tree, k, seed);
        *out = new hg_build_s{build(*o->o, tree, k, *plan, with_derivatives != 0)};
        sync();
    });
}

hg_status hg_build_free(hg_build_t b) {
    delete b;
    return HG_OK;
}

hg_status hg_build_h(hg_build_t b, hg_hodlr_t* out) {
    return guard(nullptr, [&] { *out = new hg_hodlr_s{b->r.h}; });
}

hg_status hg_build_deriv(hg_build_t b, int j, hg_hodlr_t* out) {
    return guard(nullptr, [&] {
        if (j < 0 || j >= int(b->r.deriv.size())) throw std::invalid_argument("build_deriv: index");
        *out = new hg_hodlr_s{b->r.deriv[static_cast<size_t>(j)]};
    });
}

int hg_build_num_warnings(hg_build_t b) { return b->r.warnings; }

int hg_build_decisions(hg_build_t b, int p, int64_t* out) {
    const int stride = 2 + b->r.p;
    const size_t cnt = b->r.decisions.size() / static_cast<size_t>(stride);
    for (size_t i = 0; i < cnt; ++i)
        for (int c = 0; c < 2 + p; ++c)
            out[i * static_cast<size_t>(2 + p) + static_cast<size_t>(c)] = c < stride ? b->r.decisions[i * static_cast<size_t>(stride) + static_cast<size_t>(c)] : 0;
    return int(cnt);
}

// --------------------------------------------------------------------- mle
namespace {
DVec residual(const double* y, const double* ybar, i64 n) {
    std::vector<double> r(y, y + n);
    if (ybar)
        for (i64 i = 0; i < n; ++i) r[static_cast<size_t>(i)] -= ybar[i];
    DVec d;
    d.upload(r);
    return d;
}
}  // namespace

hg_status hg_log_likelihood(hg_ctx_t ctx, hg_factor_t f, const double* y, const double* ybar, double* out) {
    return guard(ctx, [&] {
        DVec r = residual(y, ybar, f->f.n());
        *out = log_likelihood(f->f, r.get());
    });
}

hg_status hg_score(hg_ctx_t ctx, hg_factor_t f, const hg_hodlr_t* deriv, int p, const double* y, const double* ybar,
                   double* out) {
    return guard(ctx, [&] {
        DVec r = residual(y, ybar, f->f.n());
        std::vector<const DHodlr*> d;
        for (int j = 0; j < p; ++j) d.push_back(&deriv[j]->h);
        auto s = score(f->f, d, r.get(), nullptr);
        for (int j = 0; j < p; ++j) out[j] = s[static_cast<size_t>(j)];
    });
}

hg_status hg_fisher_information(hg_ctx_t ctx, hg_factor_t f, const hg_hodlr_t* deriv, int p, double* out) {
    return guard(ctx, [&] {
        std::vector<const DHodlr*> d;
        for (int j = 0; j < p; ++j) d.push_back(&deriv[j]->h);
        auto fi = fisher_from_reps(pipeline_multi(f->f, d, true));
        for (size_t i = 0; i < fi.size(); ++i) out[i] = fi[i];
    });
}

hg_status hg_mle_iteration(hg_ctx_t ctx, hg_oracle_t o, int tau, int64_t k, uint64_t seed, const double* y,
                           double* loglik, double* score_out, double* fisher, double* times) {
    return guard(ctx, [&] {
        auto& c = current();
        const i64 n = o->o->dim();
        DTreeP tree = get_tree(n, tau);
        DSketchPlanP plan = get_plan(tree, k, seed);
        cudaEvent_t ev[6];
        for (auto& e : ev) HG_CUDA(cudaEventCreate(&e));
        DVec r = residual(y, nullptr, n);
        HG_CUDA(cudaEventRecord(ev[0], c.stream));
        DBuildResult br = build(*o->o, tree, k, *plan, true);
        HG_CUDA(cudaEventRecord(ev[1], c.stream));
        DFactor f = factorize(br.h, HG_LEFT);
        HG_CUDA(cudaEventRecord(ev[2], c.stream));
        *loglik = log_likelihood(f, r.get());
        HG_CUDA(cudaEventRecord(ev[3], c.stream));
        std::vector<const DHodlr*> d;
        for (auto& x : br.deriv) d.push_back(&x);
        std::vector<DProductRep> reps;
        auto s = score(f, d, r.get(), &reps);
        for (size_t j = 0; j < s.size(); ++j) score_out[j] = s[j];
        HG_CUDA(cudaEventRecord(ev[4], c.stream));
        auto fi = fisher_from_reps(reps);
        for (size_t i = 0; i < fi.size(); ++i) fisher[i] = fi[i];
        HG_CUDA(cudaEventRecord(ev[5], c.stream));
        HG_CUDA(cudaEventSynchronize(ev[5]));
        for (int i = 0; i < 5; ++i) {
            float ms = 0;
            HG_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
            times[i] = ms * 1e-3;
        }
        for (auto& e : ev) cudaEventDestroy(e);
    });
}

}  // extern "C"
