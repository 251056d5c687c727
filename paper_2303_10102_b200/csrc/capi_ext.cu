// C ABI: full MLE evaluation on host or device buffers, per-kernel profiling.
#include <cuda_runtime.h>

#include <functional>

#include "../../include/hodlrgp_b200.h"
#include "api.cuh"
#include "dense.cuh"
#include "fit.cuh"
#include "prof.cuh"

using namespace hg;

// Handle layouts shared with capi.cu.
struct hg_ctx_s {
    Ctx c;
};
struct hg_oracle_s {
    std::unique_ptr<DOracle> o;
};

namespace hg {
hg_status capi_guard(hg_ctx_t ctx, const std::function<void()>& f);
}

extern "C" {

hg_status hg_mle_evaluate(hg_ctx_t ctx, hg_oracle_t o, int tau, int64_t k, uint64_t seed, const double* y,
                          const double* B, int64_t nrhs, double* X, int loc, double* loglik, double* score_out,
                          double* fisher, double* times) {
    return capi_guard(ctx, [&] {
        auto& c = current();
        const i64 n = o->o->dim();
        DTreeP tree = get_tree(n, tau);
        DSketchPlanP plan = get_plan(tree, k, seed);
        cudaEvent_t ev[7];
        for (auto& e : ev) HG_CUDA(cudaEventCreate(&e));
        HG_CUDA(cudaEventRecord(ev[0], c.stream));
        // inputs (host -> device when loc == HG_HOST)
        DVec ybuf, Bbuf;
        const double* yd = y;
        const double* Bd = B;
        if (loc == HG_HOST) {
            ybuf.upload(y, size_t(n));
            yd = ybuf.get();
            if (nrhs > 0) {
                Bbuf.upload(B, size_t(n) * size_t(nrhs));
                Bd = Bbuf.get();
            }
        }
        DBuildResult br = build(*o->o, tree, k, *plan, true);
        HG_CUDA(cudaEventRecord(ev[1], c.stream));
        DFactor f = factorize(br.h, HG_LEFT);
        HG_CUDA(cudaEventRecord(ev[2], c.stream));
        *loglik = log_likelihood(f, yd);
        if (nrhs > 0) {  // the seeded right-hand sides (BASELINE.json C4)
            DVec Xd(size_t(n) * size_t(nrhs));
            panel_axpby(n, int(nrhs), 1.0, Bd, n, 0.0, Xd.get(), n);
            factor_solve(f, Xd.get(), n, int(nrhs));
            HG_CUDA(cudaMemcpyAsync(X, Xd.get(), sizeof(double) * size_t(n) * size_t(nrhs),
                                    loc == HG_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c.stream));
        }
        HG_CUDA(cudaEventRecord(ev[3], c.stream));
        std::vector<const DHodlr*> d;
        for (auto& x : br.deriv) d.push_back(&x);
        std::vector<DProductRep> reps;
        auto s = score(f, d, yd, &reps);
        for (size_t j = 0; j < s.size(); ++j) score_out[j] = s[j];
        HG_CUDA(cudaEventRecord(ev[4], c.stream));
        auto fi = fisher_from_reps(reps);
        for (size_t i = 0; i < fi.size(); ++i) fisher[i] = fi[i];
        HG_CUDA(cudaEventRecord(ev[5], c.stream));
        HG_CUDA(cudaEventSynchronize(ev[5]));
        if (times)
            for (int i = 0; i < 5; ++i) {
                float ms = 0;
                HG_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
                times[i] = ms * 1e-3;
            }
        for (auto& e : ev) cudaEventDestroy(e);
    });
}

namespace {
/// Device copy of a host (loc = HG_HOST) or device rows x cols block.
struct In {
    DVec buf;
    const double* p;
    i64 ld;
    In(const double* src, i64 lds, i64 rows, i64 cols, int loc) {
        if (loc == HG_DEVICE) {
            p = src;
            ld = lds;
            return;
        }
        buf.alloc(static_cast<size_t>(rows * cols));
        if (rows * cols)
            HG_CUDA(cudaMemcpy2DAsync(buf.get(), sizeof(double) * rows, src, sizeof(double) * lds, sizeof(double) * rows,
                                      static_cast<size_t>(cols), cudaMemcpyHostToDevice, current().stream));
        p = buf.get();
        ld = rows;
    }
};
/// Device destination; copied back to the host by finish().
struct Out {
    DVec buf;
    double* p;
    i64 ld;
    double* host;
    i64 ldh, rows, cols;
    Out(double* dst, i64 ldd, i64 r, i64 c, int loc) : host(nullptr), ldh(ldd), rows(r), cols(c) {
        if (loc == HG_DEVICE) {
            p = dst;
            ld = ldd;
            return;
        }
        buf.alloc(static_cast<size_t>(r * c));
        p = buf.get();
        ld = r;
        host = dst;
    }
    void finish() {
        if (host && rows * cols)
            HG_CUDA(cudaMemcpy2DAsync(host, sizeof(double) * ldh, p, sizeof(double) * rows, sizeof(double) * rows,
                                      static_cast<size_t>(cols), cudaMemcpyDeviceToHost, current().stream));
    }
};
}  // namespace

hg_status hg_randomized_range(hg_ctx_t ctx, const double* y, int64_t ldy, int64_t rows, int64_t k, double* q,
                              int64_t ldq, double* r, int* perm, int64_t* numeric_rank, int loc) {
    return capi_guard(ctx, [&] {
        In Y(y, ldy, rows, k, loc);
        Out Q(q, ldq, rows, k, loc);
        DVec R(static_cast<size_t>(k * k));
        DBuf<int> P(static_cast<size_t>(k)), nr(1);
        randomized_range(Y.p, Y.ld, int(rows), int(k), Q.p, Q.ld, R.get(), P.get(), nr.get());
        Q.finish();
        std::vector<double> rh = R.download();
        std::vector<int> ph = P.download(), nh = nr.download();
        std::copy(rh.begin(), rh.end(), r);
        std::copy(ph.begin(), ph.end(), perm);
        *numeric_rank = nh[0];
    });
}

hg_status hg_diff_qr(hg_ctx_t ctx, const double* db, int64_t lddb, const double* q, int64_t ldq, const double* r,
                     int64_t rows, int64_t k, double* dq, int64_t lddq, double* dq_span, int64_t ldds, double* dr,
                     int* ill_conditioned, int loc) {
    return capi_guard(ctx, [&] {
        In dB(db, lddb, rows, k, loc), Q(q, ldq, rows, k, loc);
        DVec R;
        R.upload(r, static_cast<size_t>(k * k));
        Out dQ(dq, lddq, rows, k, loc), dS(dq_span, ldds, rows, k, loc);
        DVec dR(static_cast<size_t>(k * k));
        DBuf<int> ill(1);
        diff_qr(dB.p, dB.ld, Q.p, Q.ld, R.get(), int(rows), int(k), dQ.p, dQ.ld, dS.p, dS.ld, dR.get(), ill.get());
        dQ.finish();
        dS.finish();
        std::vector<double> rh = dR.download();
        std::copy(rh.begin(), rh.end(), dr);
        *ill_conditioned = ill.download()[0];
    });
}

hg_status hg_sketch_sampler(hg_ctx_t ctx, int64_t n, int tau, int64_t k, uint64_t seed, int level, double* out,
                            int64_t ldo, int loc) {
    return capi_guard(ctx, [&] {
        DTreeP tree = get_tree(n, tau);
        DSketchPlanP plan = get_plan(tree, k, seed);
        if (level < 0 || level > tau) throw std::invalid_argument("sketch_sampler: level in [0, tau]");
        const double* src = level == 0 ? plan->leaf->get() : plan->level[static_cast<size_t>(level - 1)]->get();
        const i64 cols = level == 0 ? tree->bmax : k;
        Out o(out, ldo, n, cols, loc);
        panel_axpby(n, int(cols), 1.0, src, n, 0.0, o.p, o.ld);
        o.finish();
        sync();
    });
}

hg_status hg_fit_mle(hg_ctx_t ctx, hg_oracle_t o, int tau, int64_t k, uint64_t seed, const double* y,
                     const double* ybar, int p, const int* transforms, const double* theta0, int max_iter,
                     double rel_tol, int dense, double* theta_hat, double* fisher, double* ci, int* ci_valid, int* iterations,
                     int* converged, char* status, int status_len, double* loglik_trace, double* grad_norm_trace,
                     double* theta_trace, int trace_cap, int* trace_len, uint64_t* columns, double* seconds) {
    return capi_guard(ctx, [&] {
        const i64 n = o->o->dim();
        std::vector<double> r(y, y + n);
        if (ybar)
            for (i64 i = 0; i < n; ++i) r[static_cast<size_t>(i)] -= ybar[i];
        DVec rd;
        rd.upload(r);
        FitReport rep = fit_mle(*o->o, get_tree(n, tau), k, seed, rd.get(), std::vector<int>(transforms, transforms + p),
                                std::vector<double>(theta0, theta0 + p), max_iter, rel_tol, dense != 0);
        for (int i = 0; i < p; ++i) theta_hat[i] = rep.theta_hat[static_cast<size_t>(i)];
        for (int i = 0; i < p * p; ++i) fisher[i] = rep.fisher.empty() ? NAN : rep.fisher[static_cast<size_t>(i)];
        for (int i = 0; i < 2 * p; ++i) ci[i] = rep.ci.empty() ? NAN : rep.ci[static_cast<size_t>(i)];
        *ci_valid = rep.ci_valid ? 1 : 0;
        *iterations = rep.iterations;
        *converged = rep.converged ? 1 : 0;
        if (status && status_len > 0) {
            const size_t m = std::min(rep.status.size(), size_t(status_len - 1));
            std::copy(rep.status.begin(), rep.status.begin() + m, status);
            status[m] = 0;
        }
        const int len = int(std::min<size_t>(rep.loglik_trace.size(), size_t(std::max(trace_cap, 0))));
        for (int t = 0; t < len; ++t) {
            if (loglik_trace) loglik_trace[t] = rep.loglik_trace[static_cast<size_t>(t)];
            if (grad_norm_trace) grad_norm_trace[t] = rep.grad_norm_trace[static_cast<size_t>(t)];
            if (theta_trace)
                for (int i = 0; i < p; ++i) theta_trace[i + t * p] = rep.theta_trace[static_cast<size_t>(t)][static_cast<size_t>(i)];
        }
        *trace_len = len;
        columns[0] = rep.apply_columns;
        columns[1] = rep.derivative_columns;
        *seconds = rep.seconds;
    });
}

hg_status hg_dense_exact(hg_ctx_t ctx, hg_oracle_t o, const double* y, const double* ybar, double* loglik,
                         double* score_out, double* fisher) {
    return capi_guard(ctx, [&] {
        const i64 n = o->o->dim();
        std::vector<double> r(y, y + n);
        if (ybar)
            for (i64 i = 0; i < n; ++i) r[static_cast<size_t>(i)] -= ybar[i];
        DVec rd;
        rd.upload(r);
        DenseExact d = dense_exact(*o->o, rd.get());
        *loglik = d.loglik;
        std::copy(d.score.begin(), d.score.end(), score_out);
        std::copy(d.fisher.begin(), d.fisher.end(), fisher);
    });
}

hg_status hg_accuracy_metrics(int p, double loglik, const double* score_exact, const double* fisher_exact,
                              double loglik_approx, const double* score_approx, const double* fisher_approx,
                              double* out) {
    return capi_guard(nullptr, [&] {
        const size_t pp = static_cast<size_t>(p) * static_cast<size_t>(p);
        AccuracyMetrics m = accuracy_metrics(
            loglik, std::vector<double>(score_exact, score_exact + p), std::vector<double>(fisher_exact, fisher_exact + pp),
            loglik_approx, std::vector<double>(score_approx, score_approx + p),
            std::vector<double>(fisher_approx, fisher_approx + pp));
        out[0] = m.eps_L;
        out[1] = m.eps_S;
        out[2] = m.eps_I;
        out[3] = m.eta_g;
        out[4] = m.eta_I;
    });
}

void hg_prof_enable(int on) { prof_enable(on != 0); }

int hg_prof_read(int reset, double* ms, double* flops, double* bytes, int64_t* launches) {
    auto t = prof_read(reset != 0);
    for (size_t i = 0; i < t.size(); ++i) {
        ms[i] = t[i].ms;
        flops[i] = t[i].flops;
        bytes[i] = t[i].bytes;
        launches[i] = t[i].launches;
    }
    return int(t.size());
}

}  // extern "C"
