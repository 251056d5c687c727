// fit_mle (mle.cpp:188-322) on the device path: BFGS over transformed
// parameters with a backtracking line search, every objective / gradient /
// Fisher evaluation a full HODLR build + factorization on the GPU. The
// p-dimensional quasi-Newton algebra (p <= a handful) stays on the host, as
// in the reference; the SketchPlan is fixed once for the whole fit
// (mle.cpp:195), so the objective is a deterministic function of theta.
#include <chrono>
#include <cmath>
#include <limits>

#include "api.cuh"
#include "fit.cuh"
#include "dense.cuh"

namespace hg {

namespace {

using Vec = std::vector<double>;

double dot(const Vec& a, const Vec& b) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
    return s;
}
double norm(const Vec& a) { return std::sqrt(dot(a, a)); }

// mle.cpp:82-121: theta = exp(u) (positive), tanh(u) (correlation), u.
Vec to_natural(const Vec& u, const std::vector<int>& tr) {
    Vec t(u.size());
    for (size_t i = 0; i < u.size(); ++i)
        t[i] = tr[i] == FIT_POSITIVE ? std::exp(u[i]) : (tr[i] == FIT_CORRELATION ? std::tanh(u[i]) : u[i]);
    return t;
}
Vec from_natural(const Vec& t, const std::vector<int>& tr) {
    Vec u(t.size());
    for (size_t i = 0; i < t.size(); ++i) {
        if (tr[i] == FIT_POSITIVE) {
            if (t[i] <= 0) throw std::invalid_argument("positive parameter required");
            u[i] = std::log(t[i]);
        } else if (tr[i] == FIT_CORRELATION) {
            if (std::abs(t[i]) >= 1) throw std::invalid_argument("|rho| < 1 required");
            u[i] = std::atanh(t[i]);
        } else {
            u[i] = t[i];
        }
    }
    return u;
}
Vec jacobian_diag(const Vec& t, const std::vector<int>& tr) {  // dtheta/du
    Vec d(t.size());
    for (size_t i = 0; i < t.size(); ++i)
        d[i] = tr[i] == FIT_POSITIVE ? t[i] : (tr[i] == FIT_CORRELATION ? 1.0 - t[i] * t[i] : 1.0);
    return d;
}

/// Cholesky solve of a small SPD system; false if not positive definite.
bool chol_solve(std::vector<double> A, int p, Vec& b) {
    for (int j = 0; j < p; ++j) {
        double d = A[j + j * p];
        for (int k = 0; k < j; ++k) d -= A[j + k * p] * A[j + k * p];
        if (!(d > 0)) return false;
        d = std::sqrt(d);
        A[j + j * p] = d;
        for (int i = j + 1; i < p; ++i) {
            double s = A[i + j * p];
            for (int k = 0; k < j; ++k) s -= A[i + k * p] * A[j + k * p];
            A[i + j * p] = s / d;
        }
    }
    for (int i = 0; i < p; ++i) {
        double s = b[i];
        for (int k = 0; k < i; ++k) s -= A[i + k * p] * b[k];
        b[i] = s / A[i + i * p];
    }
    for (int i = p - 1; i >= 0; --i) {
        double s = b[i];
        for (int k = i + 1; k < p; ++k) s -= A[k + i * p] * b[k];
        b[i] = s / A[i + i * p];
    }
    return true;
}

/// Symmetric eigen-decomposition by cyclic Jacobi (p x p, p small).
void sym_eig(std::vector<double> A, int p, Vec& w, std::vector<double>& V) {
    V.assign(static_cast<size_t>(p) * p, 0.0);
    for (int i = 0; i < p; ++i) V[i + i * p] = 1.0;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int i = 0; i < p; ++i)
            for (int j = i + 1; j < p; ++j) off += A[i + j * p] * A[i + j * p];
        if (off < 1e-30) break;
        for (int i = 0; i < p; ++i)
            for (int j = i + 1; j < p; ++j) {
                const double aij = A[i + j * p];
                if (aij == 0.0) continue;
                const double th = (A[j + j * p] - A[i + i * p]) / (2.0 * aij);
                const double t = (th >= 0 ? 1.0 : -1.0) / (std::abs(th) + std::sqrt(th * th + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < p; ++k) {
                    const double akj = A[k + j * p], aki = A[k + i * p];
                    A[k + i * p] = c * aki - s * akj;
                    A[k + j * p] = s * aki + c * akj;
                }
                for (int k = 0; k < p; ++k) {
                    const double ajk = A[j + k * p], aik = A[i + k * p];
                    A[i + k * p] = c * aik - s * ajk;
                    A[j + k * p] = s * aik + c * ajk;
                }
                for (int k = 0; k < p; ++k) {
                    const double vkj = V[k + j * p], vki = V[k + i * p];
                    V[k + i * p] = c * vki - s * vkj;
                    V[k + j * p] = s * vki + c * vkj;
                }
            }
    }
    w.resize(static_cast<size_t>(p));
    for (int i = 0; i < p; ++i) w[i] = A[i + i * p];
}

struct Evaluator {
    DOracle& o;
    DTreeP tree;
    i64 k;
    const DSketchPlan& plan;
    const double* r;  // device residual y - ybar
    bool dense;       // FitOptions::dense (mle.cpp:131-169)

    double value(const Vec& th) const {  // -loglik (line-search probes)
        o.set_parameters(th.data(), int(th.size()));
        if (dense) return dense_objective(o, r);
        DBuildResult br = build(o, tree, k, plan, false);
        DFactor f = factorize(br.h, 1);
        return -log_likelihood(f, r);
    }
    double value_grad(const Vec& th, Vec& grad) const {  // accepted iterates
        o.set_parameters(th.data(), int(th.size()));
        if (dense) return dense_objective_grad(o, r, grad);
        DBuildResult br = build(o, tree, k, plan, true);
        DFactor f = factorize(br.h, 1);
        const double ll = log_likelihood(f, r);
        std::vector<const DHodlr*> d;
        for (auto& x : br.deriv) d.push_back(&x);
        const Vec s = score(f, d, r, nullptr);
        grad.resize(s.size());
        for (size_t i = 0; i < s.size(); ++i) grad[i] = -s[i];
        return -ll;
    }
    Vec fisher_at(const Vec& th) const {
        o.set_parameters(th.data(), int(th.size()));
        if (dense) return dense_exact(o, r).fisher;
        DBuildResult br = build(o, tree, k, plan, true);
        DFactor f = factorize(br.h, 1);
        std::vector<const DHodlr*> d;
        for (auto& x : br.deriv) d.push_back(&x);
        std::vector<DProductRep> reps;
        score(f, d, r, &reps);
        return fisher_from_reps(reps);
    }
};

}  // namespace

ConfidenceIntervals confidence_intervals(const Vec& theta, const Vec& fisher) {
    const int p = int(theta.size());
    ConfidenceIntervals out;
    out.bounds.assign(static_cast<size_t>(2 * p), std::numeric_limits<double>::quiet_NaN());
    if (int(fisher.size()) != p * p) return out;
    Vec w;
    std::vector<double> V;
    sym_eig(fisher, p, w, V);
    for (double x : w)
        if (!(x > 0)) return out;
    const double z = 1.959964;  // 95% normal quantile (mle.cpp:335)
    for (int i = 0; i < p; ++i) {
        double inv_ii = 0.0;
        for (int m = 0; m < p; ++m) inv_ii += V[i + m * p] * V[i + m * p] / w[m];
        const double hw = z * std::sqrt(inv_ii);
        out.bounds[i] = theta[i] - hw;
        out.bounds[i + p] = theta[i] + hw;
    }
    out.valid = true;
    return out;
}

FitReport fit_mle(DOracle& o, DTreeP tree, i64 k, std::uint64_t seed, const double* r_dev,
                  const std::vector<int>& transforms, const Vec& theta0, int max_iter, double rel_tol,
                  bool dense) {
    const auto t0 = std::chrono::steady_clock::now();
    const int p = int(theta0.size());
    if (int(transforms.size()) != p) throw std::invalid_argument("fit_mle: transforms must match parameter count");
    if (p != o.num_params()) throw std::invalid_argument("fit_mle: theta0 must have one entry per oracle parameter");
    o.reset_counters();
    DSketchPlanP plan = get_plan(tree, k, seed);
    Evaluator ev{o, tree, k, *plan, r_dev, dense};
    FitReport rep;
    rep.status = "max_iter";
    Vec u = from_natural(theta0, transforms), theta = theta0, grad_theta(static_cast<size_t>(p));
    double fval;
    try {
        fval = ev.value_grad(theta, grad_theta);
    } catch (const NotPositiveDefinite&) {
        rep.status = "not_positive_definite_at_start";
        rep.theta_hat = theta0;
        return rep;
    }
    auto chain = [&](const Vec& g, const Vec& th) {
        Vec gu = g, jd = jacobian_diag(th, transforms);
        for (int i = 0; i < p; ++i) gu[i] *= jd[i];
        return gu;
    };
    Vec gu = chain(grad_theta, theta);
    std::vector<double> hinv(static_cast<size_t>(p) * p, 0.0);
    for (int i = 0; i < p; ++i) hinv[i + i * p] = 1.0;
    Vec fisher_cache;
    const double inf = std::numeric_limits<double>::infinity();
    for (int it = 0; it < max_iter; ++it) {
        rep.loglik_trace.push_back(-fval);
        rep.grad_norm_trace.push_back(norm(gu));
        rep.theta_trace.push_back(theta);
        rep.iterations = it;
        Vec dir(static_cast<size_t>(p), 0.0);
        for (int i = 0; i < p; ++i)
            for (int j = 0; j < p; ++j) dir[i] -= hinv[i + j * p] * gu[j];
        if (dot(dir, gu) >= 0)
            for (int i = 0; i < p; ++i) dir[i] = -gu[i];  // reset on loss of descent
        double step = 1.0, fnew = inf;
        Vec unew(static_cast<size_t>(p));
        bool accepted = false;
        for (int ls = 0; ls <= 20; ++ls) {
            for (int i = 0; i < p; ++i) unew[i] = u[i] + step * dir[i];
            double ftrial;
            try {
                ftrial = ev.value(to_natural(unew, transforms));
            } catch (const NotPositiveDefinite&) {
                ftrial = inf;
            }
            if (std::isfinite(ftrial) && ftrial <= fval + 1e-4 * step * dot(gu, dir)) {
                fnew = ftrial;
                accepted = true;
                break;
            }
            step *= 0.5;
        }
        if (!accepted) {
            // stationary if the score test statistic S^T I^-1 S is negligible
            bool stationary = norm(gu) < 1e-5 * std::max(1.0, std::abs(fval));
            if (!stationary) {
                try {
                    fisher_cache = ev.fisher_at(theta);
                    Vec g = grad_theta;
                    if (chol_solve(fisher_cache, p, g)) stationary = dot(grad_theta, g) <= 1e-3 * double(p);
                } catch (const NotPositiveDefinite&) {
                }
            }
            rep.status = stationary ? "converged" : "line_search_failed";
            rep.converged = stationary;
            break;
        }
        const Vec theta_new = to_natural(unew, transforms);
        Vec grad_new(static_cast<size_t>(p));
        try {
            fnew = ev.value_grad(theta_new, grad_new);
        } catch (const NotPositiveDefinite&) {
            rep.status = "not_positive_definite";
            break;
        }
        const Vec gu_new = chain(grad_new, theta_new);
        Vec s(static_cast<size_t>(p)), yv(static_cast<size_t>(p));
        for (int i = 0; i < p; ++i) {
            s[i] = unew[i] - u[i];
            yv[i] = gu_new[i] - gu[i];
        }
        const double sy = dot(s, yv);
        if (sy > 1e-12 * norm(s) * norm(yv)) {  // inverse BFGS update
            Vec hy(static_cast<size_t>(p), 0.0);
            for (int i = 0; i < p; ++i)
                for (int j = 0; j < p; ++j) hy[i] += hinv[i + j * p] * yv[j];
            const double yhy = dot(yv, hy), a = (sy + yhy) / (sy * sy);
            for (int i = 0; i < p; ++i)
                for (int j = 0; j < p; ++j)
                    hinv[i + j * p] += a * s[i] * s[j] - (hy[i] * s[j] + s[i] * hy[j]) / sy;
        }
        const bool small_f = std::abs(fnew - fval) <= rel_tol * std::max(1.0, std::abs(fval));
        const bool small_x = norm(s) <= rel_tol * std::max(1.0, norm(u));
        u = unew;
        theta = theta_new;
        fval = fnew;
        gu = gu_new;
        grad_theta = grad_new;
        if (small_f && small_x) {
            rep.converged = true;
            rep.status = "converged";
            rep.iterations = it + 1;
            rep.loglik_trace.push_back(-fval);
            rep.grad_norm_trace.push_back(norm(gu));
            rep.theta_trace.push_back(theta);
            break;
        }
    }
    rep.theta_hat = theta;
    try {
        rep.fisher = !fisher_cache.empty() ? fisher_cache : ev.fisher_at(theta);
        const ConfidenceIntervals ci = confidence_intervals(theta, rep.fisher);
        rep.ci = ci.bounds;
        rep.ci_valid = ci.valid;
    } catch (const NotPositiveDefinite&) {
        rep.fisher.clear();
        rep.ci_valid = false;
    }
    rep.apply_columns = o.apply_columns();
    rep.derivative_columns = o.derivative_columns();
    rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return rep;
}

}  // namespace hg
