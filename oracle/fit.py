"""CPU restatement of fit_mle (mle.cpp:188-322) — TEST INFRASTRUCTURE ONLY.

BFGS on transformed parameters (positive: theta = exp(u); correlation:
theta = tanh(u); unbounded) with a backtracking Armijo line search (1e-4,
<= 20 halvings, non-SPD iterates rejected), the inverse-BFGS update under the
curvature test s.y > 1e-12 |s||y|, the relative f / x stopping rule, the
score-test stationarity check on a failed line search, and 95% confidence
intervals from the Fisher matrix at the optimum (mle.cpp:327-343). The
objective, gradient and Fisher come from `evaluate` — here the CPU oracle
pipeline (build, factorize, log-likelihood, score, Fisher)."""
import numpy as np

from . import pyoracle as O

POSITIVE, CORRELATION, UNBOUNDED = 0, 1, 2


def _to_nat(u, tr):
    return np.array([np.exp(a) if t == POSITIVE else (np.tanh(a) if t == CORRELATION else a) for a, t in zip(u, tr)])


def _from_nat(th, tr):
    return np.array([np.log(a) if t == POSITIVE else (np.arctanh(a) if t == CORRELATION else a) for a, t in zip(th, tr)])


def _jac(th, tr):
    return np.array([a if t == POSITIVE else (1 - a * a if t == CORRELATION else 1.0) for a, t in zip(th, tr)])


def confidence_intervals(theta, fisher):
    w, V = np.linalg.eigh(fisher)
    if w.min() <= 0:
        return np.full((len(theta), 2), np.nan), False
    inv = (V / w) @ V.T
    hw = 1.959964 * np.sqrt(np.diag(inv))
    return np.stack([theta - hw, theta + hw], axis=1), True


def fit_mle(value, value_grad, fisher_at, theta0, tr, max_iter=100, rel_tol=1e-6):
    p = len(theta0)
    rep = {"status": "max_iter", "converged": False, "loglik_trace": [], "grad_norm_trace": [], "theta_trace": []}
    u, theta = _from_nat(theta0, tr), np.array(theta0, dtype=float)
    try:
        fval, g = value_grad(theta)
    except O.NotPositiveDefinite:
        rep.update(status="not_positive_definite_at_start", theta_hat=theta)
        return rep
    gu = g * _jac(theta, tr)
    hinv = np.eye(p)
    fisher_cache = None
    for it in range(max_iter):
        rep["loglik_trace"].append(-fval)
        rep["grad_norm_trace"].append(np.linalg.norm(gu))
        rep["theta_trace"].append(theta.copy())
        rep["iterations"] = it
        d = -(hinv @ gu)
        if d @ gu >= 0:
            d = -gu
        step, accepted = 1.0, False
        for _ in range(21):
            unew = u + step * d
            try:
                ft = value(_to_nat(unew, tr))
            except O.NotPositiveDefinite:
                ft = np.inf
            if np.isfinite(ft) and ft <= fval + 1e-4 * step * (gu @ d):
                accepted = True
                break
            step *= 0.5
        if not accepted:
            stationary = np.linalg.norm(gu) < 1e-5 * max(1.0, abs(fval))
            if not stationary:
                try:
                    fisher_cache = fisher_at(theta)
                    L = np.linalg.cholesky(fisher_cache)
                    z = np.linalg.solve(L, g)
                    stationary = z @ z <= 1e-3 * p
                except (O.NotPositiveDefinite, np.linalg.LinAlgError):
                    pass
            rep["status"] = "converged" if stationary else "line_search_failed"
            rep["converged"] = bool(stationary)
            break
        th_new = _to_nat(unew, tr)
        try:
            fnew, gnew = value_grad(th_new)
        except O.NotPositiveDefinite:
            rep["status"] = "not_positive_definite"
            break
        gu_new = gnew * _jac(th_new, tr)
        s, yv = unew - u, gu_new - gu
        sy = s @ yv
        if sy > 1e-12 * np.linalg.norm(s) * np.linalg.norm(yv):
            hy = hinv @ yv
            hinv = hinv + ((sy + yv @ hy) / sy**2) * np.outer(s, s) - (np.outer(hy, s) + np.outer(s, hy)) / sy
        small_f = abs(fnew - fval) <= rel_tol * max(1.0, abs(fval))
        small_x = np.linalg.norm(s) <= rel_tol * max(1.0, np.linalg.norm(u))
        u, theta, fval, gu, g = unew, th_new, fnew, gu_new, gnew
        if small_f and small_x:
            rep.update(converged=True, status="converged", iterations=it + 1)
            rep["loglik_trace"].append(-fval)
            rep["grad_norm_trace"].append(np.linalg.norm(gu))
            rep["theta_trace"].append(theta.copy())
            break
    rep["theta_hat"] = theta
    try:
        rep["fisher"] = fisher_cache if fisher_cache is not None else fisher_at(theta)
        rep["ci"], rep["ci_valid"] = confidence_intervals(theta, rep["fisher"])
    except O.NotPositiveDefinite:
        rep["fisher"], rep["ci_valid"] = None, False
    return rep


def matern_evaluators(x, nu2, nugget, tau, k, seed, y):
    """value / value_grad / fisher_at of the CPU oracle pipeline for a 1D
    Matern oracle with theta = (sigma2, ell) (device product association)."""

    def pipeline(theta, deriv):
        oo = O.CovOracle.matern(x, nu2, theta[0], theta[1], nugget, True)
        b = O.Build(oo, tau, k, seed, deriv, p=2 if deriv else 0)
        f = O.factorize(b.h(), 1)
        return b, f

    def value(theta):
        _, f = pipeline(theta, False)
        return -O.log_likelihood(f, y)

    def value_grad(theta):
        b, f = pipeline(theta, True)
        d = [b.deriv(0), b.deriv(1)]
        try:
            O.set_solve_association(True)
            s = O.score(f, d, y)
        finally:
            O.set_solve_association(False)
        return -O.log_likelihood(f, y), -np.asarray(s)

    def fisher_at(theta):
        b, f = pipeline(theta, True)
        d = [b.deriv(0), b.deriv(1)]
        try:
            O.set_solve_association(True)
            return np.asarray(O.fisher_information(f, d, cache=True))
        finally:
            O.set_solve_association(False)

    return value, value_grad, fisher_at
