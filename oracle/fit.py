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


LOG2PI = 1.8378770664093454836


def dense_exact(K, dKs, r):
    """mle.cpp:345-380 in numpy: exact log-likelihood, score and Fisher of the
    dense covariance K with derivatives dKs at residual r = y - ybar."""
    n = K.shape[0]
    L = np.linalg.cholesky(K)
    w = np.linalg.solve(L.T, np.linalg.solve(L, r))
    ld = 2.0 * np.sum(np.log(np.diag(L)))
    ll = -0.5 * n * LOG2PI - 0.5 * ld - 0.5 * r @ w
    M = [np.linalg.solve(L.T, np.linalg.solve(L, kj)) for kj in dKs]
    s = np.array([-0.5 * np.trace(m) + 0.5 * w @ (kj @ w) for m, kj in zip(M, dKs)])
    p = len(dKs)
    f = np.array([[0.5 * np.sum(M[i] * M[j].T) for j in range(p)] for i in range(p)])
    return ll, s, f


def accuracy_metrics(ll, se, fe, lla, sa, fa):
    """mle.cpp:382-403 in numpy."""
    se, sa, fe, fa = map(np.asarray, (se, sa, fe, fa))
    ds, di = se - sa, fe - fa
    L = np.linalg.cholesky(fe)  # raises LinAlgError when not SPD (the reference: invalid_argument)
    inv_e = np.linalg.inv(fe)
    inv_a = np.linalg.inv(fa)
    return {"eps_L": abs(ll - lla) / abs(ll), "eps_S": np.linalg.norm(ds) / np.linalg.norm(se),
            "eps_I": np.linalg.norm(di) / np.linalg.norm(fe),
            "eta_g": float(np.sqrt(ds @ np.linalg.solve(L.T, np.linalg.solve(L, ds)))),
            "eta_I": float(np.sqrt(max(0.0, np.trace(di @ (inv_e - inv_a)))))}


def dense_evaluators(kfun, r):
    """value / value_grad / fisher_at of fit_mle's dense path (mle.cpp:128-175)
    for kfun(theta) -> (K, [dK_j])."""

    def value(theta):
        K, _ = kfun(theta)
        try:
            L = np.linalg.cholesky(K)
        except np.linalg.LinAlgError as e:
            raise O.NotPositiveDefinite(1, "dense covariance") from e
        w = np.linalg.solve(L.T, np.linalg.solve(L, r))
        return -(-0.5 * len(r) * LOG2PI - np.sum(np.log(np.diag(L))) - 0.5 * r @ w)

    def value_grad(theta):
        K, dKs = kfun(theta)
        try:
            L = np.linalg.cholesky(K)
        except np.linalg.LinAlgError as e:
            raise O.NotPositiveDefinite(1, "dense covariance") from e
        w = np.linalg.solve(L.T, np.linalg.solve(L, r))
        kinv = np.linalg.solve(L.T, np.linalg.solve(L, np.eye(len(r))))
        g = np.array([-(-0.5 * np.sum(kinv * kj) + 0.5 * w @ (kj @ w)) for kj in dKs])
        return -(-0.5 * len(r) * LOG2PI - np.sum(np.log(np.diag(L))) - 0.5 * r @ w), g

    def fisher_at(theta):
        K, dKs = kfun(theta)
        return dense_exact(K, dKs, r)[2]

    return value, value_grad, fisher_at
