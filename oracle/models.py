"""CPU restatement of the forward-model covariances of BASELINE.json configs
2, 3 and 5 — TEST INFRASTRUCTURE ONLY.

The reference's own forward models are FEM wind/ADR problems (out of scope);
the configs' models are new, so this file states them directly, with the same
formulas as the device oracles (paper_2303_10102_b200/csrc/models.cu):

C2 co-kriging: f ~ GP Matern nu = 1/2 (sigma2, ell) on x_i = i h, i = 1..m,
h = 1/(m+1); A = tridiag(-1, 2, -1)/h^2 + kappa^2 I (Dirichlet FD);
K = [[A^-1 Kf A^-1, A^-1 Kf], [Kf A^-1, Kf]] in the per-point interleaved
order (rows 2i = u_i, 2i+1 = f_i) plus a fixed nugget on the diagonal,
theta = (sigma2, ell, kappa).

C3/C5 SPDE: u = (-Lap_h + kappa^2)^-1 f (plus a fixed nugget, default 10
Var(u): the field alone is singular in FP64 and its weak HODLR at the configs'
ranks is positive definite only above that) on the N x N periodic grid of the
unit square (5-point stencil, h = 1/N; point g = iy*N + ix), f stationary
with the 2D Matern 3/2 spectral density at the centred integer frequencies,
normalised to Var f = sigma2:
    s(k) = (3/ell^2 + 4 pi^2 |k|^2)^(-5/2),   lam_f = sigma2 N^2 s / sum s,
    mu(k) = (4/h^2)(sin^2(pi kx/N) + sin^2(pi ky/N)) + kappa^2,
    K = F^-1 diag(lam_f / mu^2) F  (F the unnormalised 2D DFT),
dK/dsigma2 = K/sigma2, dK/dell from d(lam_f)/dell, dK/dkappa from
-4 kappa lam_f / mu^3. Exact spectral log-determinant and Fisher matrix are
available (spde2d_exact) as analytic cross-checks of the HODLR pipeline.
"""
import numpy as np


# --------------------------------------------------------------------- C2
def cokriging_dense(m, sigma2, ell, kappa, nugget=1e-6):
    """(K, [dK/dsigma2, dK/dell, dK/dkappa]) of size 2m, interleaved order; K
    carries `nugget` on its diagonal (needed in FP64, see models.cu)."""
    h = 1.0 / (m + 1)
    x = np.arange(1, m + 1) * h
    A = (np.diag(np.full(m, 2.0)) - np.diag(np.ones(m - 1), 1) - np.diag(np.ones(m - 1), -1)) / h**2
    A += kappa**2 * np.eye(m)
    Ai = np.linalg.inv(A)
    d = np.abs(x[:, None] - x[None, :])
    Kf = sigma2 * np.exp(-d / ell)
    dKf_s = Kf / sigma2
    dKf_l = sigma2 * (d / ell**2) * np.exp(-d / ell)
    dAi = -2.0 * kappa * Ai @ Ai

    def joint(uu, uf, ff):
        K = np.zeros((2 * m, 2 * m))
        K[0::2, 0::2] = uu
        K[0::2, 1::2] = uf
        K[1::2, 0::2] = uf.T
        K[1::2, 1::2] = ff
        return K

    K = joint(Ai @ Kf @ Ai, Ai @ Kf, Kf) + nugget * np.eye(2 * m)
    dS = joint(Ai @ dKf_s @ Ai, Ai @ dKf_s, dKf_s)
    dL = joint(Ai @ dKf_l @ Ai, Ai @ dKf_l, dKf_l)
    dK = joint(dAi @ Kf @ Ai + Ai @ Kf @ dAi, dAi @ Kf, np.zeros((m, m)))
    return K, [dS, dL, dK]


# -------------------------------------------------------------------- SPDE
def spde2d_variance(N, sigma2, ell, kappa):
    """Var(u) = mean of lam_f / mu^2 (the nugget defaults to a fraction of it)."""
    return float(spde2d_spectra(N, sigma2, ell, kappa, 0.0)[0].mean())


def spde2d_spectra(N, sigma2, ell, kappa, nugget=None):
    """Full N x N multipliers (K, dK/dsigma2, dK/dell, dK/dkappa) of the DFT
    diagonalisation, without the 1/N^2 of the inverse transform. K carries the
    fixed nugget (default 10 Var(u), as the device wrapper)."""
    k = np.arange(N)
    kc = np.where(k <= N // 2, k, k - N).astype(float)
    KY, KX = np.meshgrid(kc, kc, indexing="ij")
    b = 4.0 * np.pi**2 * (KX**2 + KY**2)
    a = 3.0 / ell**2
    s = (a + b) ** -2.5
    ds = 15.0 / ell**3 * (a + b) ** -3.5
    S, Sd = s.sum(), ds.sum()
    iy, ix = np.meshgrid(k, k, indexing="ij")
    mu = 4.0 * N**2 * (np.sin(np.pi * ix / N) ** 2 + np.sin(np.pi * iy / N) ** 2) + kappa**2
    lf = sigma2 * N * N * s / S
    dlf = sigma2 * N * N * (ds * S - s * Sd) / S**2
    if nugget is None:
        nugget = 10.0 * float((lf / mu**2).mean())
    return [lf / mu**2 + nugget, lf / sigma2 / mu**2, dlf / mu**2, -4.0 * kappa * lf / mu**3]


def spde2d_apply(N, sigma2, ell, kappa, V, order=None, j=-1, nugget=None):
    """K V (j = -1) or dK/dtheta_j V through numpy's FFT; rows of V in `order`."""
    lam = spde2d_spectra(N, sigma2, ell, kappa, nugget)[j + 1]
    V = np.asarray(V, dtype=float)
    vec = V.ndim == 1
    V = V.reshape(N * N, -1)
    order = np.arange(N * N) if order is None else np.asarray(order)
    G = np.zeros_like(V)
    G[order] = V
    out = np.empty_like(G)
    for c in range(G.shape[1]):
        g = G[:, c].reshape(N, N)
        out[:, c] = np.real(np.fft.ifft2(lam * np.fft.fft2(g))).ravel()
    Y = out[order]
    return Y[:, 0] if vec else Y


def spde2d_dense(N, sigma2, ell, kappa, order=None, nugget=None):
    """(K, [dK_j]) densely, rows/columns in `order` (N <= 32)."""
    n = N * N
    mats = [spde2d_apply(N, sigma2, ell, kappa, np.eye(n), order, j, nugget) for j in (-1, 0, 1, 2)]
    mats = [0.5 * (M + M.T) for M in mats]
    return mats[0], mats[1:]


def spde2d_exact(N, sigma2, ell, kappa, y=None, order=None, nugget=None):
    """Exact log-determinant, Fisher matrix (1/2 sum d_i log lam d_j log lam) and,
    with y, the log-likelihood and score of the SPDE covariance."""
    lam = spde2d_spectra(N, sigma2, ell, kappa, nugget)
    L = lam[0]
    dlog = [d / L for d in lam[1:]]
    n = N * N
    logdet = float(np.log(L).sum())
    fisher = np.array([[0.5 * float((a * b).sum()) for b in dlog] for a in dlog])
    out = {"logdet": logdet, "fisher": fisher}
    if y is not None:
        order = np.arange(n) if order is None else np.asarray(order)
        g = np.zeros(n)
        g[order] = y
        yh = np.fft.fft2(g.reshape(N, N))
        quad = float(np.real(np.sum(np.abs(yh) ** 2 / L)) / n)
        out["loglik"] = -0.5 * n * np.log(2 * np.pi) - 0.5 * logdet - 0.5 * quad
        score = []
        for d in dlog:  # -1/2 tr(K^-1 dK) + 1/2 y^T K^-1 dK K^-1 y
            score.append(-0.5 * float(d.sum()) + 0.5 * float(np.real(np.sum(np.abs(yh) ** 2 * d / L)) / n))
        out["score"] = np.array(score)
    return out
