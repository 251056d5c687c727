// TEST INFRASTRUCTURE ONLY — CPU forward model for BASELINE.json configs C1
// and C4 (1D Matérn on sorted points), shared by the restated oracle
// (oracle/hodlr.cpp) and the reference build's C API (oracle/ref_capi.cpp) so
// both consume identical K·V bytes. Not a reference component: the
// reference's models are FEM/SPDE; the product
// implements the same formulas on the GPU (csrc/oracle.cu,
// csrc/matern_chunk.cuh).
//   k(d) = sigma2 * p_nu(a) * exp(-a), a = c_nu d / ell,
//   p_{1/2} = 1, p_{3/2} = 1 + a, p_{5/2} = 1 + a + a^2/3, plus nugget * I;
//   dk/dsigma2 = k_noiseless / sigma2, dk/dell = sigma2 q_nu(a) exp(-a) / ell
//   with q_{1/2} = a, q_{3/2} = a^2, q_{5/2} = a^2 (1 + a) / 3.
#pragma once

#include <cmath>
#include <cstdint>
#include <vector>

namespace matern1d {

using Index = std::int64_t;

inline double c_nu(int nu2) { return nu2 == 1 ? 1.0 : (nu2 == 3 ? std::sqrt(3.0) : std::sqrt(5.0)); }

/// exp(-lambda d) * sum_m coef[m] d^m representation of each kernel
/// (which = -1 value, 0 d/dsigma2, 1 d/dell); returns the number of terms.
inline int poly(int nu2, int which, double sigma2, double ell, double coef[4], double& lambda) {
    lambda = c_nu(nu2) / ell;
    const double L = lambda;
    for (int m = 0; m < 4; ++m) coef[m] = 0;
    const double s = which == 0 ? 1.0 : sigma2;  // d/dsigma2 drops the sigma2 factor
    if (which <= 0) {
        coef[0] = s;
        if (nu2 >= 3) coef[1] = s * L;
        if (nu2 == 5) coef[2] = s * L * L / 3.0;
        return nu2 == 1 ? 1 : (nu2 == 3 ? 2 : 3);
    }
    if (nu2 == 1) {
        coef[1] = s * L / ell;
        return 2;
    }
    if (nu2 == 3) {
        coef[2] = s * L * L / ell;
        return 3;
    }
    coef[2] = s * L * L / (3.0 * ell);
    coef[3] = s * L * L * L / (3.0 * ell);
    return 4;
}

inline double kernel(int nu2, int which, double sigma2, double ell, double d) {
    double coef[4], lambda;
    const int nt = poly(nu2, which, sigma2, ell, coef, lambda);
    double p = 0, dm = 1;
    for (int m = 0; m < nt; ++m) {
        p += coef[m] * dm;
        dm *= d;
    }
    return p * std::exp(-lambda * d);
}

/// Y = K V (which = -1, nugget included) or dK/dtheta_which V; dense O(n^2)
/// per column or the O(n) two-sided exponential-polynomial recurrence
///   F_m(i) = rho sum_{q<=m} C(m,q) d^{m-q} F_q(i-1) + [m=0] v_i.
inline void apply(const double* x, Index n, int nu2, double sigma2, double ell, double nugget, int which,
                  bool scan, const double* v, Index ldv, Index s, double* y, Index ldy) {
    double coef[4], lambda;
    const int nt = poly(nu2, which, sigma2, ell, coef, lambda);
    if (!scan) {
#pragma omp parallel for schedule(static)
        for (Index i = 0; i < n; ++i) {
            std::vector<double> kr(static_cast<size_t>(n));
            for (Index j = 0; j < n; ++j) kr[static_cast<size_t>(j)] = kernel(nu2, which, sigma2, ell, std::abs(x[i] - x[j]));
            for (Index c = 0; c < s; ++c) {
                double acc = 0;
                for (Index j = 0; j < n; ++j) acc += kr[static_cast<size_t>(j)] * v[j + c * ldv];
                y[i + c * ldy] = acc;
            }
        }
    } else {
        static const double binom[4][4] = {{1, 0, 0, 0}, {1, 1, 0, 0}, {1, 2, 1, 0}, {1, 3, 3, 1}};
#pragma omp parallel for schedule(static)
        for (Index c = 0; c < s; ++c) {
            const double* vc = v + c * ldv;
            double* yc = y + c * ldy;
            double st[4] = {0, 0, 0, 0};
            for (Index i = 0; i < n; ++i) {
                if (i > 0) {
                    const double d = x[i] - x[i - 1];
                    const double rho = std::exp(-lambda * d);
                    double ns[4];
                    for (int m = nt - 1; m >= 0; --m) {
                        double acc = 0, dp = 1;
                        for (int q = m; q >= 0; --q) {
                            acc += binom[m][q] * dp * st[q];
                            dp *= d;
                        }
                        ns[m] = rho * acc;
                    }
                    for (int m = 0; m < nt; ++m) st[m] = ns[m];
                }
                st[0] += vc[i];
                double acc = 0;
                for (int m = 0; m < nt; ++m) acc += coef[m] * st[m];
                yc[i] = acc;
            }
            for (int m = 0; m < 4; ++m) st[m] = 0;
            for (Index i = n - 1; i >= 0; --i) {
                if (i < n - 1) {
                    const double d = x[i + 1] - x[i];
                    const double rho = std::exp(-lambda * d);
                    double ns[4];
                    for (int m = nt - 1; m >= 0; --m) {
                        double acc = 0, dp = 1;
                        for (int q = m; q >= 0; --q) {
                            acc += binom[m][q] * dp * st[q];
                            dp *= d;
                        }
                        ns[m] = rho * acc;
                    }
                    for (int m = 0; m < nt; ++m) st[m] = ns[m];
                }
                st[0] += vc[i];
                double acc = 0;
                for (int m = 0; m < nt; ++m) acc += coef[m] * st[m];
                yc[i] += acc - coef[0] * vc[i];
            }
        }
    }
    if (which < 0 && nugget != 0.0)
        for (Index c = 0; c < s; ++c)
            for (Index i = 0; i < n; ++i) y[i + c * ldy] += nugget * v[i + c * ldv];
}

}  // namespace matern1d
