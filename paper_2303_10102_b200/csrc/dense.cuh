// Exact dense evaluation on the device (the accuracy reference of the MLE
// path): dense_exact (mle.cpp:345-380), the dense objective of fit_mle's
// Evaluator (mle.cpp:128-175) and accuracy_metrics (mle.cpp:382-403).
#pragma once

#include <vector>

#include "oracle.cuh"

namespace hg {

/// mle.hpp:93-99. fisher p x p column-major.
struct DenseExact {
    double loglik = 0.0;
    std::vector<double> score, fisher;
};

/// mle.hpp:102-108.
struct AccuracyMetrics {
    double eps_L = 0.0, eps_S = 0.0, eps_I = 0.0, eta_g = 0.0, eta_I = 0.0;
};

/// K = oracle.apply(I), Cholesky, loglik, score -1/2 tr(K^-1 K_j) + 1/2 w^T K_j w,
/// Fisher 1/2 sum(M_i .* M_j^T) with M_j = K^-1 K_j. r = y - ybar on the
/// device. n <= 2^13 (the reference's guard, std::length_error).
DenseExact dense_exact(const DOracle& o, const double* r);

/// -loglik of the dense path (Evaluator::value, dense branch).
double dense_objective(const DOracle& o, const double* r);

/// -loglik and its natural-parameter gradient through one explicit inverse
/// (Evaluator::value_grad, dense branch).
double dense_objective_grad(const DOracle& o, const double* r, std::vector<double>& grad);

/// mle.cpp:382-403 (host arithmetic on p-vectors / p x p column-major).
AccuracyMetrics accuracy_metrics(double loglik, const std::vector<double>& score_exact,
                                 const std::vector<double>& fisher_exact, double loglik_approx,
                                 const std::vector<double>& score_approx, const std::vector<double>& fisher_approx);

}  // namespace hg
