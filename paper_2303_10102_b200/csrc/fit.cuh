// fit_mle (mle.hpp:37-90) on the device path — see fit.cu.
#pragma once

#include <string>
#include <vector>

#include "oracle.cuh"

namespace hg {

enum FitTransform { FIT_POSITIVE = 0, FIT_CORRELATION = 1, FIT_UNBOUNDED = 2 };  // ParamTransform

struct ConfidenceIntervals {  // mle.hpp:84-87; bounds p x 2 column-major (lo, hi)
    std::vector<double> bounds;
    bool valid = false;
};

struct FitReport {  // mle.hpp:59-73
    std::vector<double> theta_hat;
    int iterations = 0;
    bool converged = false;
    std::string status;
    std::vector<double> loglik_trace, grad_norm_trace;
    std::vector<std::vector<double>> theta_trace;
    std::vector<double> fisher;  // p x p at theta_hat
    std::vector<double> ci;      // p x 2
    bool ci_valid = false;
    std::uint64_t apply_columns = 0, derivative_columns = 0;
    double seconds = 0;
};

/// mle.cpp:327-343 (level 0.95 only).
ConfidenceIntervals confidence_intervals(const std::vector<double>& theta, const std::vector<double>& fisher);

/// mle.cpp:188-322: BFGS on the transformed parameters, backtracking line
/// search (Armijo 1e-4, <= 20 halvings, non-SPD iterates rejected), score-test
/// stationarity on a failed search, Fisher and 95% intervals at the optimum.
/// r_dev = y - ybar on the device. dense: FitOptions::dense, the exact dense
/// evaluation path (dense.cu) instead of the HODLR build.
FitReport fit_mle(DOracle& o, DTreeP tree, i64 k, std::uint64_t seed, const double* r_dev,
                  const std::vector<int>& transforms, const std::vector<double>& theta0, int max_iter,
                  double rel_tol, bool dense = false);

}  // namespace hg
