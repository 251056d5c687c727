// Aggregate header of the device hot path (used by the C ABI).
#pragma once

#include "build.cuh"
#include "prodrep.cuh"

namespace hg {

DHodlr hodlr_deep_copy(const DHodlr& h);

/// mle.cpp:25-30 — r is the residual y - ybar (device, length n).
double log_likelihood(const DFactor& f, const double* r);

/// mle.cpp:32-41 with the p ProductReps K^-1 K_j kept in `reps` for reuse by
/// the Fisher matrix (the same arithmetic the reference repeats per pair).
std::vector<double> score(const DFactor& f, const std::vector<const DHodlr*>& deriv, const double* r,
                          std::vector<DProductRep>* reps);

/// mle.cpp:56-75 — Rademacher-probe estimate of tr(K^-1 B): the probes are
/// generated on the host in the reference's order (mt19937_64 +
/// bernoulli_distribution(0.5)) and applied in blocks of 64 columns; returns
/// {estimate, std_error} accumulated probe by probe as the reference does.
std::pair<double, double> hutchinson_trace(const DFactor& f, const DHodlr& b, int n_samples, std::uint64_t seed);

/// mle.cpp:43-54 (p x p, column-major) from the cached ProductReps.
std::vector<double> fisher_from_reps(const std::vector<DProductRep>& reps);

}  // namespace hg
