// Statistics glue of one MLE iteration (mle.cpp:25-54) on the device.
#include <algorithm>
#include <cmath>
#include <random>

#include "api.cuh"

namespace hg {

namespace {
constexpr double kLog2Pi = 1.8378770664093454836;
}

double log_likelihood(const DFactor& f, const double* r) {
    const i64 n = f.n();
    DVec w(static_cast<size_t>(n)), d(1);
    panel_axpby(n, 1, 1.0, r, n, 0.0, w.get(), n);
    factor_solve(f, w.get(), n, 1);
    dot_panels(n, 1, r, n, w.get(), n, d.get(), false);
    const double ld = factor_logdet(f);
    return -0.5 * double(n) * kLog2Pi - 0.5 * ld - 0.5 * read_scalar(d.get());
}

std::vector<double> score(const DFactor& f, const std::vector<const DHodlr*>& deriv, const double* r,
                          std::vector<DProductRep>* reps) {
    const i64 n = f.n();
    const size_t p = deriv.size();
    DVec w(static_cast<size_t>(n)), kw(static_cast<size_t>(n)), acc(2 * std::max<size_t>(p, 1));
    panel_axpby(n, 1, 1.0, r, n, 0.0, w.get(), n);
    factor_solve(f, w.get(), n, 1);
    std::vector<DProductRep> local;
    std::vector<DProductRep>& rp = reps ? *reps : local;
    rp = pipeline_multi(f, deriv, true);
    for (size_t j = 0; j < p; ++j) {
        trace_product_rep(rp[j], acc.get() + 2 * j, false);
        hodlr_apply(*deriv[j], w.get(), n, 1, kw.get(), n, 1, deriv[j]->tau(), true, false, 0.0);
        dot_panels(n, 1, w.get(), n, kw.get(), n, acc.get() + 2 * j + 1, false);
    }
    std::vector<double> h = acc.download();
    std::vector<double> s(p);
    for (size_t j = 0; j < p; ++j) s[j] = -0.5 * h[2 * j] + 0.5 * h[2 * j + 1];
    return s;
}

std::pair<double, double> hutchinson_trace(const DFactor& f, const DHodlr& b, int n_samples, std::uint64_t seed) {
    if (n_samples < 2) throw std::invalid_argument("hutchinson_trace: need >= 2 samples");
    if (b.n() != f.n()) throw std::invalid_argument("hutchinson_trace: dimension mismatch");
    const i64 n = f.n();
    constexpr int CH = 64;
    std::mt19937_64 rng(seed);
    std::bernoulli_distribution coin(0.5);
    DVec Z(static_cast<size_t>(n) * CH), X(static_cast<size_t>(n) * CH), d(CH);
    std::vector<double> hz(static_cast<size_t>(n) * CH);
    double sum = 0, sumsq = 0;
    for (int s0 = 0; s0 < n_samples; s0 += CH) {
        const int sc = std::min(CH, n_samples - s0);
        for (int s = 0; s < sc; ++s)
            for (i64 i = 0; i < n; ++i) hz[static_cast<size_t>(i + i64(s) * n)] = coin(rng) ? 1.0 : -1.0;
        Z.upload(hz.data(), static_cast<size_t>(n) * CH);
        hodlr_apply(b, Z.get(), n, sc, X.get(), n, 1, b.tau(), true, false, 0.0);
        factor_solve(f, X.get(), n, sc);
        for (int s = 0; s < sc; ++s) dot_panels(n, 1, Z.get() + i64(s) * n, n, X.get() + i64(s) * n, n, d.get() + s, false);
        const std::vector<double> v = d.download();  // synchronises: hz may be refilled
        for (int s = 0; s < sc; ++s) {
            sum += v[static_cast<size_t>(s)];
            sumsq += v[static_cast<size_t>(s)] * v[static_cast<size_t>(s)];
        }
    }
    const double var = (sumsq - sum * sum / n_samples) / (n_samples - 1);
    return {sum / n_samples, std::sqrt(std::max(var, 0.0) / n_samples)};
}

std::vector<double> fisher_from_reps(const std::vector<DProductRep>& reps) {
    const size_t p = reps.size();
    DVec acc(std::max<size_t>(p * p, 1));
    acc.zero();
    for (size_t i = 0; i < p; ++i)
        for (size_t j = i; j < p; ++j) trace_pair(reps[i], reps[j], acc.get() + i + j * p, false, false);
    const std::vector<double> pairs = fisher_corrections(reps);  // products shared across the pairs
    std::vector<double> t = acc.download();
    for (size_t e = 0; e < t.size(); ++e) t[e] += pairs[e];
    std::vector<double> info(p * p), out(p * p);
    for (size_t i = 0; i < p; ++i)
        for (size_t j = i; j < p; ++j) {
            const double v = 0.5 * t[i + j * p];
            info[i + j * p] = v;
            info[j + i * p] = v;
        }
    for (size_t i = 0; i < p; ++i)
        for (size_t j = 0; j < p; ++j) out[i + j * p] = 0.5 * (info[i + j * p] + info[j + i * p]);
    return out;
}

}  // namespace hg
