// Exact representation of A*B / A^{-1}B as an asymmetric HODLR base plus one
// block-diagonal low-rank correction per level, and the exact traces built
// on it (score: tr(K^-1 K_j); Fisher: tr(K^-1 K_i K^-1 K_j)).
//
// Reference: product_rep.hpp:14-55, product_rep.cpp:9-245.
// Device layout: correction level i (2^(i-1) depth-(i-1) blocks of width
// C_i = 2 R_i) is an n x C_i column block of two n x sum(C) panels Cu / Cv;
// the base's right factors alias the operand's panels (the pipeline only
// rewrites left factors, product_rep.cpp:92-104).
#pragma once

#include "factor.cuh"

namespace hg {

struct DProductRep {
    DHodlr base;
    std::vector<int> C, coff;  // [i-1]
    int sumC = 0;
    DVecP Cu, Cv;  // n x max(sumC, 1)
    i64 n() const { return base.n(); }
    int tau() const { return base.tau(); }
    double* Cul(int i) const { return Cu->get() + i64(coff[static_cast<size_t>(i - 1)]) * n(); }
    double* Cvl(int i) const { return Cv->get() + i64(coff[static_cast<size_t>(i - 1)]) * n(); }
};

/// product_rep.cpp:47-155 (inverse = solve_multiply, else multiply).
DProductRep pipeline(const DFactor& f, const DHodlr& b, bool inverse);
/// The pipeline for several operands of one factorization in one pass: the
/// correction left factors Cu depend on the factorization only, so the reps
/// share one Cu panel (formed and updated once) and every factor level
/// streams its panels once for all operands.
std::vector<DProductRep> pipeline_multi(const DFactor& f, const std::vector<const DHodlr*>& bs, bool inverse);

/// out (+)= trace_product_rep (product_rep.cpp:188-194).
void trace_product_rep(const DProductRep& p, double* out, bool accumulate);
/// out (+)= trace_pair (product_rep.cpp:204-235). with_corr = false keeps
/// only the base-base trace (:206-210), for fisher_corrections.
void trace_pair(const DProductRep& p, const DProductRep& q, double* out, bool accumulate, bool with_corr = true);
/// The correction terms of trace_pair — cross terms (:212-224) and
/// correction pairs (:227-233) — for every i <= j of p solve_multiply reps of
/// ONE factorization (pipeline_multi). Their Cu panel is shared, so every
/// product that involves only a base and Cu (leaf products, V_l^T Cu, the
/// Grams Cu^T Cv_f and Cv^T Cu_f) is formed once and reused by every pair.
/// Returns, per (i, j) column-major, the terms to add to
/// trace_pair(reps[i], reps[j], .., with_corr = false).
std::vector<double> fisher_corrections(const std::vector<DProductRep>& reps);

/// Dense assembly on the host (test support; n <= 2^14).
std::vector<double> prodrep_densify(const DProductRep& p);

/// Y <- (I + u v^T) Y for level i of a Right factorization (multiply path).
void level_multiply(const DFactor& f, int i, double* Y, i64 ldy, int w);
/// rows += p (q^T rows) with q = u (the reference association, product_rep.cpp:32-45).
void level_update_pq(const DFactor& f, int i, const double* P, double* Y, int w);

}  // namespace hg
