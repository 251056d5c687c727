// Basic HODLR factorization A = Abar (I + U^(tau) V^(tau)T) ... (I + U^(1) V^(1)T)
// with Cholesky (LU fallback) leaves and LU-factored capacitances.
//
// Reference: factorization.hpp:25-82, factorization.cpp:7-224.
// Device layout: the Woodbury factors of level i are never formed densely.
// u = diag(wbar, xbar) is the n x R_i panel Wbar_i (wbar on left-child rows,
// xbar on right-child rows), v = antidiag(w, x) is the source matrix's own
// upper-factor panel F_i (w on left-child rows, x on right-child rows), so
//   cap_j = I + v^T u = [[I, x^T xbar], [w^T wbar, I]]   (2R_i x 2R_i).
#pragma once

#include "hodlr.cuh"

namespace hg {

struct DFactor {
    DTreeP tree;
    int orient = 0;  // 0 Right, 1 Left
    std::vector<int> R, off;  // per level capacity, column offset in Wbar
    int sumR = 0;
    std::vector<DVecP> F;     // [l-1] n x R_l source factors (aliases when symmetric)
    DVecP Wbar;               // n x sumR
    DVecP leaf_mat;           // original leaves (LeafFactor::multiply)
    DVecP leaf_fac;           // factored leaves (LLT lower or packed LU)
    std::shared_ptr<DBuf<int>> leaf_kind;  // 1 LLT, 0 LU
    std::shared_ptr<DBuf<int>> leaf_piv;   // LU row swaps per leaf (bmax each)
    DVecP leaf_ld;                         // log|det| per leaf
    std::shared_ptr<DBuf<int>> leaf_sign;  // +1 / -1 (sign of det)
    bool all_llt = false;                  // every leaf Cholesky-factored
    std::vector<DVecP> cap;                // [i-1] nodes x (2R)^2 LU
    std::vector<std::shared_ptr<DBuf<int>>> cap_piv;  // [i-1] nodes x 2R swaps
    std::vector<DVecP> cap_ld;             // [i-1] nodes
    std::vector<std::shared_ptr<DBuf<int>>> cap_sign;
    // Explicit capacitance inverses computed once by substitution, so every
    // later capacitance solve is batched tensor-core GEMMs: x0 = S b followed
    // by one step of refinement x = x0 + S (b - A x0) with the operator A.
    // [i-1] node panels (nodes*2R) x 2R, ld nodes*2R, Pi = half swap:
    std::vector<DVecP> capinv, capR;       // Right: cap^{-1} Pi and Pi cap
    std::vector<DVecP> capinvT, capT;      // Left : cap^{-T} and cap^T

    i64 n() const { return tree->n(); }
    int tau() const { return tree->tau(); }
    int bmax() const { return tree->bmax; }
    i64 lstride() const { return i64(bmax()) * bmax(); }
    double* Fl(int l) const { return F[static_cast<size_t>(l - 1)] ? F[static_cast<size_t>(l - 1)]->get() : nullptr; }
    double* Wl(int l) const { return Wbar->get() + i64(off[static_cast<size_t>(l - 1)]) * n(); }
    int Rl(int l) const { return R[static_cast<size_t>(l - 1)]; }
};

/// factorization.cpp:62-168
DFactor factorize(const DHodlr& h, int orient);

/// Y <- Abar^{-1} Y on all leaf row blocks (LeafFactor::solve, :20-22).
void leaf_solve(const DFactor& f, double* Y, i64 ldy, int w);

/// Woodbury step of level i on an n x w panel Y:
///   transposed = false: Y -= u cap^{-1} v^T Y   (Right solve, factorize)
///   transposed = true : Y -= v cap^{-T} u^T Y   (Left solve, pipeline)
void level_inverse(const DFactor& f, int i, bool transposed, double* Y, i64 ldy, int w);
/// p = -v cap^{-T} (n x 2R, ld n) of level i by LU substitution per row, the
/// reference's association (HG_ASSOC_REFERENCE; product_rep.cpp:74-78).
void form_p_reference(const DFactor& f, int i, double* P);

/// HodlrFactorization::solve (factorization.cpp:170-212), in place.
void factor_solve(const DFactor& f, double* Y, i64 ldy, int w);

/// HodlrFactorization::logdet (factorization.cpp:214-224); throws
/// NotPositiveDefinite like the reference.
double factor_logdet(const DFactor& f);

/// leaf-kind flags (1 = LLT) to host.
std::vector<int> leaf_kinds(const DFactor& f);

}  // namespace hg
