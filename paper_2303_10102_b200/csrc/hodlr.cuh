// Device-resident HODLR matrix in flattened per-level panel form.
//
// Reference container: hodlr_matrix.hpp:48-106 (vectors of per-block Eigen
// factors). Here level l (1..tau) is two n x R_l column-major panels:
//   U_l: rows of each node's left child hold upper.left, rows of its right
//        child hold lower.left;
//   V_l: rows of the right child hold upper.right, rows of the left child hold
//        lower.right.
// so block (cl,cr) = U_l[cl] V_l[cr]^T and block (cr,cl) = U_l[cr] V_l[cl]^T.
// Symmetric storage has V_l == U_l (one buffer). R_l is the largest block
// rank of the level; columns past a block's own rank are zero. Leaves are
// nleaves x (bmax x bmax) column-major blocks, zero padded.
#pragma once

#include "kernels.cuh"

namespace hg {

struct DHodlr {
    DTreeP tree;
    bool sym = true;
    std::vector<int> R;                        // [l-1]
    std::vector<DVecP> U, V;                   // [l-1], n x R
    std::vector<std::vector<int>> rank_up, rank_lo;  // [l-1][node]
    DVecP leaves;                              // nleaves * bmax^2
    bool leaves_zero = false;

    i64 n() const { return tree->n(); }
    int tau() const { return tree->tau(); }
    int bmax() const { return tree->bmax; }
    i64 lstride() const { return i64(bmax()) * bmax(); }
    double* Ul(int l) const { return U[static_cast<size_t>(l - 1)] ? U[static_cast<size_t>(l - 1)]->get() : nullptr; }
    double* Vl(int l) const { return V[static_cast<size_t>(l - 1)] ? V[static_cast<size_t>(l - 1)]->get() : nullptr; }
    int Rl(int l) const { return R[static_cast<size_t>(l - 1)]; }

    /// hodlr_matrix.cpp:68-81 (empty off-diagonal blocks, zero leaves).
    static DHodlr zero(DTreeP t, bool symmetric = true);
    /// hodlr_matrix.cpp:126-172 (host mt19937_64 draws, same fill order).
    static DHodlr random(DTreeP t, i64 k, std::uint64_t seed, bool spd);
    /// hodlr_matrix.cpp:83-88
    static DHodlr identity(DTreeP t);

    /// Panel exchange format (host): per level U_l then V_l (n x R_l each),
    /// then leaves concatenated m_b x m_b col-major. ranks: 2^tau - 1 per array.
    static DHodlr import_panels(DTreeP t, bool symmetric, const int* R, const double* flat, const int* ranks_up,
                                const int* ranks_lo);
    size_t export_size() const;
    void export_panels(double* flat, int* ranks_up, int* ranks_lo) const;

    /// hodlr_matrix.cpp:187-196: lower blocks become explicit (shares storage
    /// until a factor is rewritten; every writer allocates fresh panels).
    void make_asymmetric();
    /// Resize level l to capacity r (zero panels).
    void set_level(int l, int r, bool symmetric_panel);
};

/// Y = beta Y + alpha H_sel X over an n x s block, where H_sel keeps levels
/// [lmin, lmax] (and the leaves when with_leaves). lmin = d+1 gives the
/// block-diagonal of all depth-d sub-blocks at once (sub_matvec,
/// hodlr_matrix.cpp:228-265); lmin = 1 is the full matvec (:198-222).

void hodlr_apply(const DHodlr& h, const double* X, i64 ldx, int s, double* Y, i64 ldy, int lmin, int lmax,
                 bool with_leaves, bool transpose, double beta = 0.0, double alpha = 1.0, ZeroRows zero = {});

/// Streaming path of hodlr_apply for s <= 4 (hmatvec.cu): returns false when
/// the call is outside its domain (transpose, zero hints, ranks > 256).
bool hodlr_apply_narrow(const DHodlr& h, const double* X, i64 ldx, int s, double* Y, i64 ldy, int lmin, int lmax,
                        bool with_leaves, bool transpose, double beta, double alpha, ZeroRows zero);

/// Projections of all levels at once: T_l[s] = P_l[s]^T X[s] (P = U when
/// transpose, else V) for the first ncol[l-1] columns of X, as nseg_l
/// blocks of R_l x s (ld R_l). Entries of missing levels are null.
std::vector<DVecP> hodlr_project(const DHodlr& h, const double* X, i64 ldx, int s, bool transpose,
                                 const std::vector<int>& ncol);

/// Leaves <-> n x bmax panel (leaf b occupies its rows, columns [0, m_b)).
void leaves_panel(const DTree& t, double* leaves, double* P, bool to_panel);

/// out (+)= trace(H) (hodlr_matrix.cpp:267-271).
void hodlr_trace(const DHodlr& h, double* out, bool accumulate);
/// out (+)= tr(A B) from matched block pairs (hodlr_matrix.cpp:294-318).
void hodlr_trace_product(const DHodlr& a, const DHodlr& b, double* out, bool accumulate);

}  // namespace hg
