// Batched FP64 primitives over flattened per-level row panels.
//
// Every HODLR operation of the hot path reduces to a handful of segmented
// kernels over the row ranges of one tree depth ("segments"):
//   seg_tn    T_s = alpha * A[s]^T B[s] + beta T_s      (projections, Gram blocks)
//   seg_nn    Y[s] = alpha * X[s] T_{map(s)} + beta Y[s]  (low-rank updates)
//   leaf_mm   Y[leaf] = alpha * op(L_b) X[leaf] + beta Y[leaf]
//   reductions (deterministic, fixed order) for traces.
// Panels are column-major n x w arrays; segment s of depth d covers rows
// [bounds[s], bounds[s+1]).
#pragma once

#include "tree.cuh"

namespace hg {

/// Selects the small right factor of segment s in seg_nn:
/// index = ((s >> shift) ^ xr) * mult + add; first row = (s & 1) ? row_odd : row_even.
struct TMap {
    int shift = 0, xr = 0, row_even = 0, row_odd = 0, mult = 1, add = 0;
    static TMap same() { return TMap{}; }
    static TMap sibling() { return TMap{0, 1, 0, 0, 1, 0}; }
    static TMap parent(int re, int ro) { return TMap{1, 0, re, ro, 1, 0}; }
    /// child (2s + c) of segment s of a coarser partition
    static TMap child(int c) { return TMap{0, 0, 0, 0, 2, c}; }
};

/// T_s (ca x cb, col-major, ld ldt, stride tstride per segment) =
/// alpha A[s]^T B[s] + beta T_s. Deterministic split-K over row chunks.
void seg_tn(const Partition& p, const double* A, i64 lda, int ca, const double* B, i64 ldb, int cb,
            double* T, i64 tstride, int ldt, double alpha = 1.0, double beta = 0.0);

/// Y[s] (rows x w) = alpha X[s] (rows x k) * T_sel (k x w) + beta Y[s].
void seg_nn(const Partition& p, const double* X, i64 ldx, int k, const double* T, i64 tstride, int ldt,
            TMap map, double* Y, i64 ldy, int w, double alpha = 1.0, double beta = 0.0);

/// Leaves: Y[leaf b] = alpha op(L_b) X[leaf b] + beta Y[leaf b]; L_b at
/// L + b*lstride with ld ldl (m_b x m_b).
void leaf_mm(const Partition& leaves, const double* L, i64 lstride, int ldl, bool trans, const double* X,
             i64 ldx, double* Y, i64 ldy, int w, double alpha = 1.0, double beta = 0.0);

/// Copy / scale / add panels: Y = alpha X + beta Y over n x w.
void panel_axpby(i64 n, int w, double alpha, const double* X, i64 ldx, double beta, double* Y, i64 ldy);

/// Y rows of even segments = a_even Xe, of odd segments = a_odd Xo (a null
/// source writes zeros); each row reads only the source it keeps.
void panel_parity_select(const Partition& p, int w, const double* Xe, i64 ldxe, double a_even, const double* Xo,
                         i64 ldxo, double a_odd, double* Y, i64 ldy);

/// out[0] (+)= sum_s sum_{e<len} A[s gsa + e] B[(s^xr) gsb + e] (deterministic
/// streaming reduction; the HBM-bound core of every trace).
void seg_dot(int nseg, int xr, const double* A, i64 gsa, const double* B, i64 gsb, i64 len, double* out,
             bool accumulate);

/// out[0] (+)= alpha sum((L_b X) .* Z) over the leaves (no n x w product stored).
void leaf_mm_dot(const Partition& leaves, const double* L, i64 lstride, int ldl, const double* X, i64 ldx,
                 const double* Z, i64 ldz, int w, double alpha, double* out, bool accumulate);
/// outs[z] (+)= alphas[z] sum((L_b X) .* Zs[z]) for several Z with ONE leaf
/// product (the cross terms of every Fisher pair with the same base).
constexpr int LEAF_DOT_MAXZ = 4;
/// outs[z * nl + a] (+)= tr(As[z]^T L_a B) over the leaves, L_a = Ls[a] (leaf
/// arrays, stride lstride, ld ldl), As[z], B n x K (ld ld): per-leaf Grams
/// As[z][b] B[b]^T formed once and dotted with every L_a.
void leaf_gram_dot(const Partition& leaves, const std::vector<const double*>& As, const double* B, i64 ld, int K,
                   const std::vector<const double*>& Ls, i64 lstride, int ldl, const std::vector<double*>& outs,
                   bool accumulate);
void leaf_mm_dot_multi(const Partition& leaves, const double* L, i64 lstride, int ldl, const double* X, i64 ldx,
                       const std::vector<const double*>& Zs, i64 ldz, int w, const std::vector<double>& alphas,
                       const std::vector<double*>& outs, bool accumulate);

/// out[0] (+)= sum(A .* B) over n x w (deterministic).
void dot_panels(i64 n, int w, const double* A, i64 lda, const double* B, i64 ldb, double* out, bool accumulate);

/// out[0] (+)= sum_s sum_{a<ra,b<rb} G_s(a,b) H_{s^xr}(b,a) with G_s ra x rb (ld
/// ldg, stride gs), H_s rb x ra (ld ldh, stride hs).
void seg_pair_dot(int nseg, int xr, const double* G, i64 gs, int ldg, int ra, int rb, const double* H, i64 hs,
                  int ldh, double* out, bool accumulate);

/// out[0] (+)= sum_s sum_{a<ra,c<rc} G_s(a,c) H_{s^xr}(a,c), both ra x rc
/// (ld ld, stride gs).
void seg_xor_dot(int nseg, int xr, const double* G, const double* H, i64 gs, int ld, int ra, int rc, double* out,
                 bool accumulate);

/// out[0] (+)= sum_b trace(L_b) (leaves, ld ldl, stride lstride).
void leaf_trace(const Partition& leaves, const double* L, i64 lstride, int ldl, double* out, bool accumulate);
/// out[0] (+)= sum_b sum(A_b^T .* B_b).
void leaf_pair_dot(const Partition& leaves, const double* A, const double* B, i64 lstride, int ldl, double* out,
                   bool accumulate);

/// Optional input-support hint for hodlr_apply / DOracle::apply_masked: X is zero on every row of
/// the depth-`depth` segments whose index parity equals `parity` (the sketch
/// samplers of the build are zero on one child of every level-l node); the
/// projections skip chunks that lie entirely in such a segment.
/// With out_depth >= 0 the caller also declares that it reads Y only on
/// those same rows (the depth-out_depth segments of that parity): the peel
/// samples blocks of the still-unknown level from rows where its sampler is
/// zero, so the level updates skip every other row tile.
struct ZeroRows {
    const int* bounds = nullptr;  // partition bounds of that depth (device)
    int nseg = 0, parity = 0;
    int out_depth = -1;
    /// hodlr_apply only: X is the leaf sampler, the stacked identities
    /// X[lo_b + c, c] = 1 (sketch.cpp:25-30), so a level's projection is the
    /// sum of its panel's leaf blocks over each segment (no GEMM).
    bool leaf_identity = false;
};

/// Final host read of a device scalar (synchronizes the stream).
double read_scalar(const double* d);

}  // namespace hg
