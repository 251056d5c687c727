// Strong-admissibility H-matrix (eta-admissible far field, geometric KD
// block-cluster tree) for the 2D periodic-grid covariances of BASELINE.json
// configs 3 and 5.
//
// The reference is weak-HODLR only (sibling blocks only,
// SPEC.md:90-96); this format has no reference counterpart and no parity
// oracle: it is validated against the dense covariance (n <= 2^12) and against
// the exact FFT apply of the forward model at full size.
//
// Block-cluster tree: the reference's uniform cluster tree over the KD order of
// the grid (every node is a rectangle of grid points); a pair (t, s) of one
// depth is admissible when min(diam t, diam s) <= eta dist(t, s), with the
// distance measured on the torus (the grid is periodic). Admissible pairs are
// rank-k blocks U V^T, inadmissible leaf pairs dense; only t <= s is stored
// (the matrix is symmetric).
//
// Construction is matrix-free: the oracle declares the covariance translation
// invariant on the grid, so one apply of K (or dK/dtheta_j) to a unit vector
// gives its generating column c, every entry is K(i, j) = c(g_i - g_j mod N),
// and the admissible blocks are compressed by a batched randomized range
// finder whose products A Omega and A^T Q are formed with the entries
// generated inside the GEMM tiles (nothing n x n is ever stored).
#pragma once

#include "oracle.cuh"
#include "qr.cuh"

namespace hg {

struct HsPlan {
    struct Lr {
        int d, t, s;  // node indices at depth d, t < s
    };
    struct Dn {
        int t, s;  // leaf indices, t <= s
    };
    i64 n = 0;
    int tau = 0, nside = 0, k = 0;
    double eta = 1.0;
    ClusterTree tree;
    std::vector<Lr> lr;
    std::vector<Dn> dn;
};

/// Host block-cluster tree of the nside x nside periodic grid in the row order
/// `order` (order[i] = grid index iy*nside + ix of row i; must be a KD order so
/// that tree nodes are rectangles). Admissible pairs whose smaller side has at
/// most k rows are kept dense (a rank-k factorization would not be smaller).
HsPlan hs_plan(const std::int64_t* order, int nside, int tau, double eta, int k);

/// Entry generator of a grid-stationary covariance (device pointers).
struct GridEntries {
    const double* c;  // generating column, grid order (N*N)
    const int* gx;    // per row: grid x index
    const int* gy;    // per row: grid y index
    int N;
};

class DHStrong {
public:
    DHStrong() = default;
    DHStrong(const DHStrong&) = delete;  // the work lists hold pointers into U/V/D
    DHStrong& operator=(const DHStrong&) = delete;
    DHStrong(DHStrong&&) = default;
    DHStrong& operator=(DHStrong&&) = default;
    HsPlan plan;
    // factor storage: block b's U (t_m x k) at U + uoff[b], V (s_m x k) at V + voff[b]
    DVec U, V, D;
    std::vector<i64> uoff, voff, doff;
    // apply work lists (built once)
    struct ProjItem {
        const double* M;
        i64 ldm;
        const double* X;  // null: the call's X
        i64 xoff, ldx;
        int rows, part;
    };
    struct Contrib {
        const double* M;
        i64 ldm, moff, ridx;
        int trans, K, rkind, pad;
    };
    struct Tile {
        int row0, rin, rows, cfirst, clast, pad;  // rin: row offset inside its leaf
    };
    DBuf<ProjItem> proj;       // call-X projections: part = slot chunk
    std::vector<int> slot_first;  // per slot (2 b + side) its first partial; size 2 nlr + 1
    DBuf<int> dslot_first;
    int nparts = 0;
    DBuf<Contrib> contrib;
    DBuf<Tile> tiles;
    int ntiles = 0;
    int max_contrib = 0;  // most contributions of one leaf
    i64 n() const { return plan.n; }
    int k() const { return plan.k; }
    size_t bytes() const { return (U.size() + V.size() + D.size()) * sizeof(double); }
};

/// Build K (param = -1) or dK/dtheta_param in the strong format. power_iters
/// subspace iterations per block (0 = plain range finder of width k).
DHStrong hs_build(const DOracle& o, int param, const std::int64_t* order, int nside, int tau, double eta, int k,
                  int power_iters, std::uint64_t seed);

/// Y = H X (n x s, column-major).
void hs_apply(const DHStrong& h, const double* X, i64 ldx, int s, double* Y, i64 ldy);

/// out[0] = tr(A B) = <A, B>_F (both symmetric, same plan), deterministic.
void hs_trace_product(const DHStrong& a, const DHStrong& b, double* out);

}  // namespace hg
