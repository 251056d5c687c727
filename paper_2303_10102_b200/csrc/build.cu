// Sketch construction of H and dH/dtheta_j on the device (sketch.cpp:128-356).
//
// Level l is processed for all of its 2^(l-1) nodes at once: oracle applies
// and peeling matvecs act on full n x k panels, the per-node range finders
// are one batched (TSQR + column-pivoted Householder) QR, and the per-node
// small algebra (sign fix, numeric rank, completion, diff_qr, q2 width,
// recompression) runs one CTA per node.
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <cmath>
#include <mutex>
#include <random>

#include "build.cuh"

namespace hg {

namespace {

constexpr int MAX_RANK = 128;  // sketch width k: per-node k x k work arrays live in shared memory

__global__ void k_leaf_identity(const int* bounds, double* P, i64 ldp) {
    const int b = blockIdx.x;
    const int lo = bounds[b], m = bounds[b + 1] - lo;
    for (int i = threadIdx.x; i < m; i += blockDim.x) P[i64(lo + i) + i64(i) * ldp] = 1.0;
}

/// Node arrays from the batched QR (or the full-width shortcut, sketch.cpp:159-170):
/// R (k x k, sign-fixed, rows >= numeric rank zeroed), perm, sign, numeric rank.
__global__ void k_range_post(int k, const int* qmap, const double* qR, const int* qperm, double* R, int* perm,
                             double* sign, int* nr) {
    const int j = blockIdx.x;
    const int q = qmap[j];
    double* Rj = R + i64(j) * k * k;
    if (q < 0) {  // full width: q = I, r = 0
        for (int e = threadIdx.x; e < k * k; e += blockDim.x) Rj[e] = 0.0;
        for (int i = threadIdx.x; i < k; i += blockDim.x) {
            perm[j * k + i] = i;
            sign[j * k + i] = 1.0;
        }
        if (threadIdx.x == 0) nr[j] = k;
        return;
    }
    const double* Q = qR + i64(q) * k * k;
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int r = e % k;
        const double s = Q[r + r * k] < 0 ? -1.0 : 1.0;
        Rj[e] = s * Q[e];
    }
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
        perm[j * k + i] = qperm[q * k + i];
        sign[j * k + i] = Q[i + i * k] < 0 ? -1.0 : 1.0;
    }
    __syncthreads();
    __shared__ int s_nr;
    if (threadIdx.x == 0) {
        const double d0 = fabs(Rj[0]);
        int r = 0;
        while (r < k && fabs(Rj[r + r * k]) > 64 * DBL_EPSILON * d0) ++r;
        s_nr = r;
        nr[j] = r;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k * k; e += blockDim.x)
        if (e % k >= s_nr) Rj[e] = 0.0;
}

__device__ double cta_sum(double v) {
    __shared__ double sh[32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) t += sh[i];
    return t;
}

/// sketch.cpp:60-74: complete deficient columns with canonical basis vectors
/// orthogonalised twice against the kept ones (skipping norms below 0.5).
__global__ void k_complete(const int* bounds, int k, const int* nr, double* S, i64 lds, double* scratch,
                           int max_rows) {
    const int j = blockIdx.x;
    int filled = nr[j];
    if (filled >= k) return;
    const int lo = bounds[2 * j], m = bounds[2 * j + 1] - lo;
    if (m > max_rows) return;  // long blocks take the batched path (complete_batched)
    double* Q = S + lo;
    double* v = scratch + lo;
    __shared__ double g[512];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int e = 0; e < m && filled < k; ++e) {
        // pass 1: v = e_e - Q_f Q_f[e,:]^T
        for (int c = tid; c < filled; c += blockDim.x) g[c] = Q[e + i64(c) * lds];
        __syncthreads();
        for (int i = tid; i < m; i += blockDim.x) {
            double s = (i == e) ? 1.0 : 0.0;
            for (int c = 0; c < filled; ++c) s -= Q[i + i64(c) * lds] * g[c];
            v[i] = s;
        }
        __syncthreads();
        // pass 2: g = Q_f^T v ; v -= Q_f g
        for (int c = warp; c < filled; c += nw) {
            double s = 0.0;
            for (int i = lane; i < m; i += 32) s += Q[i + i64(c) * lds] * v[i];
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) g[c] = s;
        }
        __syncthreads();
        double part = 0.0;
        for (int i = tid; i < m; i += blockDim.x) {
            double s = v[i];
            for (int c = 0; c < filled; ++c) s -= Q[i + i64(c) * lds] * g[c];
            v[i] = s;
            part += s * s;
        }
        const double nv = sqrt(cta_sum(part));
        if (nv < 0.5) {
            __syncthreads();
            continue;
        }
        for (int i = tid; i < m; i += blockDim.x) Q[i + i64(filled) * lds] = v[i] / nv;
        ++filled;
        __syncthreads();
    }
}

/// Row-parallel S[cl] = Q diag(sign) (identity for full-width nodes).
__global__ void k_q_sign_rows(const WorkItem* items, const int* bounds, int k, const int* qmap, const double* sign,
                              double* S, i64 lds) {
    const WorkItem it = items[blockIdx.x];
    if (it.seg & 1) return;  // right children hold no basis
    const int j = it.seg >> 1;
    const bool full = qmap[j] < 0;
    const int clo = bounds[2 * j];
    for (int e = threadIdx.x; e < it.rows * k; e += blockDim.x) {
        const int r = e % it.rows, c = e / it.rows;
        double* p = S + i64(it.row0 + r) + i64(c) * lds;
        if (full)
            *p = (it.row0 + r - clo) == c ? 1.0 : 0.0;
        else
            *p *= sign[j * k + c];
    }
}

/// presc partial sums: per work item and param, sum of squares of dY rows.
__global__ void k_presc_part(const WorkItem* items, int k, int p, const double* dY, i64 ld, double* part) {
    const WorkItem it = items[blockIdx.x];
    for (int q = 0; q < p; ++q) {
        double s = 0.0;
        if (!(it.seg & 1))
            for (int e = threadIdx.x; e < it.rows * k; e += blockDim.x) {
                const int r = e % it.rows, c = e / it.rows;
                const double v = dY[i64(it.row0 + r) + i64(q * k + c) * ld];
                s += v * v;
            }
        s = cta_sum(s);
        if (threadIdx.x == 0) part[i64(blockIdx.x) * p + q] = s;
        __syncthreads();
    }
}

__global__ void k_presc_final(int nodes, const int* seg_first, int p, const double* part, double* presc) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nodes) return;
    double best = 0.0;
    for (int q = 0; q < p; ++q) {
        double s = 0.0;
        for (int it = seg_first[2 * j]; it < seg_first[2 * j + 1]; ++it) s += part[i64(it) * p + q];
        best = fmax(best, sqrt(s));
    }
    presc[j] = best;
}

/// Completion of long deficient blocks, batched (equivalent to the
/// sequential loop of sketch.cpp:60-74 when every candidate is accepted):
/// G_j = S[cl.lo + t, :]^T for t < c_j (the rows of the canonical candidates).
__global__ void k_cand_rows(const int* bounds, int k, int cmax, const int* cj, const double* S, i64 lds, double* G) {
    const int j = blockIdx.x;
    const int lo = bounds[2 * j];
    double* Gj = G + i64(j) * k * cmax;
    for (int e = threadIdx.x; e < k * cmax; e += blockDim.x) {
        const int a = e % k, t = e / k;
        Gj[e] = t < cj[j] ? S[i64(lo + t) + i64(a) * lds] : 0.0;
    }
}

/// W[cl.lo + t, t] += 1 (t < c_j): W = E - S G.
__global__ void k_add_canonical(const int* bounds, const int* cj, double* W, i64 ldw) {
    const int j = blockIdx.x;
    const int lo = bounds[2 * j];
    for (int t = threadIdx.x; t < cj[j]; t += blockDim.x) W[i64(lo + t) + i64(t) * ldw] += 1.0;
}

/// S[cl, nr_j + t] = sign(R_tt) Qw[cl, t] for t < c_j.
__global__ void k_place_completion(const WorkItem* items, const int* cj, const int* nr, const double* Rw, int cmax,
                                   const int* rmap, const double* Qw, i64 ldq, double* S, i64 lds) {
    const WorkItem it = items[blockIdx.x];
    if (it.seg & 1) return;
    const int j = it.seg >> 1;
    const int c = cj[j];
    if (c <= 0 || rmap[j] < 0) return;
    const double* R = Rw + i64(rmap[j]) * cmax * cmax;
    for (int e = threadIdx.x; e < it.rows * c; e += blockDim.x) {
        const int r = e % it.rows, t = e / it.rows;
        const double sg = R[t + t * cmax] < 0 ? -1.0 : 1.0;
        S[i64(it.row0 + r) + i64(nr[j] + t) * lds] = sg * Qw[i64(it.row0 + r) + i64(t) * ldq];
    }
}

/// Completion basis of one long deficient node by CholeskyQR: the projected
/// canonical candidates W (left-child rows, c_j columns) have Gram matrix
/// G = W^T W = I - S_c S_c^T-like and every accepted column has norm >= 0.5
/// after projection, so cond(W) <= 2 and W R^-1 (R = chol(G)^T, positive
/// diagonal) is orthonormal to O(eps cond^2). R_tt is exactly the
/// sequential loop's projected norm (sketch.cpp:60-74), so R_tt < 0.5 sends
/// the node back to that loop. One warp per node: writes R^-1 (upper,
/// cmax x cmax per even segment, zero-padded), diag(R) for the placement
/// and a fail flag.
__global__ void k_completion_cholqr(const int* cj, int cmax, const double* Gw, double* Rinv, double* Rdiag, int* fail) {
    const int j = blockIdx.x, lane = threadIdx.x;
    const int c = cj[j];
    const double* G = Gw + i64(2 * j) * cmax * cmax;
    double* Ri = Rinv + i64(2 * j) * cmax * cmax;
    double* Rd = Rdiag + i64(j) * cmax * cmax;
    extern __shared__ double L[];  // cmax x cmax, row stride ls (odd)
    const int ls = cmax | 1;
    for (int e = lane; e < cmax * cmax; e += 32) {
        Ri[e] = 0.0;
        Rinv[i64(2 * j + 1) * cmax * cmax + e] = 0.0;
        Rd[e] = 0.0;
    }
    if (c <= 0) {
        if (lane == 0) fail[j] = 0;
        return;
    }
    for (int e = lane; e < c * c; e += 32) L[(e % c) * ls + e / c] = G[(e % c) + i64(e / c) * cmax];
    __syncwarp();
    int bad = 0;
    for (int t = 0; t < c; ++t) {  // right-looking Cholesky, lower L (row r, col t at L[r * ls + t])
        const double d = L[t * ls + t];
        const double ltt = d > 0.0 ? sqrt(d) : 0.0;
        bad |= !(ltt >= 0.5);
        __syncwarp();
        for (int r = t + 1 + lane; r < c; r += 32) L[r * ls + t] = ltt > 0.0 ? L[r * ls + t] / ltt : 0.0;
        __syncwarp();
        if (lane == 0) L[t * ls + t] = ltt;
        for (int r = t + 1 + lane; r < c; r += 32)
            for (int q = t + 1; q <= r; ++q) L[r * ls + q] -= L[r * ls + t] * L[q * ls + t];
        __syncwarp();
    }
    if (lane == 0) fail[j] = bad;
    if (bad) return;
    // R = L^T (upper); R^-1 column by column (lane = column), back substitution
    for (int col = lane; col < c; col += 32) {
        for (int i = col; i >= 0; --i) {
            double s = (i == col) ? 1.0 : 0.0;
            for (int q = i + 1; q <= col; ++q) s -= L[q * ls + i] * Ri[q + i64(col) * cmax];
            Ri[i + i64(col) * cmax] = s / L[i * ls + i];
        }
        Rd[col + i64(col) * cmax] = L[col * ls + col];
    }
}

/// q2 width (sketch.cpp:214-221).
__global__ void k_w2_nodes(int nodes, const int* bounds, int k, int kp, const int* qmap, const double* R2,
                           const double* presc, int* w2out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nodes) return;
    const int q = qmap[j];
    if (q < 0) {
        w2out[j] = 0;
        return;
    }
    const int m = bounds[2 * j + 1] - bounds[2 * j];
    const double* R = R2 + i64(q) * kp * kp;
    const double d0 = fabs(R[0]);
    const double fl = fmax(1e-10 * d0, 1e-12 * presc[j]);
    const int cap = min(kp, m - k);
    int w2 = 0;
    while (w2 < cap && fabs(R[w2 + w2 * kp]) > fl) ++w2;
    w2out[j] = w2;
}

/// Column c < w_j of node j's left-child rows scaled to unit norm (after the
/// re-orthogonalisation of q2 against q, HG_Q2_REORTHOGONALIZED).
__global__ void k_col_normalize(const int* bounds, const int* wj, double* P, i64 ldp) {
    const int j = blockIdx.x, c = blockIdx.y;
    if (c >= wj[j]) return;
    const int lo = bounds[2 * j], m = bounds[2 * j + 1] - lo;
    double* col = P + i64(lo) + i64(c) * ldp;
    double s = 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) s += col[r] * col[r];
    s = cta_sum(s);
    const double inv = s > 0.0 ? 1.0 / sqrt(s) : 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) col[r] *= inv;
}

/// Zero columns [w_j, wtot) of the rows of one child (odd = right) of node j.
__global__ void k_mask_cols(const int* bounds, int odd, const int* wj, int wtot, double* P, i64 ldp) {
    const int j = blockIdx.x;
    const int c = 2 * j + odd;
    const int lo = bounds[c], m = bounds[c + 1] - lo;
    const int w0 = wj[j];
    for (int col = w0; col < wtot; ++col)
        for (int r = threadIdx.x; r < m; r += blockDim.x) P[i64(lo + r) + i64(col) * ldp] = 0.0;
}

/// diff_qr restricted to the in-span rotation (sketch.cpp:78-111,245-268):
/// y = (Q_rw^T dY[:, perm[:rw]]) R_rw^{-1}; Omega = skew(strict lower of y).
/// G holds Q^T dY (k x k) per child; one thread per row of y.
__global__ void k_diffqr(int k, const double* G, const double* R, const int* perm, const int* nr, const int* qmap,
                         double* Om, int* rw_out, int* ill) {
    const int j = blockIdx.x;
    const double* Gj = G + i64(2 * j) * k * k;  // left child block
    const double* Rj = R + i64(j) * k * k;
    double* O = Om + i64(j) * k * k;
    __shared__ int s_rw;
    extern __shared__ double y[];  // k x k, row stride ys (odd); blockDim >= k
    const int ys = k | 1;
    if (threadIdx.x == 0) {
        int rw = 0;
        const int r = nr[j];
        if (qmap[j] >= 0 && r > 0) {
            const double r00 = fabs(Rj[0]);
            while (rw < r && fabs(Rj[rw + rw * k]) > 1e-6 * r00) ++rw;
        }
        s_rw = rw;
        rw_out[j] = rw;
        double dmax = 0.0, dmin = INFINITY;
        for (int i = 0; i < rw; ++i) {
            dmax = fmax(dmax, fabs(Rj[i + i * k]));
            dmin = fmin(dmin, fabs(Rj[i + i * k]));
        }
        ill[j] = (rw > 0 && (!(dmin > 0) || dmax / dmin > 1e12)) ? 1 : 0;
    }
    __syncthreads();
    const int rw = s_rw;
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) O[e] = 0.0;
    const int a = threadIdx.x;
    if (a < rw) {
        for (int c = 0; c < rw; ++c) {  // y(a,:) R_rw = y0(a,:), column by column
            double s = Gj[a + perm[j * k + c] * k];
            for (int i = 0; i < c; ++i) s -= y[a * ys + i] * Rj[i + c * k];
            y[a * ys + c] = s / Rj[c + c * k];
        }
    }
    __syncthreads();
    if (a < rw)
        for (int c = 0; c < a; ++c) {
            O[a + c * k] = y[a * ys + c];
            O[c + a * k] = -y[a * ys + c];
        }
}

// ------------------------------------------------------------ recompression
/// M_j = T_L T_R^T (W x W, zero outside wl x wr) from the per-child R factors.
/// Truncation rank at rtol relative to the leading pivoted diagonal.
__global__ void k_trunc_rank(int nodes, int W, const double* RM, const int* wmin, double rtol, int* r_out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= nodes) return;
    const double* R = RM + i64(j) * W * W;
    const double d0 = fabs(R[0]);
    int r = 0;
    while (r < wmin[j] && fabs(R[r + r * W]) > rtol * d0) ++r;
    r_out[j] = r;
}

/// TinL = Q_M[:, :r] (columns >= r zeroed, in place); TinR[perm[i], a] = R_M[a, i], a < r.
__global__ void k_tins(int W, int rmax, const int* r, const double* RM, const int* permM, double* Tin) {
    const int j = blockIdx.x;
    const int rj = r[j];
    double* TL = Tin + i64(2 * j) * W * rmax;
    double* TR = Tin + i64(2 * j + 1) * W * rmax;
    const double* R = RM + i64(j) * W * W;
    for (int e = threadIdx.x; e < W * rmax; e += blockDim.x) {
        if (e / W >= rj) TL[e] = 0.0;
        TR[e] = 0.0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < W * rmax; e += blockDim.x) {
        const int i = e % W, a = e / W;
        if (a < rj) TR[permM[j * W + i] + i64(a) * W] = R[a + i64(i) * W];
    }
}

/// Direct truncation (Z P = Q_Z R_Z pivoted, stopped at rank r):
/// TinL[perm[i], a] = R_Z[a, i] (a < r), TinR = [I_r; 0] (w x rmax each).
__global__ void k_tins_direct(int W, int rmax, const int* r, const double* RZ, const int* permZ, double* Tin) {
    const int j = blockIdx.x;
    const int rj = r[j];
    double* TL = Tin + i64(2 * j) * W * rmax;
    double* TR = Tin + i64(2 * j + 1) * W * rmax;
    const double* R = RZ + i64(j) * W * W;
    for (int e = threadIdx.x; e < W * rmax; e += blockDim.x) {
        TL[e] = 0.0;
        TR[e] = (e % W == e / W && e / W < rj) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < W * rmax; e += blockDim.x) {
        const int i = e % W, a = e / W;
        if (a < rj) TL[permZ[j * W + i] + i64(a) * W] = R[a + i64(i) * W];
    }
}

std::vector<int> dl_int(const DBuf<int>& d) { return d.download(); }

__global__ void k_transpose_blocks(int w, const double* A, double* B) {
    const int j = blockIdx.x;
    const double* a = A + i64(j) * w * w;
    double* b = B + i64(j) * w * w;
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
        const int r = e % w, c = e / w;
        b[c + r * w] = a[e];
    }
}

/// Batched one-sided (Hestenes) Jacobi SVD of the w x w cores M_j, one CTA
/// per node: columns of A = M_j are rotated pairwise (round-robin tournament,
/// one warp per pair) until every pair is orthogonal to eps, V accumulates the
/// rotations, so A = U Sigma and M_j = (U Sigma) V^T. Columns are then sorted
/// by norm (the singular values, non-increasing) and the truncation rank is
/// the reference's rule: r = #{sigma_i > rtol sigma_0}, i < wmin
/// (hodlr_matrix.cpp:56-60). Outputs, per node: US (w x w, sorted A columns)
/// and V (w x w, sorted), both in the workspace, and r. This is the
/// HG_COMPRESS_JACOBI_SVD mode of the recompression (parity with JacobiSVD).
__global__ void __launch_bounds__(256) k_jacobi_svd(int w, const double* M, const int* wmin, double rtol,
                                                    double* A_ws, double* V_ws, double* US, double* Vs,
                                                    int* r_out) {
    const int j = blockIdx.x;
    const i64 ww = i64(w) * w;
    double* A = A_ws + j * ww;
    double* V = V_ws + j * ww;
    for (i64 e = threadIdx.x; e < ww; e += blockDim.x) {
        A[e] = M[j * ww + e];
        V[e] = (e % w) == (e / w) ? 1.0 : 0.0;
    }
    __shared__ int s_rot;
    __shared__ double s_norm[320];
    __shared__ int s_perm[320];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int wp = (w + 1) & ~1;  // players (one dummy when w is odd)
    const double eps = 2.220446049250313e-16;
    for (int sweep = 0; sweep < 60; ++sweep) {
        if (threadIdx.x == 0) s_rot = 0;
        __syncthreads();
        for (int step = 0; step < wp - 1; ++step) {
            for (int t = warp; t < wp / 2; t += nwarps) {
                auto pos = [&](int k) { return k == 0 ? 0 : 1 + (k - 1 + step) % (wp - 1); };
                int p = pos(t), q = pos(wp - 1 - t);
                if (p >= w || q >= w) continue;
                if (p > q) { const int x = p; p = q; q = x; }
                double* ap = A + i64(p) * w;
                double* aq = A + i64(q) * w;
                double al = 0, be = 0, ga = 0;
                for (int i = lane; i < w; i += 32) {
                    const double x = ap[i], y = aq[i];
                    al += x * x;
                    be += y * y;
                    ga += x * y;
                }
                for (int o = 16; o; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                if (ga == 0.0 || fabs(ga) <= eps * sqrt(al * be)) continue;
                const double zeta = (be - al) / (2.0 * ga);
                const double tt = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / sqrt(1.0 + tt * tt), sn = c * tt;
                for (int i = lane; i < w; i += 32) {
                    const double x = ap[i], y = aq[i];
                    ap[i] = c * x - sn * y;
                    aq[i] = sn * x + c * y;
                }
                double* vp = V + i64(p) * w;
                double* vq = V + i64(q) * w;
                for (int i = lane; i < w; i += 32) {
                    const double x = vp[i], y = vq[i];
                    vp[i] = c * x - sn * y;
                    vq[i] = sn * x + c * y;
                }
                if (lane == 0) s_rot = 1;
            }
            __syncthreads();
        }
        if (!s_rot) break;
        __syncthreads();
    }
    // singular values = column norms; stable sort non-increasing
    for (int c = warp; c < w; c += nwarps) {
        double s2 = 0;
        for (int i = lane; i < w; i += 32) s2 += A[i64(c) * w + i] * A[i64(c) * w + i];
        for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        if (lane == 0) s_norm[c] = sqrt(s2);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int c = 0; c < w; ++c) s_perm[c] = c;
        for (int a = 1; a < w; ++a) {  // insertion sort, stable
            const int x = s_perm[a];
            int b = a - 1;
            while (b >= 0 && s_norm[s_perm[b]] < s_norm[x]) {
                s_perm[b + 1] = s_perm[b];
                --b;
            }
            s_perm[b + 1] = x;
        }
        const double s0 = s_norm[s_perm[0]];
        int r = 0;
        while (r < wmin[j] && s_norm[s_perm[r]] > rtol * s0) ++r;
        r_out[j] = r;
    }
    __syncthreads();
    for (i64 e = threadIdx.x; e < ww; e += blockDim.x) {
        const int i = int(e % w), c = int(e / w);
        US[j * ww + e] = A[i64(s_perm[c]) * w + i];
        Vs[j * ww + e] = V[i64(s_perm[c]) * w + i];
    }
}

/// Tin[2j] = US[:, :r_j], Tin[2j+1] = V[:, :r_j] (w x rmax, zero past r_j).
__global__ void k_svd_tins(int w, int rmax, const int* r, const double* US, const double* Vs, double* Tin) {
    const int j = blockIdx.x;
    const int rj = r[j];
    const i64 ww = i64(w) * w;
    double* TL = Tin + i64(2 * j) * w * rmax;
    double* TR = Tin + i64(2 * j + 1) * w * rmax;
    for (int e = threadIdx.x; e < w * rmax; e += blockDim.x) {
        const bool keep = e / w < rj;
        TL[e] = keep ? US[j * ww + e] : 0.0;
        TR[e] = keep ? Vs[j * ww + e] : 0.0;
    }
}

/// Structured recompression of a derivative level built by the sketch
/// (sketch.cpp:297-311 then :331-341). Its left factor is
/// [dqc | Q | q2] = [Q | q2] [[Omega, I, 0], [0, 0, I]] with [Q | q2]
/// orthonormal (dqc = Q Omega, q2 projected off Q twice), so the block is
/// [Q | q2] Z^T with Z = [t Omega^T + dt | dt2] = [dt - t Omega | dt2]
/// (Omega skew). Only Z needs a QR (c' x (k + w2) instead of two c x
/// (2k + w2) QRs); the core R_Z^T is truncated by a rank-revealing pivoted QR
/// at rtol (SVD truncation in hodlr_matrix.cpp:56-60).
void compress_level_pieces(DHodlr& D, int l, int k, int w, const double* Om, double rtol, const double* B,
                           const double* T, double* Zw);

void compress_level_structured(DHodlr& D, int l, int k, const double* Om, double rtol) {
    const int W = D.Rl(l);
    if (W == 0) return;
    const int w = W - k;
    const i64 n = D.tree->n();
    double* P = D.Ul(l);
    DVec Z(static_cast<size_t>(n) * w);
    panel_axpby(n, w, 1.0, P + i64(k) * n, n, 0.0, Z.get(), n);
    compress_level_pieces(D, l, k, w, Om, rtol, P + i64(k) * n, P, Z.get());
}

/// The recompression from the level's pieces instead of its assembled panel:
/// B = [q | q2] (left-child rows, n x w), T = t (right-child rows, n x k), and
/// Zw = [dt | dt2] (right-child rows, n x w), overwritten (Z = [dt - t Omega | dt2]
/// is formed in place and factored there).
void compress_level_pieces(DHodlr& D, int l, int k, int w, const double* Om, double rtol, const double* B,
                           const double* T, double* Zw) {
    const DTree& t = *D.tree;
    const i64 n = t.n();
    const Partition& pc = t.part(l);
    const int nodes = 1 << (l - 1);
    const auto& hb = pc.hbounds();
    auto& ctx = current();
    struct ZView {
        double* p;
        double* get() const { return p; }
    } Z{Zw};
    seg_nn(pc, T, n, k, Om, i64(k) * k, k, TMap::parent(0, 0), Z.get(), n, k, -1.0, 1.0);
    std::vector<int> wmin(static_cast<size_t>(nodes));
    int zrows = 0;
    for (int j = 0; j < nodes; ++j) {
        const int cl = hb[static_cast<size_t>(2 * j + 1)] - hb[static_cast<size_t>(2 * j)];
        const int cr = hb[static_cast<size_t>(2 * j + 2)] - hb[static_cast<size_t>(2 * j + 1)];
        wmin[static_cast<size_t>(j)] = std::min({cl, cr, w});
        zrows = std::max(zrows, cr);
    }
    const bool svd = ctx.compression == HG_COMPRESS_JACOBI_SVD;
    // Blocks one CTA factors directly: a column-pivoted QR of Z itself,
    // stopped at the truncation rank, is the rank-revealing factorization
    // (Z P = Q_Z R_Z; block = [Q|q2] P R_Z[:r]^T Q_Z[:, :r]^T), ~r/w of the
    // work of a full QR of Z plus the pivoted QR of its core.
    static const bool direct_ok = [] {  // HG_Z_DIRECT=0: always the two-stage path (A/B knob)
        const char* e = std::getenv("HG_Z_DIRECT");
        return !(e && e[0] == '0');
    }();
    const bool direct = direct_ok && !svd && zrows <= qr_chunk_rows(w);
    std::vector<BatchedQR::Block> blocks;
    for (int j = 0; j < nodes; ++j) {
        QrStop st;
        if (direct) {
            st.rel = rtol;
            st.max_steps = std::max(wmin[static_cast<size_t>(j)], 1);
            st.active = true;
        }
        blocks.push_back({Z.get() + hb[static_cast<size_t>(2 * j + 1)], n,
                          hb[static_cast<size_t>(2 * j + 2)] - hb[static_cast<size_t>(2 * j + 1)], st});
    }
    BatchedQR qz(blocks, w, direct);
    DBuf<int> dwmin, dr(static_cast<size_t>(nodes));
    dwmin.upload(wmin);
    if (direct) {
        k_trunc_rank<<<cdiv(nodes, 128), 128, 0, ctx.stream>>>(nodes, w, qz.R(), dwmin.get(), rtol, dr.get());
        HG_LAUNCH();
        count_launch();
        std::vector<int> r = dl_int(dr);
        int rmax = 0;
        for (int x : r) rmax = std::max(rmax, x);
        auto Pn = rmax ? make_dvec(static_cast<size_t>(n) * static_cast<size_t>(rmax), true) : nullptr;
        if (rmax) {
            DVec Tin(static_cast<size_t>(2 * nodes) * w * rmax);
            k_tins_direct<<<nodes, 256, 0, ctx.stream>>>(w, rmax, dr.get(), qz.R(), qz.perm(), Tin.get());
            HG_LAUNCH();
            count_launch();
            // left' = [Q | q2] P R_Z[:r]^T on left-child rows
            seg_nn(pc, B, n, w, Tin.get(), i64(2) * w * rmax, w, TMap::parent(0, 0), Pn->get(), n,
                   rmax, 1.0, 0.0);
            // right' = Q_Z[:, :r] on right-child rows
            std::vector<double*> out;
            std::vector<i64> ld;
            for (int j = 0; j < nodes; ++j) {
                out.push_back(Pn->get() + hb[static_cast<size_t>(2 * j + 1)]);
                ld.push_back(n);
            }
            qz.form_q(rmax, Tin.get() + i64(w) * rmax, i64(2) * w * rmax, w, out, ld);
        }
        D.R[static_cast<size_t>(l - 1)] = rmax;
        D.U[static_cast<size_t>(l - 1)] = Pn;
        D.V[static_cast<size_t>(l - 1)] = Pn;
        for (int j = 0; j < nodes; ++j) {
            D.rank_up[static_cast<size_t>(l - 1)][static_cast<size_t>(j)] = r[static_cast<size_t>(j)];
            D.rank_lo[static_cast<size_t>(l - 1)][static_cast<size_t>(j)] = r[static_cast<size_t>(j)];
        }
        return;
    }
    DVec M(static_cast<size_t>(nodes) * w * w);
    k_transpose_blocks<<<nodes, 256, 0, ctx.stream>>>(w, qz.R(), M.get());
    HG_LAUNCH();
    count_launch();
    std::unique_ptr<BatchedQR> mq;
    std::unique_ptr<DVec> US, VS;
    if (svd) {
        if (w > 320) throw std::length_error("compress: Jacobi SVD core wider than 320");
        const size_t ws = static_cast<size_t>(nodes) * w * w;
        DVec Aw(ws), Vw(ws);
        US = std::make_unique<DVec>(ws);
        VS = std::make_unique<DVec>(ws);
        k_jacobi_svd<<<nodes, 256, 0, ctx.stream>>>(w, M.get(), dwmin.get(), rtol, Aw.get(), Vw.get(), US->get(),
                                                    VS->get(), dr.get());
        HG_LAUNCH();
        count_launch();
    } else {
        std::vector<BatchedQR::Block> mb;
        for (int j = 0; j < nodes; ++j) {  // k_trunc_rank stops at rtol |r00| or wmin
            QrStop st;
            st.rel = rtol;
            st.max_steps = std::max(wmin[static_cast<size_t>(j)], 1);
            st.active = true;
            mb.push_back({M.get() + i64(j) * w * w, w, w, st});
        }
        mq = std::make_unique<BatchedQR>(mb, w, true);
        k_trunc_rank<<<cdiv(nodes, 128), 128, 0, ctx.stream>>>(nodes, w, mq->R(), dwmin.get(), rtol, dr.get());
        HG_LAUNCH();
        count_launch();
    }
    std::vector<int> r = dl_int(dr);
    int rmax = 0;
    for (int x : r) rmax = std::max(rmax, x);
    auto Pn = rmax ? make_dvec(static_cast<size_t>(n) * static_cast<size_t>(rmax), true) : nullptr;
    if (rmax) {
        // QR mode:  Tin[2j] = Q_M[:, :r_j]; Tin[2j+1] = P_M R_M[:r_j, :]^T
        // SVD mode: Tin[2j] = U_r Sigma_r;  Tin[2j+1] = V_r           (w x rmax each)
        DVec Tin(static_cast<size_t>(2 * nodes) * w * rmax);
        if (svd) {
            k_svd_tins<<<nodes, 256, 0, ctx.stream>>>(w, rmax, dr.get(), US->get(), VS->get(), Tin.get());
        } else {
            std::vector<double*> qo;
            std::vector<i64> ql;
            for (int j = 0; j < nodes; ++j) {
                qo.push_back(Tin.get() + i64(2 * j) * w * rmax);
                ql.push_back(w);
            }
            mq->form_q(rmax, nullptr, 0, 0, qo, ql);
            k_tins<<<nodes, 256, 0, ctx.stream>>>(w, rmax, dr.get(), mq->R(), mq->perm(), Tin.get());
        }
        HG_LAUNCH();
        count_launch();
        // left' = [Q | q2] Q_M[:, :r] on left-child rows (odd rows are overwritten next)
        seg_nn(pc, B, n, w, Tin.get(), i64(2) * w * rmax, w, TMap::parent(0, 0), Pn->get(), n, rmax,
               1.0, 0.0);
        // right' = Q_Z P_M R_M[:r, :]^T on right-child rows
        std::vector<double*> out;
        std::vector<i64> ld;
        for (int j = 0; j < nodes; ++j) {
            out.push_back(Pn->get() + hb[static_cast<size_t>(2 * j + 1)]);
            ld.push_back(n);
        }
        qz.form_q(rmax, Tin.get() + i64(w) * rmax, i64(2) * w * rmax, w, out, ld);
    }
    D.R[static_cast<size_t>(l - 1)] = rmax;
    D.U[static_cast<size_t>(l - 1)] = Pn;
    D.V[static_cast<size_t>(l - 1)] = Pn;
    for (int j = 0; j < nodes; ++j) {
        D.rank_up[static_cast<size_t>(l - 1)][static_cast<size_t>(j)] = r[static_cast<size_t>(j)];
        D.rank_lo[static_cast<size_t>(l - 1)][static_cast<size_t>(j)] = r[static_cast<size_t>(j)];
    }
}

constexpr int COMPLETE_BATCH_ROWS = 0;  // every deficient block takes the batched CholeskyQR path first

/// sketch.cpp:60-74 for every node of a level whose numeric rank is below k.
/// Every deficient block (COMPLETE_BATCH_ROWS = 0) first takes the batched path; a node whose candidates fail the 0.5 test runs the sequential loop one CTA per node (k_complete). Long
/// blocks project the canonical candidates e_0..e_{c-1} twice against the
/// kept columns and orthonormalise them with a (TSQR) Householder QR: the
/// sequential loop computes exactly this Q when every candidate passes the
/// 0.5 norm test, and R_tt is that norm, so a failing test sends the node
/// back to the sequential loop.
void complete_deficient(const Partition& pc, int k, const DBuf<int>& nr, double* S, i64 n) {
    auto& ctx = current();
    const int nodes = pc.nseg() / 2;
    const auto& hb = pc.hbounds();
    const std::vector<int> nrh = nr.download();
    bool any_small = false;
    std::vector<int> big, cj(static_cast<size_t>(nodes), 0), wkeep(static_cast<size_t>(nodes), k);
    int cmax = 0;
    for (int j = 0; j < nodes; ++j) {
        const int m = hb[static_cast<size_t>(2 * j + 1)] - hb[static_cast<size_t>(2 * j)];
        if (nrh[static_cast<size_t>(j)] >= k) continue;
        if (m <= COMPLETE_BATCH_ROWS) {
            any_small = true;
        } else {
            big.push_back(j);
            cj[static_cast<size_t>(j)] = k - nrh[static_cast<size_t>(j)];
            wkeep[static_cast<size_t>(j)] = nrh[static_cast<size_t>(j)];
            cmax = std::max(cmax, cj[static_cast<size_t>(j)]);
        }
    }
    DVec scratch;
    if (any_small) {
        scratch.alloc(static_cast<size_t>(n));
        k_complete<<<nodes, 256, 0, ctx.stream>>>(pc.dbounds(), k, nr.get(), S, n, scratch.get(),
                                                  COMPLETE_BATCH_ROWS);
        HG_LAUNCH();
        count_launch();
    }
    if (big.empty()) return;
    DBuf<int> dcj, dkeep;
    dcj.upload(cj);
    dkeep.upload(wkeep);
    k_mask_cols<<<nodes, 256, 0, ctx.stream>>>(pc.dbounds(), 0, dkeep.get(), k, S, n);
    HG_LAUNCH();
    DVec G(static_cast<size_t>(nodes) * k * cmax), H(static_cast<size_t>(2 * nodes) * k * cmax),
        W(static_cast<size_t>(n) * cmax);
    k_cand_rows<<<nodes, 256, 0, ctx.stream>>>(pc.dbounds(), k, cmax, dcj.get(), S, n, G.get());
    HG_LAUNCH();
    seg_nn(pc, S, n, k, G.get(), i64(k) * cmax, k, TMap::parent(0, 0), W.get(), n, cmax, -1.0, 0.0);
    k_add_canonical<<<nodes, 64, 0, ctx.stream>>>(pc.dbounds(), dcj.get(), W.get(), n);
    HG_LAUNCH();
    seg_tn(pc, S, n, k, W.get(), n, cmax, H.get(), i64(k) * cmax, k);
    seg_nn(pc, S, n, k, H.get(), i64(k) * cmax, k, TMap::same(), W.get(), n, cmax, -1.0, 1.0);
    k_mask_cols<<<nodes, 256, 0, ctx.stream>>>(pc.dbounds(), 0, dcj.get(), cmax, W.get(), n);
    HG_LAUNCH();
    ctx.launches += 4;
    if (cmax > MAX_RANK) throw std::length_error("complete_deficient: more than 128 completion columns");
    std::vector<int> rmap(static_cast<size_t>(nodes), -1);
    for (int j : big) rmap[static_cast<size_t>(j)] = j;
    DVec Gw(static_cast<size_t>(2 * nodes) * cmax * cmax), Rinv(static_cast<size_t>(2 * nodes) * cmax * cmax),
        Rd(static_cast<size_t>(nodes) * cmax * cmax);
    DBuf<int> dfail(static_cast<size_t>(nodes));
    seg_tn(pc, W.get(), n, cmax, W.get(), n, cmax, Gw.get(), i64(cmax) * cmax, cmax);
    {
        const size_t lbytes = sizeof(double) * size_t(cmax) * size_t(cmax | 1);
        if (lbytes > 48 * 1024)
            HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_completion_cholqr),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(lbytes)));
        k_completion_cholqr<<<nodes, 32, lbytes, ctx.stream>>>(dcj.get(), cmax, Gw.get(), Rinv.get(), Rd.get(),
                                                                dfail.get());
    }
    HG_LAUNCH();
    count_launch();
    const std::vector<int> failh = dfail.download();
    std::vector<int> fallback_nr(static_cast<size_t>(nodes), k);
    bool any_fallback = false;
    for (int j : big)
        if (failh[static_cast<size_t>(j)]) {
            rmap[static_cast<size_t>(j)] = -1;
            fallback_nr[static_cast<size_t>(j)] = nrh[static_cast<size_t>(j)];
            any_fallback = true;
        }
    DVec Qw(static_cast<size_t>(n) * cmax);
    seg_nn(pc, W.get(), n, cmax, Rinv.get(), i64(cmax) * cmax, cmax, TMap::same(), Qw.get(), n, cmax, 1.0, 0.0);
    DBuf<int> drmap;
    drmap.upload(rmap);
    const TileList& tl = pc.tiles(256);
    k_place_completion<<<tl.count, 256, 0, ctx.stream>>>(tl.items.get(), dcj.get(), nr.get(), Rd.get(), cmax,
                                                         drmap.get(), Qw.get(), n, S, n);
    HG_LAUNCH();
    count_launch();
    if (any_fallback) {
        DBuf<int> dfb;
        dfb.upload(fallback_nr);
        if (scratch.empty()) scratch.alloc(static_cast<size_t>(n));
        k_complete<<<nodes, 256, 0, ctx.stream>>>(pc.dbounds(), k, dfb.get(), S, n, scratch.get(), 1 << 30);
        HG_LAUNCH();
        count_launch();
    }
}

/// Y = K X - H X with H restricted to levels < l (peeling), full n x s panels.
/// zparity: X is zero on the level-(lmax+1) children of that parity (0: the
/// sketch R_l lives on right children, 1: the bases S, ds, S2 on left ones);
/// -1: no structure (leaf sampler).
/// The oracle half of a peel (Y = K_j X under the sampler's zero-row hint);
/// returns the hint the H half uses.
ZeroRows peel_oracle(const DOracle& o, int j, const DHodlr& H, int lmax, const double* X, int s, double* Y,
                     int zparity) {
    const i64 n = H.n();
    ZeroRows z;
    if (zparity >= 0 && lmax + 1 <= H.tau()) {
        const Partition& pz = H.tree->part(lmax + 1);
        z = ZeroRows{pz.dbounds(), pz.nseg(), zparity, lmax + 1};  // Y is read on the sampler's zero rows only
        o.apply_masked(j, X, n, s, Y, n, z);
    } else {
        o.apply(j, X, n, s, Y, n);
        z.leaf_identity = zparity == -1 && s == H.bmax();  // the leaf sampler
    }
    return z;
}

void peel(const DOracle& o, int j, const DHodlr& H, int lmax, const double* X, int s, double* Y, int zparity) {
    const ZeroRows z = peel_oracle(o, j, H, lmax, X, s, Y, zparity);
    hodlr_apply(H, X, H.n(), s, Y, H.n(), 1, lmax, true, false, 1.0, -1.0, z);
}

/// Peels of one sampler X for the value and every derivative. A derivative
/// that is an affine function of the value, dK/dtheta_q = a K + b I (sigma2
/// of a covariance sigma2 C + nugget I: a = 1/sigma2, b = -nugget/sigma2;
/// DOracle::affine_derivative), is formed from the value apply instead of a
/// second forward-model evaluation of the same columns.
void peel_all(const DOracle& o, const DHodlr& H, const std::vector<DHodlr>& D, int lmax, const double* X, int s,
              double* Yh, const std::vector<double*>& Yd, int zparity) {
    const i64 n = H.n();
    const ZeroRows z = peel_oracle(o, -1, H, lmax, X, s, Yh, zparity);
    for (size_t q = 0; q < D.size(); ++q) {
        double a = 0.0, b = 0.0;
        if (o.affine_derivative(int(q), &a, &b)) {
            panel_axpby(n, s, a, Yh, n, 0.0, Yd[q], n);
            if (b != 0.0) panel_axpby(n, s, b, X, n, 1.0, Yd[q], n);
            o.count_derivative_columns(s);
            hodlr_apply(D[q], X, n, s, Yd[q], n, 1, lmax, true, false, 1.0, -1.0, z);
        } else {
            peel(o, int(q), D[q], lmax, X, s, Yd[q], zparity);
        }
    }
    hodlr_apply(H, X, n, s, Yh, n, 1, lmax, true, false, 1.0, -1.0, z);
}

/// diff_qr core (sketch.cpp:78-111) on one k x k problem: Y = G R^-1 (row
/// substitution, column by column as solve_upper_right), dOmega = skew(strict
/// lower of Y), dR = triu((Y - dOmega) R), ill = !(dmin > 0) || dmax/dmin > 1e12.
__global__ void k_diffqr_core(int k, const double* G, const double* R, double* Y, double* Om, double* dR, int* ill) {
    extern __shared__ double ys[];  // k x k
    const int t = threadIdx.x;
    for (int e = t; e < k * k; e += blockDim.x) ys[e] = G[e];
    __syncthreads();
    for (int j = 0; j < k; ++j) {  // Y(:, j) = (G(:, j) - sum_{i<j} Y(:, i) R(i, j)) / R(j, j)
        for (int row = t; row < k; row += blockDim.x) {
            double x = ys[row + j * k];
            for (int i = 0; i < j; ++i) {
                const double rij = R[i + j * k];
                if (rij != 0.0) x -= ys[row + i * k] * rij;
            }
            ys[row + j * k] = x / R[j + j * k];
        }
        __syncthreads();
    }
    for (int e = t; e < k * k; e += blockDim.x) {
        const int i = e % k, j = e / k;
        Y[e] = ys[e];
        Om[e] = i > j ? ys[e] : (i < j ? -ys[j + i * k] : 0.0);
    }
    __syncthreads();
    for (int e = t; e < k * k; e += blockDim.x) {
        const int i = e % k, j = e / k;
        double s = 0.0;
        if (i <= j)
            for (int l = 0; l <= j; ++l) {
                const double yo = ys[i + l * k] - (i > l ? ys[i + l * k] : (i < l ? -ys[l + i * k] : 0.0));
                s += yo * R[l + j * k];
            }
        dR[e] = s;
    }
    if (t == 0) {
        double dmax = 0.0, dmin = 1.0 / 0.0;
        for (int i = 0; i < k; ++i) {
            dmax = fmax(dmax, fabs(R[i + i * k]));
            dmin = fmin(dmin, fabs(R[i + i * k]));
        }
        *ill = !(dmin > 0) || dmax / dmin > 1e12;
    }
}

/// X <- X R^-1 for an m x k panel (column by column, solve_upper_right).
__global__ void k_solve_upper_right(int m, int k, const double* R, double* X, i64 ldx) {
    for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < m; row += gridDim.x * blockDim.x)
        for (int j = 0; j < k; ++j) {
            double x = X[row + i64(j) * ldx];
            for (int i = 0; i < j; ++i) {
                const double rij = R[i + j * k];
                if (rij != 0.0) x -= X[row + i64(i) * ldx] * rij;
            }
            X[row + i64(j) * ldx] = x / R[j + j * k];
        }
}

size_t diffqr_smem(int k) {
    const size_t b = sizeof(double) * size_t(k) * size_t(k | 1);
    if (b > 48 * 1024)
        HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_diffqr), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(b)));
    return b;
}

}  // namespace

void diff_qr(const double* dB, i64 lddb, const double* Q, i64 ldq, const double* R, int rows, int k, double* dQ,
             i64 lddq, double* dQspan, i64 ldds, double* dR, int* ill) {
    if (k <= 0 || k > MAX_RANK || rows < k) throw std::invalid_argument("diff_qr: need rows >= k, 1 <= k <= 128");
    if (sizeof(double) * k * k > 48 * 1024)
        HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_diffqr_core),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(sizeof(double) * k * k)));
    auto& ctx = current();
    const Partition one(std::vector<int>{0, rows});
    DVec G(static_cast<size_t>(k) * k), Y(static_cast<size_t>(k) * k), Om(static_cast<size_t>(k) * k);
    DVec Rc(static_cast<size_t>(k) * k);
    HG_CUDA(cudaMemcpyAsync(Rc.get(), R, sizeof(double) * k * k, cudaMemcpyDeviceToDevice, ctx.stream));
    seg_tn(one, Q, ldq, k, dB, lddb, k, G.get(), i64(k) * k, k);  // q^T dB
    k_diffqr_core<<<1, 128, sizeof(double) * k * k, ctx.stream>>>(k, G.get(), Rc.get(), Y.get(), Om.get(), dR, ill);
    HG_LAUNCH();
    seg_nn(one, Q, ldq, k, Om.get(), 0, k, TMap::same(), dQspan, ldds, k, 1.0, 0.0);  // q dOmega
    panel_axpby(rows, k, 1.0, dB, lddb, 0.0, dQ, lddq);
    seg_nn(one, Q, ldq, k, G.get(), 0, k, TMap::same(), dQ, lddq, k, -1.0, 1.0);  // dB - q q^T dB
    k_solve_upper_right<<<cdiv(rows, 128), 128, 0, ctx.stream>>>(rows, k, Rc.get(), dQ, lddq);
    HG_LAUNCH();
    ctx.launches += 2;
    panel_axpby(rows, k, 1.0, dQspan, ldds, 1.0, dQ, lddq);
}

void randomized_range(const double* Y, i64 ldy, int rows, int k, double* Q, i64 ldq, double* R, int* perm,
                      int* nr) {
    if (k <= 0 || rows < k) throw std::invalid_argument("randomized_range: need rows >= k >= 1");
    if (k > MAX_RANK) throw std::length_error("randomized_range: rank above 128 not supported");
    auto& ctx = current();
    // one node: the block is the left child, the right child is empty
    const Partition pc(std::vector<int>{0, rows, rows});
    const std::vector<int> qmap{rows == k ? -1 : 0};
    DBuf<int> dqmap;
    dqmap.upload(qmap);
    DVec S(static_cast<size_t>(rows) * k), Rn(static_cast<size_t>(k) * k), sign(static_cast<size_t>(k));
    S.zero();
    DVec Yc(static_cast<size_t>(rows) * k);  // the QR overwrites its input
    panel_axpby(rows, k, 1.0, Y, ldy, 0.0, Yc.get(), rows);
    std::unique_ptr<BatchedQR> qr;
    if (qmap[0] >= 0) {
        qr = std::make_unique<BatchedQR>(std::vector<BatchedQR::Block>{{Yc.get(), rows, rows}}, k, true);
        qr->form_q(k, nullptr, 0, 0, {S.get()}, {rows});
    }
    DVec dummyR(1);
    DBuf<int> dummyP(1), dnr(1), dperm(static_cast<size_t>(k));
    k_range_post<<<1, 128, 0, ctx.stream>>>(k, dqmap.get(), qr ? qr->R() : dummyR.get(), qr ? qr->perm() : dummyP.get(),
                                            Rn.get(), dperm.get(), sign.get(), dnr.get());
    HG_LAUNCH();
    const TileList& tl = pc.tiles(256);
    k_q_sign_rows<<<tl.count, 256, 0, ctx.stream>>>(tl.items.get(), pc.dbounds(), k, dqmap.get(), sign.get(), S.get(),
                                                    rows);
    HG_LAUNCH();
    ctx.launches += 2;
    complete_deficient(pc, k, dnr, S.get(), rows);
    panel_axpby(rows, k, 1.0, S.get(), rows, 0.0, Q, ldq);
    HG_CUDA(cudaMemcpyAsync(R, Rn.get(), sizeof(double) * k * k, cudaMemcpyDeviceToDevice, ctx.stream));
    HG_CUDA(cudaMemcpyAsync(perm, dperm.get(), sizeof(int) * k, cudaMemcpyDeviceToDevice, ctx.stream));
    HG_CUDA(cudaMemcpyAsync(nr, dnr.get(), sizeof(int), cudaMemcpyDeviceToDevice, ctx.stream));
}

namespace {

__device__ __forceinline__ std::uint64_t plan_mix(std::uint64_t z) {  // splitmix64 finalizer
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/// HG_SKETCH_RNG_DEVICE: level sampler rows of odd (right-child) segments get
/// N(0, 1) = Box-Muller of two hashes of (seed, level, row, column); rows of
/// even segments are zero (the pattern of sketch.cpp:12-24).
__global__ void k_plan_level_device(const WorkItem* items, int k, std::uint64_t key, double* P, i64 ldp) {
    const WorkItem it = items[blockIdx.x];
    if (int(threadIdx.x) >= it.rows) return;
    const i64 row = i64(it.row0) + threadIdx.x;
    double* p = P + row;
    if (!(it.seg & 1)) {
        for (int c = 0; c < k; ++c) p[i64(c) * ldp] = 0.0;
        return;
    }
    for (int c = 0; c < k; ++c) {
        const std::uint64_t h1 = plan_mix(key ^ (std::uint64_t(row) * 0x100000001B3ull + std::uint64_t(c)));
        const std::uint64_t h2 = plan_mix(h1 ^ 0xD1B54A32D192ED03ull);
        const double u1 = (double(h1 >> 11) + 1.0) * 0x1.0p-53, u2 = double(h2 >> 11) * 0x1.0p-53;
        p[i64(c) * ldp] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
}

/// Reference stream: `stage` holds a level's draws in draw order (per node the
/// right child's rows x k block, row-major: sketch.cpp:12-24 fills row by row);
/// scatter them into the column-major level sampler, zeros on left-child rows.
__global__ void k_plan_level_scatter(const WorkItem* items, const int* bounds, int k, const double* stage,
                                     const i64* base, double* P, i64 ldp) {
    const WorkItem it = items[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const bool right = it.seg & 1;
    const double* src = right ? stage + base[it.seg >> 1] + i64(it.row0 - bounds[it.seg]) * k : nullptr;
    for (int r = warp; r < it.rows; r += nwarps)  // a warp reads one row's k contiguous draws
        for (int c = lane; c < k; c += 32) P[i64(it.row0 + r) + i64(c) * ldp] = right ? src[i64(r) * k + c] : 0.0;
}

}  // namespace

DSketchPlanP get_plan(DTreeP tree, i64 k, std::uint64_t seed) {
    static std::mutex mu;
    static std::map<std::tuple<const DTree*, i64, std::uint64_t, int>, std::weak_ptr<const DSketchPlan>> cache;
    std::lock_guard<std::mutex> lk(mu);
    const int rng_mode = current().sketch_rng;
    auto key = std::make_tuple(tree.get(), k, seed, rng_mode);
    auto it = cache.find(key);
    if (it != cache.end())
        if (auto sp = it->second.lock()) return sp;
    auto plan = std::make_shared<DSketchPlan>();
    plan->tree = tree;
    plan->k = k;
    plan->seed = seed;
    const ClusterTree& t = tree->host;
    const i64 n = t.size();
    if (rng_mode == 1) {  // HG_SKETCH_RNG_DEVICE
        for (int l = 1; l <= t.depth(); ++l) {
            auto d = make_dvec(static_cast<size_t>(n) * static_cast<size_t>(k), false);
            const TileList& tl = tree->part(l).tiles(256);
            k_plan_level_device<<<tl.count, 256, 0, current().stream>>>(
                tl.items.get(), int(k), seed * 0x9E3779B97F4A7C15ull + std::uint64_t(l) * 0xD6E8FEB86659FD93ull,
                d->get(), n);
            HG_LAUNCH();
            count_launch();
            plan->level.push_back(d);
        }
    }
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    // The stream is sequential (2.7e8 draws at C4): draws land contiguously in draw order
    // (a strided column-major fill cost more than the generator) and are scattered on the device.
    std::vector<double> buf(rng_mode == 1 ? 0 : static_cast<size_t>(n) * static_cast<size_t>(k));
    DVec stage(buf.size());
    DBuf<i64> dbase;
    for (int l = 1; rng_mode != 1 && l <= t.depth(); ++l) {
        const auto& kids = t.level(l);
        std::vector<i64> base(t.level(l - 1).size());
        size_t pos = 0;
        for (size_t j = 0; j < t.level(l - 1).size(); ++j) {
            const Range cr = kids[2 * j + 1];
            base[j] = i64(pos);
            const size_t cnt = static_cast<size_t>(cr.size()) * static_cast<size_t>(k);
            for (size_t e = 0; e < cnt; ++e) buf[pos + e] = gauss(rng);
            pos += cnt;
        }
        auto d = make_dvec(static_cast<size_t>(n) * static_cast<size_t>(k), false);
        HG_CUDA(cudaMemcpyAsync(stage.get(), buf.data(), pos * sizeof(double), cudaMemcpyHostToDevice, current().stream));
        dbase.upload(base);
        const Partition& pl = tree->part(l);
        const TileList& tl = pl.tiles(256);
        k_plan_level_scatter<<<tl.count, 256, 0, current().stream>>>(tl.items.get(), pl.dbounds(), int(k), stage.get(),
                                                                      dbase.get(), d->get(), n);
        HG_LAUNCH();
        count_launch();
        sync();  // the host buffers are reused for the next level
        plan->level.push_back(d);
    }
    plan->leaf = make_dvec(static_cast<size_t>(n) * static_cast<size_t>(tree->bmax), true);
    k_leaf_identity<<<tree->leaves().nseg(), 128, 0, current().stream>>>(tree->leaves().dbounds(), plan->leaf->get(),
                                                                         n);
    HG_LAUNCH();
    count_launch();
    cache[key] = plan;
    // The plan is fixed for a whole fit (mle.cpp:195): keep the most recent
    // ones alive so repeated evaluations reuse the uploaded samplers.
    static std::vector<DSketchPlanP> recent;
    recent.push_back(plan);
    if (recent.size() > 2) recent.erase(recent.begin());
    return plan;
}

DBuildResult build(const DOracle& o, DTreeP tree, i64 kk, const DSketchPlan& plan, bool with_deriv) {
    const ClusterTree& T = tree->host;
    const i64 n = T.size();
    const int tau = T.depth();
    const int k = int(kk);
    if (o.dim() != n) throw std::invalid_argument("build_hodlr: oracle dimension mismatch");
    if (plan.tree.get() != tree.get() || plan.k != kk)
        throw std::invalid_argument("build_hodlr: sketch plan not dimensioned for tree");
    for (int l = 1; l <= tau; ++l) {  // sketch.cpp:115-126
        const auto& kids = T.level(l);
        for (size_t j = 0; j < T.level(l - 1).size(); ++j)
            if (kk > std::min(kids[2 * j].size(), kids[2 * j + 1].size()))
                throw std::invalid_argument("build_hodlr: rank " + std::to_string(kk) +
                                            " exceeds block dimension at level " + std::to_string(l));
    }
    if (k > MAX_RANK) throw std::length_error("build_hodlr: rank above 128 not supported");
    const int p = with_deriv ? o.num_params() : 0;
    const int kp = k * p;
    DBuildResult out;
    out.p = p;
    out.h = DHodlr::zero(tree);
    for (int q = 0; q < p; ++q) out.deriv.push_back(DHodlr::zero(tree));
    // Omega (in-span rotation of diff_qr) per param and level, for the recompression.
    std::vector<std::vector<DVecP>> omegas(static_cast<size_t>(p), std::vector<DVecP>(static_cast<size_t>(tau)));
    auto& ctx = current();
    // which derivatives are compressed as each level is committed
    // (HG_OPT_COMPRESS_AT; HG_COMPRESS_LEVEL_MASK: per-parameter bit mask, tuning knob)
    static const unsigned level_mask = [] {
        const char* e = std::getenv("HG_COMPRESS_LEVEL_MASK");
        return e ? unsigned(std::strtoul(e, nullptr, 0)) : ~0u;
    }();
    auto at_level = [&](int q) { return ctx.compress_at == HG_COMPRESS_AT_LEVEL && ((level_mask >> q) & 1u); };

    for (int l = 1; l <= tau; ++l) {
        const Partition& pc = tree->part(l);
        const auto& hb = pc.hbounds();
        const int nodes = 1 << (l - 1);
        const double* Rs = plan.level[static_cast<size_t>(l - 1)]->get();
        // Pass 1: Y = K R - H R, dY_j = K_j R - D_j R (sketch.cpp:151-154).
        DVec Y(static_cast<size_t>(n) * k), dY(static_cast<size_t>(n) * std::max(kp, 1));
        {
            std::vector<double*> yd;
            for (int q = 0; q < p; ++q) yd.push_back(dY.get() + i64(q) * k * n);
            peel_all(o, out.h, out.deriv, l - 1, Rs, k, Y.get(), yd, 0);
        }
        // Range finder per node (sketch.cpp:156-175).
        std::vector<int> qmap(static_cast<size_t>(nodes), -1);
        std::vector<BatchedQR::Block> blocks;
        for (int j = 0; j < nodes; ++j) {
            const int m = hb[static_cast<size_t>(2 * j + 1)] - hb[static_cast<size_t>(2 * j)];
            if (m == k) continue;
            qmap[static_cast<size_t>(j)] = int(blocks.size());
            // only R's diagonal up to the numeric rank (64 eps |r00|, k_range_post)
            // and Q's first nr columns are read: stop the pivoted QR there
            QrStop st;
            st.rel = 64 * DBL_EPSILON;
            st.max_steps = k;
            st.active = true;
            blocks.push_back({Y.get() + hb[static_cast<size_t>(2 * j)], n, m, st});
        }
        DBuf<int> dqmap;
        dqmap.upload(qmap);
        DVec Rn(static_cast<size_t>(nodes) * k * k), sign(static_cast<size_t>(nodes) * k);
        DBuf<int> perm(static_cast<size_t>(nodes) * k), nr(static_cast<size_t>(nodes));
        // One panel per level, [ds_0 | .. | ds_{p-1} | q | q2]: the value
        // peel reads [ds | q] and each derivative peel [q | q2] as contiguous
        // column ranges of it (no copies). q and q2 start zero (their bases
        // only fill left-child rows).
        struct PView {
            double* p;
            double* get() const { return p; }
        };
        DVec SB(static_cast<size_t>(n) * static_cast<size_t>(k * (1 + p) + kp));
        const PView S{SB.get() + i64(p) * k * n};
        panel_axpby(n, k + kp, 0.0, nullptr, 0, 0.0, S.get(), n);
        {
            std::unique_ptr<BatchedQR> qr;
            if (!blocks.empty()) qr = std::make_unique<BatchedQR>(blocks, k, true);
            DVec dummyR(1);
            DBuf<int> dummyP(1);
            k_range_post<<<nodes, 128, 0, ctx.stream>>>(k, dqmap.get(), qr ? qr->R() : dummyR.get(),
                                                        qr ? qr->perm() : dummyP.get(), Rn.get(), perm.get(),
                                                        sign.get(), nr.get());
            HG_LAUNCH();
            if (qr) {
                // Q columns past a node's numeric rank are replaced by the
                // completion below: form only the widest numeric rank
                const std::vector<int> nrh = nr.download();
                int nrmax = 1;
                std::vector<double*> qo;
                std::vector<i64> ql;
                for (int j = 0; j < nodes; ++j)
                    if (qmap[static_cast<size_t>(j)] >= 0) {
                        nrmax = std::max(nrmax, nrh[static_cast<size_t>(j)]);
                        qo.push_back(S.get() + hb[static_cast<size_t>(2 * j)]);
                        ql.push_back(n);
                    }
                qr->form_q(nrmax, nullptr, 0, 0, qo, ql);
            }
            const TileList& tl256 = pc.tiles(256);
            k_q_sign_rows<<<tl256.count, 256, 0, ctx.stream>>>(tl256.items.get(), pc.dbounds(), k, dqmap.get(),
                                                               sign.get(), S.get(), n);
            HG_LAUNCH();
            ctx.launches += 2;
            complete_deficient(pc, k, nr, S.get(), n);
        }
        // Pass 2, Z = K S - H S (sketch.cpp:177-183), and the value half of
        // every differentiated pass, K ds_q - H ds_q (:270-271), in ONE peel
        // over [S | ds_0 | .. | ds_{p-1}]: the coarser levels' panels are
        // streamed once instead of 1 + p times. ds_q = S Omega_q needs only
        // S and dY (diff_qr, :245-268), not Z.
        std::vector<DVecP> oms(static_cast<size_t>(p));
        std::vector<std::vector<int>> rws(static_cast<size_t>(p));
        DVec ZX(static_cast<size_t>(n) * k * (1 + p));
        double* SX = SB.get();  // [ds_0 | .. | ds_{p-1} | q]
        for (int q = 0; q < p; ++q) {
            DVec G(static_cast<size_t>(2 * nodes) * k * k);
            DVecP OmP = make_dvec(static_cast<size_t>(nodes) * k * k, false);
            omegas[static_cast<size_t>(q)][static_cast<size_t>(l - 1)] = OmP;
            DBuf<int> rw(static_cast<size_t>(nodes)), ill(static_cast<size_t>(nodes));
            const double* dYq = dY.get() + i64(q) * k * n;
            seg_tn(pc, S.get(), n, k, dYq, n, k, G.get(), i64(k) * k, k);
            k_diffqr<<<nodes, k <= 64 ? 64 : 128, diffqr_smem(k), ctx.stream>>>(k, G.get(), Rn.get(), perm.get(), nr.get(), dqmap.get(),
                                                   OmP->get(), rw.get(), ill.get());
            HG_LAUNCH();
            ++ctx.launches;
            seg_nn(pc, S.get(), n, k, OmP->get(), i64(k) * k, k, TMap::parent(0, 0), SX + i64(q) * k * n, n,
                   k, 1.0, 0.0);
            rws[static_cast<size_t>(q)] = rw.download();
            std::vector<int> ic = ill.download();
            for (int x : ic) out.warnings += x;
        }
        peel(o, -1, out.h, l - 1, SX, k * (1 + p), ZX.get(), 1);
        const double* Z = ZX.get() + i64(p) * k * n;

        // q2 residual bases (sketch.cpp:194-233).
        std::vector<int> w2(static_cast<size_t>(nodes), 0);
        int w2max = 0;
        const PView S2{S.get() + i64(k) * n};
        DBuf<int> dw2(static_cast<size_t>(nodes));
        dw2.zero();
        if (p > 0) {
            // the residual is projected in place: dY's last use (diff_qr) is done
            const PView resid{dY.get()};
            DVec presc(static_cast<size_t>(nodes)), G(static_cast<size_t>(2 * nodes) * k * kp);
            {
                const TileList& tl = pc.tiles(2048);
                DVec part(static_cast<size_t>(tl.count) * p);
                k_presc_part<<<tl.count, 256, 0, ctx.stream>>>(tl.items.get(), k, p, dY.get(), n, part.get());
                HG_LAUNCH();
                k_presc_final<<<cdiv(nodes, 128), 128, 0, ctx.stream>>>(nodes, tl.seg_first.get(), p, part.get(),
                                                                      presc.get());
                HG_LAUNCH();
                ctx.launches += 2;
            }
            for (int pass = 0; pass < 2; ++pass) {
                seg_tn(pc, S.get(), n, k, resid.get(), n, kp, G.get(), i64(k) * kp, k);
                seg_nn(pc, S.get(), n, k, G.get(), i64(k) * kp, k, TMap::same(), resid.get(), n, kp, -1.0, 1.0);
            }
            std::vector<BatchedQR::Block> b2;
            for (int j = 0; j < nodes; ++j)
                if (qmap[static_cast<size_t>(j)] >= 0) {
                    // k_w2_nodes reads the diagonal up to the first entry at the
                    // floor max(1e-10 |r00|, 1e-12 presc_j) or the cap: stop there
                    const int m = hb[static_cast<size_t>(2 * j + 1)] - hb[static_cast<size_t>(2 * j)];
                    QrStop st;
                    st.rel = 1e-10;
                    st.abs_scale = 1e-12;
                    st.abs_ptr = presc.get() + j;
                    st.max_steps = std::max(std::min(kp, m - k), 1);
                    st.active = true;
                    b2.push_back({resid.get() + hb[static_cast<size_t>(2 * j)], n, m, st});
                }
            std::unique_ptr<BatchedQR> qr2;
            if (!b2.empty()) {
                qr2 = std::make_unique<BatchedQR>(b2, kp, true);
                k_w2_nodes<<<cdiv(nodes, 128), 128, 0, ctx.stream>>>(nodes, pc.dbounds(), k, kp, dqmap.get(), qr2->R(),
                                                                    presc.get(), dw2.get());
                HG_LAUNCH();
                ++ctx.launches;
                w2 = dw2.download();
                for (int x : w2) w2max = std::max(w2max, x);
            }
            if (w2max > 0) {
                std::vector<double*> qo;
                std::vector<i64> ql;
                for (int j = 0; j < nodes; ++j)
                    if (qmap[static_cast<size_t>(j)] >= 0) {
                        qo.push_back(S2.get() + hb[static_cast<size_t>(2 * j)]);
                        ql.push_back(n);
                    }
                qr2->form_q(w2max, nullptr, 0, 0, qo, ql);
                k_mask_cols<<<nodes, 256, 0, ctx.stream>>>(pc.dbounds(), 0, dw2.get(), w2max, S2.get(), n);
                HG_LAUNCH();
                ++ctx.launches;
                if (ctx.q2_basis == HG_Q2_REORTHOGONALIZED) {
                    // q2 columns kept near the w2 floor are the normalised
                    // projection roundoff of the derivative sketch and overlap q
                    // by up to roundoff / floor; that overlap double-counts
                    // dK q in the committed block [dqc | q | q2][t | dt | dt2]^T.
                    // One more projection against q (CGS2) and a
                    // renormalisation make [q | q2] orthonormal to roundoff.
                    DVec G2(static_cast<size_t>(2 * nodes) * k * w2max);
                    seg_tn(pc, S.get(), n, k, S2.get(), n, w2max, G2.get(), i64(k) * w2max, k);
                    seg_nn(pc, S.get(), n, k, G2.get(), i64(k) * w2max, k, TMap::same(), S2.get(), n, w2max, -1.0,
                           1.0);
                    k_col_normalize<<<dim3(unsigned(nodes), unsigned(w2max)), 256, 0, ctx.stream>>>(
                        pc.dbounds(), dw2.get(), S2.get(), n);
                    HG_LAUNCH();
                    ++ctx.launches;
                }
            }
        }

        // Differentiated passes (sketch.cpp:236-295) and the commit (:297-311):
        // dZ_q = K_q S - D_q S + (K ds_q - H ds_q), dZ2_q = K_q q2 - D_q q2,
        // the D_q applies to [S | q2] in one peel.
        for (int q = 0; q < p; ++q) {
            const double* ds = SX + i64(q) * k * n;
            const int wq = k + w2max;
            const PView X2{S.get()};  // [q | q2]
            DVec O2(static_cast<size_t>(n) * wq);
            peel(o, q, out.deriv[static_cast<size_t>(q)], l - 1, X2.get(), wq, O2.get(), 1);
            double* dZ = O2.get();
            panel_axpby(n, k, 1.0, ZX.get() + i64(q) * k * n, n, 1.0, dZ, n);
            double* dZ2 = O2.get() + i64(k) * n;
            if (w2max > 0) {
                k_mask_cols<<<nodes, 256, 0, ctx.stream>>>(pc.dbounds(), 1, dw2.get(), w2max, dZ2, n);
                HG_LAUNCH();
                ++ctx.launches;
            }
            DHodlr& D = out.deriv[static_cast<size_t>(q)];
            if (at_level(q)) {
                // HG_COMPRESS_AT_LEVEL: compress the level as it is committed,
                // straight from its pieces (left basis [q | q2] = X2, t = Z,
                // [dt | dt2] = O2 factored in place), so every finer level's
                // peels stream the compressed (rank ~3..8) panels instead of
                // the 2k + w2 wide concatenation, which is never assembled
                for (int j = 0; j < nodes; ++j) {
                    D.rank_up[static_cast<size_t>(l - 1)][static_cast<size_t>(j)] = 2 * k + w2[static_cast<size_t>(j)];
                    D.rank_lo[static_cast<size_t>(l - 1)][static_cast<size_t>(j)] = 2 * k + w2[static_cast<size_t>(j)];
                }
                compress_level_pieces(D, l, k, wq, omegas[static_cast<size_t>(q)][static_cast<size_t>(l - 1)]->get(),
                                      1e-13, X2.get(), Z, O2.get());
                continue;
            }
            // Derivative level panel: [dqc | q | q2] on left rows, [t | dt | dt2] on right rows.
            const int Wd = 2 * k + w2max;
            D.set_level(l, Wd, true);
            double* Pd = D.Ul(l);
            panel_parity_select(pc, k, ds, n, 1.0, Z, n, 1.0, Pd, n);
            panel_parity_select(pc, k, S.get(), n, 1.0, dZ, n, 1.0, Pd + i64(k) * n, n);
            if (w2max > 0) panel_parity_select(pc, w2max, S2.get(), n, 1.0, dZ2, n, 1.0, Pd + i64(2 * k) * n, n);
            for (int j = 0; j < nodes; ++j) {
                D.rank_up[static_cast<size_t>(l - 1)][static_cast<size_t>(j)] = 2 * k + w2[static_cast<size_t>(j)];
                D.rank_lo[static_cast<size_t>(l - 1)][static_cast<size_t>(j)] = 2 * k + w2[static_cast<size_t>(j)];
            }
        }
        // Value level panel: q on left rows, t = Z on right rows.
        out.h.set_level(l, k, true);
        panel_parity_select(pc, k, S.get(), n, 1.0, Z, n, 1.0, out.h.Ul(l), n);
        for (int j = 0; j < nodes; ++j) {
            out.h.rank_up[static_cast<size_t>(l - 1)][static_cast<size_t>(j)] = k;
            out.h.rank_lo[static_cast<size_t>(l - 1)][static_cast<size_t>(j)] = k;
        }
        std::vector<int> nrh = nr.download();
        for (int j = 0; j < nodes; ++j) {
            out.decisions.push_back(nrh[static_cast<size_t>(j)]);
            out.decisions.push_back(w2[static_cast<size_t>(j)]);
            for (int q = 0; q < p; ++q) out.decisions.push_back(rws[static_cast<size_t>(q)][static_cast<size_t>(j)]);
        }
    }

    // Leaves (sketch.cpp:314-329): identity-concatenation sampler.
    {
        const int bm = tree->bmax;
        DVec Yl(static_cast<size_t>(n) * bm * (1 + p));
        std::vector<double*> yd;
        for (int q = 0; q < p; ++q) yd.push_back(Yl.get() + i64(1 + q) * bm * n);
        peel_all(o, out.h, out.deriv, tau, plan.leaf->get(), bm, Yl.get(), yd, -1);
        auto to_leaves = [&](DHodlr& h, double* P) {
            leaves_panel(*tree, h.leaves->get(), P, false);
            h.leaves_zero = false;
        };
        to_leaves(out.h, Yl.get());
        for (int q = 0; q < p; ++q) to_leaves(out.deriv[static_cast<size_t>(q)], yd[static_cast<size_t>(q)]);
    }
    // Recompress every derivative off-diagonal block (sketch.cpp:331-341).
    for (int q = 0; q < p; ++q)
        for (int l = 1; l <= tau && !at_level(q); ++l)
            compress_level_structured(out.deriv[static_cast<size_t>(q)], l, k,
                                      omegas[static_cast<size_t>(q)][static_cast<size_t>(l - 1)]->get(), 1e-13);
    return out;
}

}  // namespace hg
