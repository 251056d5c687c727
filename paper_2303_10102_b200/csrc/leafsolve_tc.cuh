// Leaf solve on the FP64 tensor cores (included by factor.cu inside its
// anonymous namespace; needs tile.cuh).
//
// Cholesky leaves of at most 128 rows. Once per factorization every 16x16
// diagonal block L_jj of every leaf factor is replaced in place by its inverse
// (k_leaf_diag_inv, substitution on identity columns; the strict upper part
// is zeroed). A solve then never runs a serial substitution: with the packed
// factor and a 128 x 32 RHS tile resident in shared memory,
//   forward  L x = b   (right-looking): x_j = L_jj^{-1} y_j,
//                                       y_{>j} -= L[>j, j] x_j
//   backward L^T x = y (left-looking):  x_j = L_jj^{-T} (y_j - L[>j, j]^T x_{>j})
// are all DMMA m8n8k4 products against the 16-column panel L[16j:, 16j:16j+16]
// (both passes use the same panel). Each warp owns 8 RHS columns end to end,
// so after the loads there are no block-wide barriers; a CTA runs several
// column tiles of one leaf against one load of its factor. Numerics: the
// diagonal-block inverses act on 16x16 triangles only (cond(L_jj) <=
// sqrt(cond(A_jj))); tests/test_gpu_build_mle.py holds the C1 parity bounds
// this path is checked against.

// Whole packed factor resident: panel j (rows [16j, mp), 16 columns) at
// ts_poff(j) with leading dimension mp - 16j + 4 (4 mod 16 doubles: the
// fragment loads below are bank-conflict free); 32 RHS columns per CTA,
// 4 warps x 8 columns, two CTAs per SM (one loads while the other computes).
constexpr int TS_NC = 32, TS_MAX = 128, TS_YLD = TS_NC + 4, TS_THREADS = 128;
#ifndef HG_TS_S
#define HG_TS_S 1
#endif
constexpr int TS_S = HG_TS_S;  // 8-column subtiles per warp in the 128-row kernel (2 measured 28% slower: fewer warps)
constexpr int TS_LSIZE = 16 * (TS_MAX * (TS_MAX / 16 + 1) / 2 + 4 * (TS_MAX / 16));  // packed panels, mp = 128
constexpr size_t TS_SMEM = (size_t(TS_MAX) * TS_YLD + TS_LSIZE) * sizeof(double);
__device__ __forceinline__ int ts_poff(int j, int mp) { return 16 * j * (mp + 4) - 128 * j * (j - 1); }

struct LeafSolveTcArgs {
    const int* bounds;
    int bmax;
    const double* fac;
    double* Y;
    i64 ldy;
    int w, ctiles, cpt;  // column tiles, tiles per CTA
};

/// In place: every 16x16 diagonal block of each leaf's Cholesky factor ->
/// its inverse (lower triangular, strict upper part zeroed). One CTA per
/// leaf, thread (block jb, column c).
__global__ void __launch_bounds__(256) k_leaf_diag_inv(const int* bounds, int bmax, double* fac) {
    __shared__ double Ls[16][16][17];  // up to 256-row leaves (blockDim = 16 per diagonal block)
    const int b = blockIdx.x, m = bounds[b + 1] - bounds[b];
    const int jb = threadIdx.x >> 4, c = threadIdx.x & 15;
    const int r0 = 16 * jb, mb = min(16, m - r0);
    double* F = fac + i64(b) * bmax * bmax;
    if (mb > 0)
        for (int r = 0; r < mb; ++r)
            if (c < mb) Ls[jb][r][c] = F[(r0 + r) + i64(r0 + c) * bmax];
    __syncthreads();
    if (mb <= 0 || c >= mb) return;
    double x[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        if (r < mb) {
            double s = (r == c) ? 1.0 : 0.0;
            for (int p = c; p < r; ++p) s -= Ls[jb][r][p] * x[p];
            x[r] = r < c ? 0.0 : s / Ls[jb][r][r];
        } else {
            x[r] = 0.0;
        }
    }
#pragma unroll
    for (int r = 0; r < 16; ++r)
        if (r < mb) F[(r0 + r) + i64(r0 + c) * bmax] = x[r];
}

/// Every panel of the factor into the packed layout (cp.async); padding
/// rows/columns (>= m) act as the identity.
__device__ __forceinline__ void ts_load_factor(double* L, const double* F, int ldf, int m, int mp) {
    const int nb = mp / 16;
    for (int j = 0; j < nb; ++j) {
        const int r0 = 16 * j, rows = mp - r0, ld = rows + 4;
        double* P = L + ts_poff(j, mp);
        for (int e = threadIdx.x; e < rows * 16; e += blockDim.x) {
            const int r = e % rows, c = e / rows;
            const int gr = r0 + r, gc = r0 + c;
            double* d = P + c * ld + r;
            if (gr < m && gc < m)
                tile::cp_async8(d, F + gr + i64(gc) * ldf, true);
            else
                *d = (gr == gc) ? 1.0 : 0.0;
        }
    }
}

/// Forward substitution L x = b on rows [row0, row0 + mp) of the RHS tile
/// (this warp's 8 columns) against the packed factor Ls of mp rows.
__device__ __forceinline__ void ts_forward(const double* Ls, int mp, double* Ys, int row0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g8 = lane >> 2, t4 = lane & 3, n0 = warp * 8;
    const int nb = mp / 16;
    // ---- forward: L x = b
    for (int j = 0; j < nb; ++j) {
        const double* P = Ls + ts_poff(j, mp);
        const int ld = mp - 16 * j + 4;
        double* Yj = Ys + (row0 + 16 * j) * TS_YLD + n0;
        {  // x_j = L_jj^{-1} y_j
            double yb[4], x0[2] = {0.0, 0.0}, x1[2] = {0.0, 0.0};
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) yb[kk] = Yj[(4 * kk + t4) * TS_YLD + g8];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                tile::dmma(x0, P[(4 * kk + t4) * ld + g8], yb[kk]);
                tile::dmma(x1, P[(4 * kk + t4) * ld + 8 + g8], yb[kk]);
            }
            __syncwarp();
            Yj[g8 * TS_YLD + 2 * t4] = x0[0];
            Yj[g8 * TS_YLD + 2 * t4 + 1] = x0[1];
            Yj[(8 + g8) * TS_YLD + 2 * t4] = x1[0];
            Yj[(8 + g8) * TS_YLD + 2 * t4 + 1] = x1[1];
            __syncwarp();
        }
        // rows [16(j+1), mp) -= L[16(j+1):, 16j:16j+16] x_j
        const int nrt = (mp - 16 * j) / 8;
        double bf[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) bf[kk] = Yj[(4 * kk + t4) * TS_YLD + g8];
        constexpr int MT = TS_MAX / 8 - 2;
        double acc[MT][2];
#pragma unroll
        for (int t = 0; t < MT; ++t) {
            acc[t][0] = acc[t][1] = 0.0;
            if (t + 2 < nrt) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) tile::dmma(acc[t], P[(4 * kk + t4) * ld + (t + 2) * 8 + g8], bf[kk]);
            }
        }
#pragma unroll
        for (int t = 0; t < MT; ++t)
            if (t + 2 < nrt) {
                double* yp = Yj + ((t + 2) * 8 + g8) * TS_YLD + 2 * t4;
                yp[0] -= acc[t][0];
                yp[1] -= acc[t][1];
            }
        __syncwarp();
    }
}

/// Backward substitution L^T x = y on rows [row0, row0 + mp) (see ts_forward).
__device__ __forceinline__ void ts_backward(const double* Ls, int mp, double* Ys, int row0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g8 = lane >> 2, t4 = lane & 3, n0 = warp * 8;
    const int nb = mp / 16;
    // ---- backward: L^T x = y
    for (int j = nb - 1; j >= 0; --j) {
        const double* P = Ls + ts_poff(j, mp);
        const int ld = mp - 16 * j + 4;
        double* Yj = Ys + (row0 + 16 * j) * TS_YLD + n0;
        // r_j = y_j - L[16(j+1):, 16j:16j+16]^T x_{>j}
        const int K = mp - 16 * (j + 1);
        double a0[2] = {0.0, 0.0}, a1[2] = {0.0, 0.0}, b0[2] = {0.0, 0.0}, b1[2] = {0.0, 0.0};
        const double* Xb = Yj + 16 * TS_YLD + g8;
        int k4 = 0;
        for (; k4 + 8 <= K; k4 += 8) {
            const double x0 = Xb[(k4 + t4) * TS_YLD], x1 = Xb[(k4 + 4 + t4) * TS_YLD];
            tile::dmma(a0, P[g8 * ld + 16 + k4 + t4], x0);
            tile::dmma(a1, P[(8 + g8) * ld + 16 + k4 + t4], x0);
            tile::dmma(b0, P[g8 * ld + 16 + k4 + 4 + t4], x1);
            tile::dmma(b1, P[(8 + g8) * ld + 16 + k4 + 4 + t4], x1);
        }
        if (k4 < K) {
            const double x0 = Xb[(k4 + t4) * TS_YLD];
            tile::dmma(a0, P[g8 * ld + 16 + k4 + t4], x0);
            tile::dmma(a1, P[(8 + g8) * ld + 16 + k4 + t4], x0);
        }
        double* y0 = Yj + g8 * TS_YLD + 2 * t4;
        double* y1 = y0 + 8 * TS_YLD;
        y0[0] -= a0[0] + b0[0];
        y0[1] -= a0[1] + b0[1];
        y1[0] -= a1[0] + b1[0];
        y1[1] -= a1[1] + b1[1];
        __syncwarp();
        {  // x_j = L_jj^{-T} r_j
            double rb[4], x0[2] = {0.0, 0.0}, x1[2] = {0.0, 0.0};
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) rb[kk] = Yj[(4 * kk + t4) * TS_YLD + g8];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                tile::dmma(x0, P[g8 * ld + 4 * kk + t4], rb[kk]);
                tile::dmma(x1, P[(8 + g8) * ld + 4 * kk + t4], rb[kk]);
            }
            __syncwarp();
            y0[0] = x0[0];
            y0[1] = x0[1];
            y1[0] = x1[0];
            y1[1] = x1[1];
            __syncwarp();
        }
    }
}

/// ts_forward / ts_backward with S 8-column subtiles per warp: every factor
/// fragment loaded from shared memory feeds S DMMAs (the single-subtile
/// kernel is bound by those fragment loads, profiles/r1_ncu_qr_leafsolve.md).
template <int S>
__device__ __forceinline__ void ts_forward_s(const double* Ls, int mp, double* Ys, int row0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g8 = lane >> 2, t4 = lane & 3, n0 = warp * 8 * S;
    const int nb = mp / 16;
    for (int j = 0; j < nb; ++j) {
        const double* P = Ls + ts_poff(j, mp);
        const int ld = mp - 16 * j + 4;
        double* Yj = Ys + (row0 + 16 * j) * TS_YLD + n0;
        {  // x_j = L_jj^{-1} y_j
            double yb[S][4], x0[S][2], x1[S][2];
#pragma unroll
            for (int u = 0; u < S; ++u) {
                x0[u][0] = x0[u][1] = x1[u][0] = x1[u][1] = 0.0;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) yb[u][kk] = Yj[(4 * kk + t4) * TS_YLD + 8 * u + g8];
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const double p0 = P[(4 * kk + t4) * ld + g8], p1 = P[(4 * kk + t4) * ld + 8 + g8];
#pragma unroll
                for (int u = 0; u < S; ++u) {
                    tile::dmma(x0[u], p0, yb[u][kk]);
                    tile::dmma(x1[u], p1, yb[u][kk]);
                }
            }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < S; ++u) {
                Yj[g8 * TS_YLD + 8 * u + 2 * t4] = x0[u][0];
                Yj[g8 * TS_YLD + 8 * u + 2 * t4 + 1] = x0[u][1];
                Yj[(8 + g8) * TS_YLD + 8 * u + 2 * t4] = x1[u][0];
                Yj[(8 + g8) * TS_YLD + 8 * u + 2 * t4 + 1] = x1[u][1];
            }
            __syncwarp();
        }
        const int nrt = (mp - 16 * j) / 8;
        double bf[S][4];
#pragma unroll
        for (int u = 0; u < S; ++u)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) bf[u][kk] = Yj[(4 * kk + t4) * TS_YLD + 8 * u + g8];
        constexpr int MT = TS_MAX / 8 - 2;
        double acc[MT][S][2];
#pragma unroll
        for (int t = 0; t < MT; ++t) {
#pragma unroll
            for (int u = 0; u < S; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
            if (t + 2 < nrt) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const double a = P[(4 * kk + t4) * ld + (t + 2) * 8 + g8];
#pragma unroll
                    for (int u = 0; u < S; ++u) tile::dmma(acc[t][u], a, bf[u][kk]);
                }
            }
        }
#pragma unroll
        for (int t = 0; t < MT; ++t)
            if (t + 2 < nrt) {
#pragma unroll
                for (int u = 0; u < S; ++u) {
                    double* yp = Yj + ((t + 2) * 8 + g8) * TS_YLD + 8 * u + 2 * t4;
                    yp[0] -= acc[t][u][0];
                    yp[1] -= acc[t][u][1];
                }
            }
        __syncwarp();
    }
}

template <int S>
__device__ __forceinline__ void ts_backward_s(const double* Ls, int mp, double* Ys, int row0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g8 = lane >> 2, t4 = lane & 3, n0 = warp * 8 * S;
    const int nb = mp / 16;
    for (int j = nb - 1; j >= 0; --j) {
        const double* P = Ls + ts_poff(j, mp);
        const int ld = mp - 16 * j + 4;
        double* Yj = Ys + (row0 + 16 * j) * TS_YLD + n0;
        const int K = mp - 16 * (j + 1);
        double a0[S][2], a1[S][2], b0[S][2], b1[S][2];
#pragma unroll
        for (int u = 0; u < S; ++u) a0[u][0] = a0[u][1] = a1[u][0] = a1[u][1] = b0[u][0] = b0[u][1] = b1[u][0] = b1[u][1] = 0.0;
        const double* Xb = Yj + 16 * TS_YLD + g8;
        int k4 = 0;
        for (; k4 + 8 <= K; k4 += 8) {
            const double p00 = P[g8 * ld + 16 + k4 + t4], p10 = P[(8 + g8) * ld + 16 + k4 + t4];
            const double p01 = P[g8 * ld + 16 + k4 + 4 + t4], p11 = P[(8 + g8) * ld + 16 + k4 + 4 + t4];
#pragma unroll
            for (int u = 0; u < S; ++u) {
                const double x0 = Xb[(k4 + t4) * TS_YLD + 8 * u], x1 = Xb[(k4 + 4 + t4) * TS_YLD + 8 * u];
                tile::dmma(a0[u], p00, x0);
                tile::dmma(a1[u], p10, x0);
                tile::dmma(b0[u], p01, x1);
                tile::dmma(b1[u], p11, x1);
            }
        }
        if (k4 < K) {
            const double p00 = P[g8 * ld + 16 + k4 + t4], p10 = P[(8 + g8) * ld + 16 + k4 + t4];
#pragma unroll
            for (int u = 0; u < S; ++u) {
                const double x0 = Xb[(k4 + t4) * TS_YLD + 8 * u];
                tile::dmma(a0[u], p00, x0);
                tile::dmma(a1[u], p10, x0);
            }
        }
#pragma unroll
        for (int u = 0; u < S; ++u) {
            double* y0 = Yj + g8 * TS_YLD + 8 * u + 2 * t4;
            double* y1 = y0 + 8 * TS_YLD;
            y0[0] -= a0[u][0] + b0[u][0];
            y0[1] -= a0[u][1] + b0[u][1];
            y1[0] -= a1[u][0] + b1[u][0];
            y1[1] -= a1[u][1] + b1[u][1];
        }
        __syncwarp();
        {  // x_j = L_jj^{-T} r_j
            double rb[S][4], x0[S][2], x1[S][2];
#pragma unroll
            for (int u = 0; u < S; ++u) {
                x0[u][0] = x0[u][1] = x1[u][0] = x1[u][1] = 0.0;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) rb[u][kk] = Yj[(4 * kk + t4) * TS_YLD + 8 * u + g8];
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const double p0 = P[g8 * ld + 4 * kk + t4], p1 = P[(8 + g8) * ld + 4 * kk + t4];
#pragma unroll
                for (int u = 0; u < S; ++u) {
                    tile::dmma(x0[u], p0, rb[u][kk]);
                    tile::dmma(x1[u], p1, rb[u][kk]);
                }
            }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < S; ++u) {
                double* y0 = Yj + g8 * TS_YLD + 8 * u + 2 * t4;
                double* y1 = y0 + 8 * TS_YLD;
                y0[0] = x0[u][0];
                y0[1] = x0[u][1];
                y1[0] = x1[u][0];
                y1[1] = x1[u][1];
            }
            __syncwarp();
        }
    }
}

template <int S>
__global__ void __launch_bounds__(TS_NC * 4 / S, 2) k_leaf_solve_tc(LeafSolveTcArgs g) {
    extern __shared__ double sm[];
    double* Ys = sm;
    double* Ls = sm + TS_MAX * TS_YLD;
    const int groups = (g.ctiles + g.cpt - 1) / g.cpt;
    const int b = blockIdx.x / groups, grp = blockIdx.x % groups;
    const int lo = g.bounds[b], m = g.bounds[b + 1] - lo, mp = (m + 15) & ~15;
    const double* F = g.fac + i64(b) * g.bmax * g.bmax;
    const int tid = threadIdx.x;
    ts_load_factor(Ls, F, g.bmax, m, mp);  // once for all of this CTA's column tiles
    const int ct_end = min(g.ctiles, (grp + 1) * g.cpt);
    for (int ct = grp * g.cpt; ct < ct_end; ++ct) {
    const int c0 = ct * TS_NC, nc = min(TS_NC, g.w - c0);
    for (int e = tid; e < mp * TS_NC; e += int(blockDim.x)) {
        const int r = e % mp, c = e / mp;
        double* d = Ys + r * TS_YLD + c;
        if (r < m && c < nc)
            tile::cp_async8(d, g.Y + (lo + r) + i64(c0 + c) * g.ldy, true);
        else
            *d = 0.0;
    }
    tile::cp_commit();
    tile::cp_wait<0>();
    __syncthreads();
    // From here on every warp works on its own 8 columns: no block barriers.
    ts_forward_s<S>(Ls, mp, Ys, 0);
    ts_backward_s<S>(Ls, mp, Ys, 0);
    __syncthreads();
    for (int e = tid; e < m * nc; e += int(blockDim.x)) {
        const int r = e % m, c = e / m;
        g.Y[(lo + r) + i64(c0 + c) * g.ldy] = Ys[r * TS_YLD + c];
    }
    __syncthreads();
    }
}

// ------------------------------------------------------------------------
// Leaves of 129..256 rows: 2 x 2 blocks of at most 128 rows,
//   L = [L11 0; L21 L22]:  forward  x1 = L11^-1 b1, b2 -= L21 x1, x2 = L22^-1 b2
//                          backward x2 = L22^-T y2, y1 -= L21^T x2, x1 = L11^-T y1
// with the packed 128-row machinery above for the diagonal blocks (one of
// them resident at a time) and the couplings as DMMA products against L21
// streamed through shared memory in 16-column panels (double-buffered).
constexpr int TS2_MAX = 256, TS2_CLD = 128 + 4;
constexpr size_t TS2_SMEM = (size_t(TS2_MAX) * TS_YLD + TS_LSIZE + 2 * 16 * TS2_CLD) * sizeof(double);

/// Thread-cooperative cp.async of a 16 x 128 coupling panel into Cb (ld TS2_CLD):
/// TRANS = false: Cb[k][r] = L21[r, 16 pk + k]  (forward, rows r < m2)
/// TRANS = true:  Cb[k][i] = L21[16 pk + k, i]  (backward, k < m2 - 16 pk)
template <bool TRANS>
__device__ __forceinline__ void ts2_panel(double* Cb, const double* F, int ldf, int m2, int pk) {
    for (int e = threadIdx.x; e < 16 * 128; e += TS_THREADS) {
        const int k = TRANS ? (e & 15) : (e >> 7), r = TRANS ? (e >> 4) : (e & 127);
        double* d = Cb + k * TS2_CLD + r;
        const int gr = TRANS ? 128 + 16 * pk + k : 128 + r, gc = TRANS ? r : 16 * pk + k;
        const bool v = TRANS ? (16 * pk + k < m2) : (r < m2);
        if (v)
            tile::cp_async8(d, F + gr + i64(gc) * ldf, true);
        else
            *d = 0.0;
    }
}

/// acc[t] (rows 8t + g8 of the target half) += A_panel x (16 rows of the source half).
__device__ __forceinline__ void ts2_couple(const double* Cb, const double* Xs, double (&acc)[16][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g8 = lane >> 2, t4 = lane & 3, n0 = warp * 8;
    double xb[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) xb[kk] = Xs[(4 * kk + t4) * TS_YLD + n0 + g8];
#pragma unroll
    for (int t = 0; t < 16; ++t)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) tile::dmma(acc[t], Cb[(4 * kk + t4) * TS2_CLD + 8 * t + g8], xb[kk]);
}

/// Y[row0 + 8t + g8, n0 + 2t4 + e] -= acc (this warp's columns)
__device__ __forceinline__ void ts2_sub(double* Ys, int row0, int rows, const double (&acc)[16][2]) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g8 = lane >> 2, t4 = lane & 3, n0 = warp * 8;
#pragma unroll
    for (int t = 0; t < 16; ++t)
        if (8 * t + g8 < rows) {
            double* y = Ys + (row0 + 8 * t + g8) * TS_YLD + n0 + 2 * t4;
            y[0] -= acc[t][0];
            y[1] -= acc[t][1];
        }
}

template <bool TRANS>
__device__ __forceinline__ void ts2_coupling(double* Cb, const double* F, int ldf, int m2, double* Ys, int src0,
                                             int dst0, int dst_rows) {
    double acc[16][2];
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t][0] = acc[t][1] = 0.0;
    const int npk = TRANS ? (m2 + 15) / 16 : 8;
    ts2_panel<TRANS>(Cb, F, ldf, m2, 0);
    tile::cp_commit();
    for (int pk = 0; pk < npk; ++pk) {
        double* cur = Cb + (pk & 1) * 16 * TS2_CLD;
        if (pk + 1 < npk) ts2_panel<TRANS>(Cb + ((pk + 1) & 1) * 16 * TS2_CLD, F, ldf, m2, pk + 1);
        tile::cp_commit();
        tile::cp_wait<1>();
        __syncthreads();
        ts2_couple(cur, Ys + (src0 + 16 * pk) * TS_YLD, acc);
        __syncthreads();
    }
    tile::cp_wait<0>();
    ts2_sub(Ys, dst0, dst_rows, acc);
    __syncthreads();
}

__global__ void __launch_bounds__(TS_THREADS, 1) k_leaf_solve_tc2(LeafSolveTcArgs g) {
    extern __shared__ double sm[];
    double* Ys = sm;
    double* Ls = Ys + TS2_MAX * TS_YLD;
    double* Cb = Ls + TS_LSIZE;
    const int groups = (g.ctiles + g.cpt - 1) / g.cpt;
    const int b = blockIdx.x / groups, grp = blockIdx.x % groups;
    const int lo = g.bounds[b], m = g.bounds[b + 1] - lo;
    const int m1 = min(m, 128), m2 = max(m - 128, 0);
    const int mp1 = (m1 + 15) & ~15, mp2 = (m2 + 15) & ~15;
    const double* F = g.fac + i64(b) * g.bmax * g.bmax;
    const double* F22 = F + 128 + i64(128) * g.bmax;
    const int tid = threadIdx.x;
    const int ct_end = min(g.ctiles, (grp + 1) * g.cpt);
    for (int ct = grp * g.cpt; ct < ct_end; ++ct) {
        const int c0 = ct * TS_NC, nc = min(TS_NC, g.w - c0);
        for (int e = tid; e < (mp1 + mp2) * TS_NC; e += TS_THREADS) {
            const int c = e / (mp1 + mp2), r = e - c * (mp1 + mp2);
            const int gr = r < mp1 ? r : 128 + (r - mp1);  // tile rows: [0, mp1) top, then the bottom half at 128
            double* d = Ys + (r < mp1 ? r : 128 + (r - mp1)) * TS_YLD + c;
            if (gr < m && c < nc && (r < mp1 ? r < m1 : true))
                tile::cp_async8(d, g.Y + (lo + gr) + i64(c0 + c) * g.ldy, true);
            else
                *d = 0.0;
        }
        ts_load_factor(Ls, F, g.bmax, m1, mp1);
        tile::cp_commit();
        tile::cp_wait<0>();
        __syncthreads();
        ts_forward(Ls, mp1, Ys, 0);
        __syncthreads();
        if (m2 > 0) {
            ts2_coupling<false>(Cb, F, g.bmax, m2, Ys, 0, 128, m2);  // b2 -= L21 x1
            ts_load_factor(Ls, F22, g.bmax, m2, mp2);
            tile::cp_commit();
            tile::cp_wait<0>();
            __syncthreads();
            ts_forward(Ls, mp2, Ys, 128);
            ts_backward(Ls, mp2, Ys, 128);
            __syncthreads();
            ts2_coupling<true>(Cb, F, g.bmax, m2, Ys, 128, 0, 128);  // y1 -= L21^T x2
            ts_load_factor(Ls, F, g.bmax, m1, mp1);
            tile::cp_commit();
            tile::cp_wait<0>();
            __syncthreads();
        }
        ts_backward(Ls, mp1, Ys, 0);
        __syncthreads();
        for (int e = tid; e < m * nc; e += TS_THREADS) {
            const int c = e / m, r = e - c * m;
            g.Y[(lo + r) + i64(c0 + c) * g.ldy] = Ys[r * TS_YLD + c];
        }
        __syncthreads();
    }
}
