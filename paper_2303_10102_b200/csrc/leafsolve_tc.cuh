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
__global__ void __launch_bounds__(128) k_leaf_diag_inv(const int* bounds, int bmax, double* fac) {
    __shared__ double Ls[8][16][17];
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
        for (int e = threadIdx.x; e < rows * 16; e += TS_THREADS) {
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

__global__ void __launch_bounds__(TS_THREADS, 2) k_leaf_solve_tc(LeafSolveTcArgs g) {
    extern __shared__ double sm[];
    double* Ys = sm;
    double* Ls = sm + TS_MAX * TS_YLD;
    const int groups = (g.ctiles + g.cpt - 1) / g.cpt;
    const int b = blockIdx.x / groups, grp = blockIdx.x % groups;
    const int lo = g.bounds[b], m = g.bounds[b + 1] - lo, mp = (m + 15) & ~15, nb = mp / 16;
    const double* F = g.fac + i64(b) * g.bmax * g.bmax;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g8 = lane >> 2, t4 = lane & 3, n0 = warp * 8;
    ts_load_factor(Ls, F, g.bmax, m, mp);  // once for all of this CTA's column tiles
    const int ct_end = min(g.ctiles, (grp + 1) * g.cpt);
    for (int ct = grp * g.cpt; ct < ct_end; ++ct) {
    const int c0 = ct * TS_NC, nc = min(TS_NC, g.w - c0);
    for (int e = tid; e < mp * TS_NC; e += TS_THREADS) {
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
    // ---- forward: L x = b
    for (int j = 0; j < nb; ++j) {
        const double* P = Ls + ts_poff(j, mp);
        const int ld = mp - 16 * j + 4;
        double* Yj = Ys + 16 * j * TS_YLD + n0;
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
    // ---- backward: L^T x = y
    for (int j = nb - 1; j >= 0; --j) {
        const double* P = Ls + ts_poff(j, mp);
        const int ld = mp - 16 * j + 4;
        double* Yj = Ys + 16 * j * TS_YLD + n0;
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
    __syncthreads();
    for (int e = tid; e < m * nc; e += TS_THREADS) {
        const int r = e % m, c = e / m;
        g.Y[(lo + r) + i64(c0 + c) * g.ldy] = Ys[r * TS_YLD + c];
    }
    __syncthreads();
    }
}
