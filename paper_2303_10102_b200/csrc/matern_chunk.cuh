// Matérn 1D apply in O(n s) with chunked moments (included by oracle.cu inside
// its anonymous namespace, after Poly / poly_eval).
//
// k(d) = exp(-lambda d) sum_m c_m d^m (m < nt <= 4) on sorted points. Rows are
// cut into chunks of 32 (one warp). For row i in chunk c:
//   Y_i = sum_{j in c} k(|x_i - x_j|) V_j                       (dense, exact)
//       + sum_q Gf_iq F_q(c) + sum_q Gb_iq B_q(c) + nugget V_i
// with the forward state F_q(c) = sum_{j < c} (r_c - x_j)^q e^{-lambda(r_c - x_j)} V_j
// at r_c = first point of c, the backward state B_q(c) = sum_{j > c}
// (x_j - r'_c)^q e^{-lambda(x_j - r'_c)} V_j at r'_c = last point of c, and
//   Gf_iq = e^{-lambda(x_i - r_c)}  sum_{m>=q} c_m C(m,q) (x_i - r_c)^{m-q},
//   Gb_iq = e^{-lambda(r'_c - x_i)} sum_{m>=q} c_m C(m,q) (r'_c - x_i)^{m-q}
// (binomial split of d^m at the reference point; every exponential decays,
// so nothing overflows). States move between reference points with
//   T(D) v: w_q = e^{-lambda D} sum_{p<=q} C(q,p) D^{q-p} v_p,
// and T(D2) T(D1) = T(D1 + D2), so a run of chunks composes to one transfer.
//   k_mat_moments: per chunk, the moments of its own rows at the next chunk's
//                  first point (forward) / the previous chunk's last point;
//   k_mat_carry:   per column and direction, a block-wide scan of the chunk
//                  moments -> F(c), B(c) for every chunk;
//   k_mat_apply:   the 32x32 in-chunk kernel block (exact pair evaluation)
//                  plus the two carried states, one pass over V and Y.
// V is read twice and Y written once; every kernel value and transfer is
// evaluated in FP64 from x. Same recurrence as the oracle's scan
// (oracle/hodlr.cpp), regrouped by chunk.

constexpr int MC_ROWS = 32;   // chunk
constexpr int MC_TILE = 256;  // rows per CTA (8 chunks)
constexpr int MC_COLS = 32;   // columns per CTA
constexpr int MC_LD = MC_COLS + 1;
constexpr int MC_CARRY_THREADS = 1024;
constexpr size_t MC_SMEM_APPLY = size_t(MC_TILE) * MC_LD * sizeof(double);
constexpr size_t MC_SMEM_MOMENTS = (size_t(MC_TILE) * MC_LD + 8 * MC_TILE) * sizeof(double);

struct MatChunkArgs {
    const double* x;
    int n, nch, s, nt;
    double lambda;
    double c[4];
    double nugget;  // added on the diagonal (value oracle only)
    const double* V;
    i64 ldv;
    double* Y;
    i64 ldy;
    double* Lf;  // [col][chunk][4] local forward moments
    double* Lb;  // [col][chunk][4] local backward moments
    double* Ff;  // [col][chunk][4] F(c)
    double* Fb;  // [col][chunk][4] B(c)
};

__device__ __forceinline__ double mc_first(const MatChunkArgs& g, int c) { return g.x[c * MC_ROWS]; }
__device__ __forceinline__ double mc_last(const MatChunkArgs& g, int c) {
    return g.x[min(g.n, (c + 1) * MC_ROWS) - 1];
}

/// v <- T(D) v
__device__ __forceinline__ void mc_transfer(double (&v)[4], double D, double lambda) {
    const double e = exp(-lambda * D), D2 = D * D;
    const double w3 = v[3] + 3.0 * D * v[2] + 3.0 * D2 * v[1] + D2 * D * v[0];
    const double w2 = v[2] + 2.0 * D * v[1] + D2 * v[0];
    const double w1 = v[1] + D * v[0];
    v[0] *= e;
    v[1] = e * w1;
    v[2] = e * w2;
    v[3] = e * w3;
}

/// Stage V[r0 : r0+256, c0 : c0+32] (zero padded) into shared memory.
__device__ __forceinline__ void mc_stage(const MatChunkArgs& g, double* Vs, int r0, int c0) {
    for (int e = threadIdx.x; e < MC_TILE * MC_COLS; e += blockDim.x) {
        const int r = e % MC_TILE, cc = e / MC_TILE;
        const int row = r0 + r, col = c0 + cc;
        Vs[r * MC_LD + cc] = (row < g.n && col < g.s) ? g.V[i64(row) + i64(col) * g.ldv] : 0.0;
    }
}

__global__ void __launch_bounds__(MC_TILE) k_mat_moments(MatChunkArgs g) {
    extern __shared__ double sm[];
    double* Vs = sm;                    // 256 x 33
    double* wf = Vs + MC_TILE * MC_LD;  // 256 x 4 forward weights
    double* wb = wf + MC_TILE * 4;      // 256 x 4 backward weights
    const int r0 = blockIdx.x * MC_TILE, c0 = blockIdx.y * MC_COLS;
    mc_stage(g, Vs, r0, c0);
    {  // per-row weights (row = thread)
        const int row = r0 + threadIdx.x, c = row / MC_ROWS;
        double f[4] = {0, 0, 0, 0}, b[4] = {0, 0, 0, 0};
        if (row < g.n) {
            if (c + 1 < g.nch) {
                const double d = mc_first(g, c + 1) - g.x[row], e = exp(-g.lambda * d);
                f[0] = e;
                f[1] = e * d;
                f[2] = e * d * d;
                f[3] = e * d * d * d;
            }
            if (c > 0) {
                const double d = g.x[row] - mc_last(g, c - 1), e = exp(-g.lambda * d);
                b[0] = e;
                b[1] = e * d;
                b[2] = e * d * d;
                b[3] = e * d * d * d;
            }
        }
        for (int q = 0; q < 4; ++q) {
            wf[threadIdx.x * 4 + q] = f[q];
            wb[threadIdx.x * 4 + q] = b[q];
        }
    }
    __syncthreads();
    const int cl = threadIdx.x >> 5, lane = threadIdx.x & 31;  // warp = chunk, lane = column
    const int c = blockIdx.x * (MC_TILE / MC_ROWS) + cl, col = c0 + lane;
    if (c >= g.nch || col >= g.s) return;
    double f[4] = {0, 0, 0, 0}, b[4] = {0, 0, 0, 0};
    for (int j = 0; j < MC_ROWS; ++j) {
        const int r = cl * MC_ROWS + j;
        const double v = Vs[r * MC_LD + lane];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            f[q] = fma(wf[r * 4 + q], v, f[q]);
            b[q] = fma(wb[r * 4 + q], v, b[q]);
        }
    }
    double* of = g.Lf + (i64(col) * g.nch + c) * 4;
    double* ob = g.Lb + (i64(col) * g.nch + c) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        of[q] = f[q];
        ob[q] = b[q];
    }
}

/// One CTA per (column, direction). Step st of the scan consumes chunk
/// consumed(st)'s local moments and lands on the reference point of chunk
/// landed(st): forward F(c+1) = T(r_{c+1} - r_c) F(c) + L(c), F(0) = 0;
/// backward B(c-1) = T(r'_c - r'_{c-1}) B(c) + L'(c), B(nch-1) = 0. Each
/// thread owns a contiguous run of steps; runs are combined by a
/// Kogge-Stone scan of (state at the run's landing point).
__global__ void __launch_bounds__(MC_CARRY_THREADS) k_mat_carry(MatChunkArgs g) {
    __shared__ double sv[MC_CARRY_THREADS][4];
    __shared__ double sp[MC_CARRY_THREADS];
    const int col = blockIdx.x, dir = blockIdx.y, t = threadIdx.x;
    const int nsteps = g.nch - 1;
    const int per = max(1, (nsteps + MC_CARRY_THREADS - 1) / MC_CARRY_THREADS);
    const int s0 = min(nsteps, t * per), s1 = min(nsteps, s0 + per);
    const bool has = s1 > s0;
    const double* L = (dir == 0 ? g.Lf : g.Lb) + i64(col) * g.nch * 4;
    double* O = (dir == 0 ? g.Ff : g.Fb) + i64(col) * g.nch * 4;
    auto consumed = [&](int st) { return dir == 0 ? st : g.nch - 1 - st; };
    auto landed = [&](int st) { return dir == 0 ? st + 1 : g.nch - 2 - st; };
    auto landpos = [&](int st) { return dir == 0 ? mc_first(g, st + 1) : mc_last(g, g.nch - 2 - st); };
    auto dist = [&](double from, double to) { return dir == 0 ? to - from : from - to; };
    double v[4] = {0, 0, 0, 0}, pos = 0.0;
    for (int st = s0; st < s1; ++st) {
        const double np = landpos(st);
        if (st > s0) mc_transfer(v, dist(pos, np), g.lambda);
        const double* l = L + i64(consumed(st)) * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] += l[q];
        pos = np;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) sv[t][q] = v[q];
    sp[t] = pos;
    __syncthreads();
    for (int off = 1; off < MC_CARRY_THREADS; off <<= 1) {
        double a[4] = {0, 0, 0, 0};
        const int u = t - off;
        const bool take = has && u >= 0;  // runs before a non-empty run are non-empty
        if (take) {
#pragma unroll
            for (int q = 0; q < 4; ++q) a[q] = sv[u][q];
            mc_transfer(a, dist(sp[u], sp[t]), g.lambda);
        }
        __syncthreads();
        if (take)
#pragma unroll
            for (int q = 0; q < 4; ++q) sv[t][q] += a[q];
        __syncthreads();
    }
    if (t == 0) {  // the first chunk in scan order has no incoming state
        double* o = O + i64(dir == 0 ? 0 : g.nch - 1) * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) o[q] = 0.0;
    }
    if (!has) return;
    double w[4] = {0, 0, 0, 0}, wpos = 0.0;
    bool hw = false;
    if (t > 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = sv[t - 1][q];
        wpos = sp[t - 1];
        hw = true;
    }
    for (int st = s0; st < s1; ++st) {
        const double np = landpos(st);
        if (hw) mc_transfer(w, dist(wpos, np), g.lambda);
        const double* l = L + i64(consumed(st)) * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] += l[q];
        wpos = np;
        hw = true;
        double* o = O + i64(landed(st)) * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) o[q] = w[q];
    }
}

__global__ void __launch_bounds__(MC_TILE) k_mat_apply(MatChunkArgs g) {
    extern __shared__ double sm[];
    double* Vs = sm;
    const int r0 = blockIdx.x * MC_TILE, c0 = blockIdx.y * MC_COLS;
    mc_stage(g, Vs, r0, c0);
    __syncthreads();
    const int i = r0 + threadIdx.x, cl = threadIdx.x >> 5;
    if (i >= g.n) return;
    const int c = i / MC_ROWS, jb = c * MC_ROWS;
    const double xi = g.x[i];
    double kv[MC_ROWS];
#pragma unroll
    for (int j = 0; j < MC_ROWS; ++j) {
        const int rj = jb + j;
        double k = 0.0;
        if (rj < g.n) {
            const double d = fabs(xi - g.x[rj]);
            double p = 0.0, dm = 1.0;
            for (int m = 0; m < g.nt; ++m) {
                p = fma(g.c[m], dm, p);
                dm *= d;
            }
            k = p * exp(-g.lambda * d);
        }
        kv[j] = k;
    }
    // Gf_q, Gb_q
    double gf[4] = {0, 0, 0, 0}, gb[4] = {0, 0, 0, 0};
    {
        const double df = xi - mc_first(g, c), db = mc_last(g, c) - xi;
        const double ef = exp(-g.lambda * df), eb = exp(-g.lambda * db);
        const double binom[4][4] = {{1, 0, 0, 0}, {1, 1, 0, 0}, {1, 2, 1, 0}, {1, 3, 3, 1}};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            double sf = 0.0, sb = 0.0;
#pragma unroll
            for (int m = q; m < 4; ++m) {
                if (m < g.nt) {
                    double pf = 1.0, pb = 1.0;
                    for (int e = 0; e < m - q; ++e) {
                        pf *= df;
                        pb *= db;
                    }
                    sf += g.c[m] * binom[m][q] * pf;
                    sb += g.c[m] * binom[m][q] * pb;
                }
            }
            gf[q] = ef * sf;
            gb[q] = eb * sb;
        }
    }
    for (int cc = 0; cc < MC_COLS; ++cc) {
        const int col = c0 + cc;
        if (col >= g.s) break;
        double acc = g.nugget * Vs[threadIdx.x * MC_LD + cc];
#pragma unroll
        for (int j = 0; j < MC_ROWS; ++j) acc = fma(kv[j], Vs[(cl * MC_ROWS + j) * MC_LD + cc], acc);
        const double* F = g.Ff + (i64(col) * g.nch + c) * 4;
        const double* B = g.Fb + (i64(col) * g.nch + c) * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) acc = fma(gf[q], F[q], fma(gb[q], B[q], acc));
        g.Y[i64(i) + i64(col) * g.ldy] = acc;
    }
}
