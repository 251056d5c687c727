// Matérn 1D apply in O(n s) with chunked moments (included by oracle.cu inside
// its anonymous namespace, after Poly / poly_eval).
//
// k(d) = exp(-lambda d) sum_m c_m d^m (m < nt <= 4) on sorted points. Rows are
// cut into chunks of 32 (one warp) and super-chunks of 256 (one CTA). For
// row i in chunk c:
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
// and T(D2) T(D1) = T(D1 + D2), so any run of chunks composes to one transfer.
//   k_mat_moments: per super-chunk, the moments of its rows at the next
//                  super-chunk's first point (forward) / the previous one's
//                  last point (backward);
//   k_mat_carry:   per column and direction, a block-wide scan over the
//                  super-chunks -> states at every super-chunk boundary;
//   k_mat_apply:   per super-chunk: chunk moments again (V is staged anyway),
//                  chunk states from the super-chunk carry-in, then the 32x32
//                  in-chunk kernel block (exact pair evaluation) plus the two
//                  carried states, one pass over V and Y.
// V is read twice and Y written once; every kernel value and transfer is
// evaluated in FP64 from x. Same recurrence as the oracle's scan
// (oracle/hodlr.cpp), regrouped by chunk.

constexpr int MC_ROWS = 32;                       // chunk
constexpr int MC_TILE = 256;                      // rows per CTA = super-chunk (8 chunks)
constexpr int MC_NCH = MC_TILE / MC_ROWS;         // chunks per super-chunk
constexpr int MC_COLS = 32;                       // columns per CTA
constexpr int MC_LD = MC_COLS + 2;                // even: 16-byte column-pair loads
constexpr int MC_CARRY_THREADS = 1024;
// Vs + per-chunk moments / states (8 chunks x 32 columns x 4, forward and backward)
constexpr size_t MC_SMEM = (size_t(MC_TILE) * MC_LD + 2 * MC_NCH * MC_COLS * 4 + 8 * MC_TILE + 8 * MC_NCH) *
                           sizeof(double);

struct MatChunkArgs {
    const double* x;
    int n, nsup, s, nt;
    double lambda;
    double c[4];
    double nugget;  // added on the diagonal (value oracle only)
    const double* V;
    i64 ldv;
    double* Y;
    i64 ldy;
    double* Lf;  // [col][super][4] super-chunk forward moments
    double* Lb;  // [col][super][4] super-chunk backward moments
    double* Ff;  // [col][super][4] forward state at the super-chunk's first point
    double* Fb;  // [col][super][4] backward state at the super-chunk's last point
    // ZeroRows hint (peeling): V is zero on the segments of parity zpar of the
    // partition zb; with zout the caller reads Y only on those segments.
    const int* zb;
    int znseg, zpar, zout;
};

/// Parity of the single segment of zb holding rows [a, b), or -1 when the
/// run straddles a boundary (or no hint is given).
__device__ __forceinline__ int mc_run_parity(const MatChunkArgs& g, int a, int b) {
    if (!g.zb) return -1;
    auto seg = [&](int r) {
        int lo = 0, hi = g.znseg - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (g.zb[mid] <= r) lo = mid; else hi = mid - 1;
        }
        return lo;
    };
    const int s0 = seg(a), s1 = seg(b - 1);
    return s0 == s1 ? (s0 & 1) : -1;
}

__device__ __forceinline__ double mc_first(const MatChunkArgs& g, int row0) { return g.x[row0]; }
__device__ __forceinline__ double mc_last(const MatChunkArgs& g, int row_end) { return g.x[min(g.n, row_end) - 1]; }

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

/// v <- T(D) v with e = exp(-lambda D) precomputed.
__device__ __forceinline__ void mc_transfer_e(double (&v)[4], double D, double e) {
    const double D2 = D * D;
    const double w3 = v[3] + 3.0 * D * v[2] + 3.0 * D2 * v[1] + D2 * D * v[0];
    const double w2 = v[2] + 2.0 * D * v[1] + D2 * v[0];
    const double w1 = v[1] + D * v[0];
    v[0] *= e;
    v[1] = e * w1;
    v[2] = e * w2;
    v[3] = e * w3;
}

/// Per-CTA tables computed once (row = thread): moment weights of each row
/// at its chunk's forward / backward reference points, and the chunk-to-chunk
/// transfers inside the super-chunk plus the super-chunk boundary transfers.
struct McTables {
    double* wf;  // 256 x 4: (r_{c+1} - x_j)^q e^{-lambda(r_{c+1} - x_j)}
    double* wb;  // 256 x 4: (x_j - r'_{c-1})^q e^{-lambda(x_j - r'_{c-1})}
    double* tf;  // 8 x 2: chunk cl -> cl+1 forward (D, e); [cl] for the super summary: (R - r_{cl+1}, e)
    double* tb;  // 8 x 2 backward
    double* sf;  // 8 x 2: super summary forward transfer of chunk cl's moment
    double* sb;  // 8 x 2
};

__device__ __forceinline__ McTables mc_tables(double* base) {
    McTables t;
    t.wf = base;
    t.wb = t.wf + MC_TILE * 4;
    t.tf = t.wb + MC_TILE * 4;
    t.tb = t.tf + 2 * MC_NCH;
    t.sf = t.tb + 2 * MC_NCH;
    t.sb = t.sf + 2 * MC_NCH;
    return t;
}
constexpr int MC_TABLE_DOUBLES = 8 * MC_TILE + 8 * MC_NCH;

__device__ __forceinline__ void mc_fill_tables(const MatChunkArgs& g, int r0, const McTables& T) {
    const int row = r0 + threadIdx.x, lo = (row / MC_ROWS) * MC_ROWS;
    double f[4] = {0, 0, 0, 0}, b[4] = {0, 0, 0, 0};
    if (row < g.n) {
        const double xj = g.x[row];
        if (lo + MC_ROWS < g.n) {
            const double d = g.x[lo + MC_ROWS] - xj, e = exp(-g.lambda * d);
            f[0] = e;
            f[1] = e * d;
            f[2] = e * d * d;
            f[3] = e * d * d * d;
        }
        if (lo > 0) {
            const double d = xj - g.x[lo - 1], e = exp(-g.lambda * d);
            b[0] = e;
            b[1] = e * d;
            b[2] = e * d * d;
            b[3] = e * d * d * d;
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        T.wf[threadIdx.x * 4 + q] = f[q];
        T.wb[threadIdx.x * 4 + q] = b[q];
    }
    if (threadIdx.x < MC_NCH) {
        const int cl = threadIdx.x, c0 = r0 + cl * MC_ROWS;
        double D = 0.0;
        if (c0 + MC_ROWS < g.n) D = g.x[c0 + MC_ROWS] - g.x[c0];  // r_cl -> r_{cl+1}
        T.tf[2 * cl] = D;
        T.tf[2 * cl + 1] = exp(-g.lambda * D);
        D = 0.0;
        if (c0 > 0 && c0 < g.n) D = g.x[min(g.n, c0 + MC_ROWS) - 1] - g.x[c0 - 1];  // r'_cl -> r'_{cl-1}
        T.tb[2 * cl] = D;
        T.tb[2 * cl + 1] = exp(-g.lambda * D);
        D = 0.0;  // super summary: chunk cl's forward moment (at r_{cl+1}) -> next super's first point
        if (r0 + MC_TILE < g.n && c0 + MC_ROWS < g.n) D = g.x[r0 + MC_TILE] - g.x[c0 + MC_ROWS];
        T.sf[2 * cl] = D;
        T.sf[2 * cl + 1] = exp(-g.lambda * D);
        D = 0.0;  // chunk cl's backward moment (at r'_{cl-1}) -> previous super's last point
        if (r0 > 0 && c0 < g.n) D = g.x[c0 - 1] - g.x[r0 - 1];
        T.sb[2 * cl] = D;
        T.sb[2 * cl + 1] = exp(-g.lambda * D);
    }
}

/// Chunk moments of the CTA's 8 chunks (warp = chunk, lane = column).
__device__ __forceinline__ void mc_chunk_moments(const double* Vs, const McTables& T, double* Mf, double* Mb) {
    const int cl = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double f[4] = {0, 0, 0, 0}, b[4] = {0, 0, 0, 0};
#pragma unroll 4
    for (int j = 0; j < MC_ROWS; ++j) {
        const int r = cl * MC_ROWS + j;
        const double v = Vs[r * MC_LD + lane];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            f[q] = fma(T.wf[r * 4 + q], v, f[q]);
            b[q] = fma(T.wb[r * 4 + q], v, b[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        Mf[(cl * MC_COLS + lane) * 4 + q] = f[q];
        Mb[(cl * MC_COLS + lane) * 4 + q] = b[q];
    }
}

__global__ void __launch_bounds__(MC_TILE) k_mat_moments(MatChunkArgs g) {
    extern __shared__ double sm[];
    double* Vs = sm;
    double* Mf = Vs + MC_TILE * MC_LD;
    double* Mb = Mf + MC_NCH * MC_COLS * 4;
    const McTables T = mc_tables(Mb + MC_NCH * MC_COLS * 4);
    const int S = blockIdx.x, r0 = S * MC_TILE;
    const int nchk = min(MC_NCH, (g.n - r0 + MC_ROWS - 1) / MC_ROWS);
    if (mc_run_parity(g, r0, min(g.n, r0 + MC_TILE)) == g.zpar) {  // V == 0 here: zero moments
        for (int col = threadIdx.x; col < g.s; col += blockDim.x)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                g.Lf[(i64(col) * g.nsup + S) * 4 + q] = 0.0;
                g.Lb[(i64(col) * g.nsup + S) * 4 + q] = 0.0;
            }
        return;
    }
    mc_fill_tables(g, r0, T);
    for (int c0 = 0; c0 < g.s; c0 += MC_COLS) {
        mc_stage(g, Vs, r0, c0);
        __syncthreads();
        mc_chunk_moments(Vs, T, Mf, Mb);
        __syncthreads();
        const int col = c0 + threadIdx.x;
        if (threadIdx.x < MC_COLS && col < g.s) {
            double f[4] = {0, 0, 0, 0}, b[4] = {0, 0, 0, 0};
            for (int cl = 0; cl < nchk; ++cl) {
                double v[4], w[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    v[q] = Mf[(cl * MC_COLS + threadIdx.x) * 4 + q];
                    w[q] = Mb[(cl * MC_COLS + threadIdx.x) * 4 + q];
                }
                mc_transfer_e(v, T.sf[2 * cl], T.sf[2 * cl + 1]);
                mc_transfer_e(w, T.sb[2 * cl], T.sb[2 * cl + 1]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    f[q] += v[q];
                    b[q] += w[q];
                }
            }
            if (r0 + MC_TILE >= g.n) f[0] = f[1] = f[2] = f[3] = 0.0;
            if (r0 == 0) b[0] = b[1] = b[2] = b[3] = 0.0;
            double* of = g.Lf + (i64(col) * g.nsup + S) * 4;
            double* ob = g.Lb + (i64(col) * g.nsup + S) * 4;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                of[q] = f[q];
                ob[q] = b[q];
            }
        }
        __syncthreads();
    }
}

/// One CTA per (column, direction). Step st of the scan consumes super-chunk
/// consumed(st)'s moments and lands on the reference point of super-chunk
/// landed(st) (forward: its first point; backward: its last point). Each
/// thread owns a contiguous run of steps; runs are combined by a Kogge-Stone
/// scan of (state at the run's landing point).
__global__ void __launch_bounds__(MC_CARRY_THREADS) k_mat_carry(MatChunkArgs g) {
    __shared__ double sv[MC_CARRY_THREADS][4];
    __shared__ double sp[MC_CARRY_THREADS];
    const int col = blockIdx.x, dir = blockIdx.y, t = threadIdx.x;
    const int ns = g.nsup, nsteps = ns - 1;
    const int per = max(1, (nsteps + MC_CARRY_THREADS - 1) / MC_CARRY_THREADS);
    const int s0 = min(nsteps, t * per), s1 = min(nsteps, s0 + per);
    const bool has = s1 > s0;
    const double* L = (dir == 0 ? g.Lf : g.Lb) + i64(col) * ns * 4;
    double* O = (dir == 0 ? g.Ff : g.Fb) + i64(col) * ns * 4;
    auto consumed = [&](int st) { return dir == 0 ? st : ns - 1 - st; };
    auto landed = [&](int st) { return dir == 0 ? st + 1 : ns - 2 - st; };
    auto landpos = [&](int st) {
        return dir == 0 ? g.x[(st + 1) * MC_TILE] : g.x[min(g.n, (ns - 1 - st) * MC_TILE) - 1];
    };
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
        const bool take = has && u >= 0;  // every run before a non-empty run is non-empty
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
    if (t == 0) {  // the first super-chunk in scan order has no incoming state
        double* o = O + i64(dir == 0 ? 0 : ns - 1) * 4;
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
    double* Mf = Vs + MC_TILE * MC_LD;       // chunk moments, then chunk states F(c)
    double* Mb = Mf + MC_NCH * MC_COLS * 4;  // chunk moments, then chunk states B(c)
    const McTables T = mc_tables(Mb + MC_NCH * MC_COLS * 4);
    const int S = blockIdx.x, r0 = S * MC_TILE;
    const int nchk = min(MC_NCH, (g.n - r0 + MC_ROWS - 1) / MC_ROWS);
    if (g.zout) {  // rows the caller never reads
        const int par = mc_run_parity(g, r0, min(g.n, r0 + MC_TILE));
        if (par >= 0 && par != g.zpar) return;
    }
    mc_fill_tables(g, r0, T);
    // per-row kernel values of the own chunk and the state coefficients (once)
    const int i = r0 + threadIdx.x, cl = threadIdx.x >> 5;
    const bool live = i < g.n;
    const int jb = r0 + cl * MC_ROWS;
    double kv[MC_ROWS];
    double gf[4] = {0, 0, 0, 0}, gb[4] = {0, 0, 0, 0};
    if (live) {
        const double xi = g.x[i];
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
        const double df = xi - g.x[jb], db = mc_last(g, jb + MC_ROWS) - xi;
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
    for (int c0 = 0; c0 < g.s; c0 += MC_COLS) {
        mc_stage(g, Vs, r0, c0);
        __syncthreads();
        mc_chunk_moments(Vs, T, Mf, Mb);
        __syncthreads();
        if (threadIdx.x < MC_COLS) {  // chunk states from the super-chunk carries (lane = column)
            const int col = c0 + threadIdx.x;
            double f[4] = {0, 0, 0, 0}, b[4] = {0, 0, 0, 0};
            if (col < g.s) {
                const double* F = g.Ff + (i64(col) * g.nsup + S) * 4;
                const double* B = g.Fb + (i64(col) * g.nsup + S) * 4;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    f[q] = F[q];
                    b[q] = B[q];
                }
            }
            double* mf = Mf + threadIdx.x * 4;
            for (int c = 0; c < nchk; ++c) {  // F(c+1) = T(r_{c+1} - r_c) F(c) + Lf(c)
                double l[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    l[q] = mf[c * MC_COLS * 4 + q];
                    mf[c * MC_COLS * 4 + q] = f[q];
                }
                mc_transfer_e(f, T.tf[2 * c], T.tf[2 * c + 1]);
#pragma unroll
                for (int q = 0; q < 4; ++q) f[q] += l[q];
            }
            double* mb = Mb + threadIdx.x * 4;
            for (int c = nchk - 1; c >= 0; --c) {  // B(c-1) = T(r'_c - r'_{c-1}) B(c) + Lb(c)
                double l[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    l[q] = mb[c * MC_COLS * 4 + q];
                    mb[c * MC_COLS * 4 + q] = b[q];
                }
                mc_transfer_e(b, T.tb[2 * c], T.tb[2 * c + 1]);
#pragma unroll
                for (int q = 0; q < 4; ++q) b[q] += l[q];
            }
        }
        __syncthreads();
        if (live) {
            const double* Fc = Mf + cl * MC_COLS * 4;
            const double* Bc = Mb + cl * MC_COLS * 4;
            for (int cc = 0; cc < MC_COLS; cc += 2) {
                if (c0 + cc >= g.s) break;
                double a0 = g.nugget * Vs[threadIdx.x * MC_LD + cc];
                double a1 = g.nugget * Vs[threadIdx.x * MC_LD + cc + 1];
#pragma unroll
                for (int j = 0; j < MC_ROWS; ++j) {
                    const double2 v = *reinterpret_cast<const double2*>(Vs + (cl * MC_ROWS + j) * MC_LD + cc);
                    a0 = fma(kv[j], v.x, a0);
                    a1 = fma(kv[j], v.y, a1);
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    a0 = fma(gf[q], Fc[cc * 4 + q], fma(gb[q], Bc[cc * 4 + q], a0));
                    a1 = fma(gf[q], Fc[(cc + 1) * 4 + q], fma(gb[q], Bc[(cc + 1) * 4 + q], a1));
                }
                g.Y[i64(i) + i64(c0 + cc) * g.ldy] = a0;
                if (c0 + cc + 1 < g.s) g.Y[i64(i) + i64(c0 + cc + 1) * g.ldy] = a1;
            }
        }
        __syncthreads();
    }
}
