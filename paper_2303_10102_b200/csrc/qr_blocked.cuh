// Blocked (compact-WY) Householder QR and Q formation for wide blocks
// (included by qr.cu inside its anonymous namespace, after qr_block_sum /
// warp_sum and the QrDesc / QfDesc types).
//
// The SMEM-resident column-at-a-time kernels (k_qr, k_form_q) stop fitting
// once rows x w exceeds shared memory (w >~ 150 at the TSQR chunk height 4w),
// and then ran every Householder step out of global memory. Here a block is
// processed in panels of 16 columns (LAPACK xGEQRF structure):
//   1. the panel (rows x 16) is factored column by column in shared memory;
//   2. T (16 x 16, upper) of the compact WY form H_p ... H_{p+15} = I - V T V^T
//      is built from G = V^T V (xLARFT, forward, columnwise);
//   3. the trailing columns get C <- (I - V T^T V^T) C as two DMMA GEMMs
//      (W = V^T C, then C -= V (T^T W)), C staying in global memory (L2).
// Same Householder vectors, taus and R as the unblocked kernel in exact
// arithmetic; only the association of the trailing-update sums differs.
// Q formation applies the panels right to left: Q <- Q - V (T (V^T Q)).

constexpr int QB_NB = 16;
constexpr int QB_THREADS = 256;
constexpr int QB_MAXROWS = 1400;  // panel (rows x 16) in shared memory
constexpr size_t QB_SMEM_MAX = 220 * 1024;  // panel + the two 16 x w work panels must fit one CTA

__host__ __device__ __forceinline__ int qb_ld(int rows) { return ((rows + 11) / 16) * 16 + 4; }  // 4 mod 16
__host__ __device__ __forceinline__ size_t qb_smem(int rows, int wmax) {
    return (static_cast<size_t>(qb_ld(rows)) * QB_NB + 2 * QB_NB * static_cast<size_t>(wmax) + 2 * QB_NB * QB_NB +
            QB_NB) *
           sizeof(double);
}

struct QbSmem {
    double* P;   // ld x 16 panel, then explicit V
    double* W1;  // 16 x wmax (a + 16 j)
    double* W2;  // 16 x wmax
    double* T;   // 16 x 16 (a + 16 i)
    double* G;   // 16 x 16
    double* tau; // 16
};

__device__ __forceinline__ QbSmem qb_layout(double* sm, int rows, int wmax) {
    QbSmem s;
    s.P = sm;
    s.W1 = s.P + size_t(qb_ld(rows)) * QB_NB;
    s.W2 = s.W1 + size_t(QB_NB) * wmax;
    s.T = s.W2 + size_t(QB_NB) * wmax;
    s.G = s.T + QB_NB * QB_NB;
    s.tau = s.G + QB_NB * QB_NB;
    return s;
}

/// P (nr x jb panel, ld) -> explicit V: zeros above the diagonal, unit
/// diagonal, zero columns past jb and zero rows past nr (to the padded ld).
__device__ __forceinline__ void qb_explicit_v(double* P, int ld, int nr, int jb) {
    for (int e = threadIdx.x; e < ld * QB_NB; e += blockDim.x) {
        const int r = e % ld, i = e / ld;
        if (i >= jb || r >= nr || r < i)
            P[r + i * ld] = 0.0;
        else if (r == i)
            P[r + i * ld] = 1.0;
    }
}

/// G = V^T V (upper part), then T by xLARFT (forward, columnwise).
__device__ __forceinline__ void qb_build_t(const QbSmem& S, int ld, int nr, int jb) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int pr = warp; pr < QB_NB * QB_NB; pr += nwarps) {
        const int a = pr % QB_NB, b = pr / QB_NB;
        if (a > b) continue;
        double s = 0.0;
        if (b < jb)
            for (int r = lane; r < nr; r += 32) s += S.P[r + a * ld] * S.P[r + b * ld];
        s = warp_sum(s);
        if (lane == 0) S.G[a + QB_NB * b] = s;
    }
    __syncthreads();
    if (warp == 0) {  // column i of T depends on columns < i; its rows a < i are independent (lane a)
        for (int i = lane; i < QB_NB * QB_NB; i += 32) S.T[i] = 0.0;
        __syncwarp();
        for (int i = 0; i < jb; ++i) {
            const double ti = S.tau[i];
            double s = 0.0;
            if (lane < i)
                for (int b = lane; b < i; ++b) s += S.T[lane + QB_NB * b] * S.G[b + QB_NB * i];
            __syncwarp();
            if (lane < i) S.T[lane + QB_NB * i] = -ti * s;
            if (lane == 0) S.T[i + QB_NB * i] = ti;
            __syncwarp();
        }
    }
    __syncthreads();
}

/// W1 = V^T C (16 x wc) with V the explicit panel (nr rows) and C = Cg[0:nr, 0:wc]
/// (global, ldc); DMMA over 8-column blocks of C, both 8-row halves of W1 per
/// warp (the C loads are shared). C is read straight from global memory (L2):
/// rows are streamed in groups of 32 with the next group's 8 loads issued
/// before the current group's 16 DMMAs.
__device__ __forceinline__ void qb_vt_c(const QbSmem& S, int ld, int nr, const double* Cg, i64 ldc, int wc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int g8 = lane >> 2, t4 = lane & 3;
    const int nct = (wc + 7) / 8;
    const int K = (nr + 3) & ~3;
    // few column blocks: one W1 half per warp (more warps busy); many: both
    // halves per warp (each C value loaded once)
    const bool split = nct < nwarps;
    const int ntask = split ? 2 * nct : nct;
    for (int task = warp; task < ntask; task += nwarps) {
        const int jt = split ? task >> 1 : task;
        const int h0 = split ? (task & 1) : 0, h1 = split ? h0 : 1;
        const int j0 = jt * 8;
        double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0}, d0[2] = {0.0, 0.0}, d1[2] = {0.0, 0.0};
        const bool colok = j0 + g8 < wc;
        const double* Bc = Cg + i64(colok ? j0 + g8 : 0) * ldc;
        const double* V0 = S.P + (8 * h0 + g8) * ld;
        const double* V1 = S.P + (8 * h1 + g8) * ld;
        double nb[8];
        auto fetch = [&](int k0) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int r = k0 + 4 * q + t4;
                nb[q] = (colok && r < nr) ? Bc[r] : 0.0;
            }
        };
        fetch(0);
        for (int k0 = 0; k0 < K; k0 += 32) {
            double b[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) b[q] = nb[q];
            if (k0 + 32 < K) fetch(k0 + 32);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (k0 + 4 * q < K) {
                    const int r = k0 + 4 * q + t4;
                    tile::dmma((q & 1) ? c1 : c0, V0[r], b[q]);
                    if (!split) tile::dmma((q & 1) ? d1 : d0, V1[r], b[q]);
                }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int j = j0 + 2 * t4 + e;
            if (j < wc) {
                S.W1[(8 * h0 + g8) + QB_NB * j] = c0[e] + c1[e];
                if (!split) S.W1[(8 + g8) + QB_NB * j] = d0[e] + d1[e];
            }
        }
    }
}

/// Cg[0:nr, 0:wc] -= V W2 (W2 16 x wc in shared memory). Each warp takes 4
/// 8x8 tiles per step (8 independent loads in flight) and loads the next 4
/// tiles' C values before the current tiles' DMMAs.
template <int TB>
__device__ __forceinline__ void qb_c_minus_vw_t(const QbSmem& S, int ld, int nr, double* Cg, i64 ldc, int wc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int g8 = lane >> 2, t4 = lane & 3;
    const int nrt = (nr + 7) / 8, nct = (wc + 7) / 8, ntl = nrt * nct;
    double nxt[TB][2];
    auto fetch = [&](int base) {
#pragma unroll
        for (int u = 0; u < TB; ++u) {
            const int tl = base + u;
            const int r = (tl % nrt) * 8 + g8, j0 = (tl / nrt) * 8;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int j = j0 + 2 * t4 + e;
                nxt[u][e] = (tl < ntl && r < nr && j < wc) ? Cg[r + i64(j) * ldc] : 0.0;
            }
        }
    };
    const int stride = nwarps * TB;
    if (warp * TB < ntl) fetch(warp * TB);
    for (int base = warp * TB; base < ntl; base += stride) {
        double acc[TB][2];
#pragma unroll
        for (int u = 0; u < TB; ++u) acc[u][0] = nxt[u][0], acc[u][1] = nxt[u][1];
        if (base + stride < ntl) fetch(base + stride);
#pragma unroll
        for (int u = 0; u < TB; ++u) {
            const int tl = base + u;
            if (tl >= ntl) break;
            const int r0 = (tl % nrt) * 8, j0 = (tl / nrt) * 8;
            const int jb = j0 + g8;
#pragma unroll
            for (int kk = 0; kk < QB_NB; kk += 4) {
                const double b = jb < wc ? S.W2[(kk + t4) + QB_NB * jb] : 0.0;
                tile::dmma(acc[u], -S.P[r0 + g8 + (kk + t4) * ld], b);
            }
        }
#pragma unroll
        for (int u = 0; u < TB; ++u) {
            const int tl = base + u;
            if (tl >= ntl) break;
            const int r = (tl % nrt) * 8 + g8, j0 = (tl / nrt) * 8;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int j = j0 + 2 * t4 + e;
                if (r < nr && j < wc) Cg[r + i64(j) * ldc] = acc[u][e];
            }
        }
    }
}

/// Batch 4 tiles per warp step only when every warp gets several batches.
__device__ __forceinline__ void qb_c_minus_vw(const QbSmem& S, int ld, int nr, double* Cg, i64 ldc, int wc) {
    const int ntl = ((nr + 7) / 8) * ((wc + 7) / 8);
    if (ntl >= 4 * 2 * int(blockDim.x >> 5))
        qb_c_minus_vw_t<4>(S, ld, nr, Cg, ldc, wc);
    else
        qb_c_minus_vw_t<1>(S, ld, nr, Cg, ldc, wc);
}

__global__ void __launch_bounds__(QB_THREADS, 3) k_qr_blocked(const QrDesc* descs, int w) {
    extern __shared__ double sm[];
    const QrDesc d = descs[blockIdx.x];
    const int rows = d.rows, ld = qb_ld(rows);
    const QbSmem S = qb_layout(sm, rows, w);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int nsz = min(rows, w);
    double* A = d.A;
    for (int p0 = 0; p0 < nsz; p0 += QB_NB) {
        const int jb = min(QB_NB, nsz - p0), nr = rows - p0;
        // 1. panel into shared memory and its level-2 factorization
        for (int e = tid; e < nr * jb; e += blockDim.x) {
            const int r = e % nr, i = e / nr;
            S.P[r + i * ld] = A[(p0 + r) + i64(p0 + i) * d.lda];
        }
        __syncthreads();
        for (int i = 0; i < jb; ++i) {
            double part = 0.0;
            for (int r = i + 1 + tid; r < nr; r += blockDim.x) part += S.P[r + i * ld] * S.P[r + i * ld];
            const double c0 = S.P[i + i * ld];  // read before the sum's barriers (thread 0 rewrites it below)
            const double tail = qr_block_sum(part);
            // every thread derives the reflector from the same sum (no extra barrier)
            const bool zero = tail <= DBL_MIN;
            double tau = 0.0, div = 1.0, beta = c0;
            if (!zero) {
                beta = sqrt(c0 * c0 + tail);
                if (c0 >= 0.0) beta = -beta;
                div = c0 - beta;
                tau = (beta - c0) / beta;
            }
            if (tid == 0) {
                if (!zero) S.P[i + i * ld] = beta;
                d.tau[p0 + i] = tau;
                S.tau[i] = tau;
            }
            for (int r = i + 1 + tid; r < nr; r += blockDim.x) S.P[r + i * ld] = zero ? 0.0 : S.P[r + i * ld] / div;
            __syncthreads();
            for (int j = i + 1 + warp; j < jb; j += nwarps) {
                double* cj = S.P + j * ld;
                if (nr - i == 1) {
                    if (lane == 0) cj[i] *= (1.0 - tau);
                } else if (tau != 0.0) {
                    double t = 0.0;
                    for (int r = i + 1 + lane; r < nr; r += 32) t += S.P[r + i * ld] * cj[r];
                    t = warp_sum(t) + cj[i];
                    for (int r = i + 1 + lane; r < nr; r += 32) cj[r] -= tau * S.P[r + i * ld] * t;
                    __syncwarp();
                    if (lane == 0) cj[i] -= tau * t;
                }
            }
            __syncthreads();
        }
        for (int e = tid; e < nr * jb; e += blockDim.x) {
            const int r = e % nr, i = e / nr;
            A[(p0 + r) + i64(p0 + i) * d.lda] = S.P[r + i * ld];
        }
        __syncthreads();
        const int wc = w - p0 - jb;
        if (wc <= 0) continue;
        // 2. explicit V and T
        qb_explicit_v(S.P, ld, nr, jb);
        __syncthreads();
        qb_build_t(S, ld, nr, jb);
        // 3. C <- C - V (T^T (V^T C))
        double* C = A + p0 + i64(p0 + jb) * d.lda;
        qb_vt_c(S, ld, nr, C, d.lda, wc);
        __syncthreads();
        for (int e = tid; e < QB_NB * wc; e += blockDim.x) {
            const int i = e % QB_NB, j = e / QB_NB;
            double s = 0.0;
            for (int a = 0; a <= i; ++a) s += S.T[a + QB_NB * i] * S.W1[a + QB_NB * j];
            S.W2[i + QB_NB * j] = s;
        }
        __syncthreads();
        qb_c_minus_vw(S, ld, nr, C, d.lda, wc);
        __syncthreads();
    }
    if (d.R)
        for (int e = tid; e < w * w; e += blockDim.x) {
            const int i = e % w, j = e / w;
            d.R[i + j * d.ldr] = (i <= j && i < nsz) ? A[i + i64(j) * d.lda] : 0.0;
        }
}

/// Columns of Q are independent given the reflectors: CTA (block, chunk)
/// forms columns [cc0, cc0 + chunk) (few large blocks still fill the GPU).
__global__ void __launch_bounds__(QB_THREADS, 3) k_form_q_blocked(const QfDesc* descs, int w, int qcols_all,
                                                                  int chunk) {
    extern __shared__ double sm[];
    const QfDesc d = descs[blockIdx.x];
    const int cc0 = blockIdx.y * chunk, qcols = min(qcols_all, cc0 + chunk) - cc0;
    if (qcols <= 0) return;
    const int rows = d.rows, ld = qb_ld(rows);
    const QbSmem S = qb_layout(sm, rows, qcols_all);
    const int tid = threadIdx.x;
    // identity Tin: H_i (i >= c) leaves e_c unchanged, so columns < cc0 + qcols
    // only see the first cc0 + qcols reflectors
    const int nref = d.Tin ? min(w, rows) : min(min(w, rows), cc0 + qcols);
    double* Q = d.Q + i64(cc0) * d.ldq;
    for (int c = 0; c < qcols; ++c)
        for (int i = tid; i < rows; i += blockDim.x) {
            const int cg = cc0 + c;
            double v = 0.0;
            if (i < nref) v = d.Tin ? d.Tin[i + i64(cg) * d.ldt] : (i == cg ? 1.0 : 0.0);
            Q[i + i64(c) * d.ldq] = v;
        }
    __syncthreads();
    for (int p0 = ((nref - 1) / QB_NB) * QB_NB; p0 >= 0; p0 -= QB_NB) {
        const int jb = min(QB_NB, nref - p0), nr = rows - p0;
        for (int e = tid; e < nr * jb; e += blockDim.x) {
            const int r = e % nr, i = e / nr;
            S.P[r + i * ld] = d.A[(p0 + r) + i64(p0 + i) * d.lda];
        }
        if (tid < QB_NB) S.tau[tid] = tid < jb ? d.tau[p0 + tid] : 0.0;
        __syncthreads();
        qb_explicit_v(S.P, ld, nr, jb);
        __syncthreads();
        qb_build_t(S, ld, nr, jb);
        double* Qp = Q + p0;
        qb_vt_c(S, ld, nr, Qp, d.ldq, qcols);
        __syncthreads();
        for (int e = tid; e < QB_NB * qcols; e += blockDim.x) {  // W2 = T W1
            const int i = e % QB_NB, j = e / QB_NB;
            double s = 0.0;
            for (int a = i; a < QB_NB; ++a) s += S.T[i + QB_NB * a] * S.W1[a + QB_NB * j];
            S.W2[i + QB_NB * j] = s;
        }
        __syncthreads();
        qb_c_minus_vw(S, ld, nr, Qp, d.ldq, qcols);
        __syncthreads();
    }
}
