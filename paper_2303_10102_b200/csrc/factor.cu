// HODLR factorization, Woodbury solves and log-determinant on the device.
// Reference: factorization.cpp:7-224 (see factor.cuh for the data layout).
#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "factor.cuh"
#include "prof.cuh"
#include "tile.cuh"

namespace hg {

namespace {

constexpr int FNT = 256;
constexpr int SOLVE_COLS = 64;
constexpr int MAX_LEAF = 320;

// ---------------------------------------------------- block-cooperative helpers
/// argmax_i |x_i| over the calling block, first index on ties.
__device__ void block_argmax(double v, int idx, double& out_v, int& out_i) {
    __shared__ double sv[32];
    __shared__ int si[32];
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_down_sync(0xffffffffu, v, o);
        int oi = __shfl_down_sync(0xffffffffu, idx, o);
        if (ov > v || (ov == v && oi < idx && oi >= 0) || (idx < 0 && oi >= 0)) {
            v = ov;
            idx = oi;
        }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        sv[wid] = v;
        si[wid] = idx;
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = blockDim.x >> 5;
        v = lane < nw ? sv[lane] : -1.0;
        idx = lane < nw ? si[lane] : -1;
        for (int o = 16; o > 0; o >>= 1) {
            double ov = __shfl_down_sync(0xffffffffu, v, o);
            int oi = __shfl_down_sync(0xffffffffu, idx, o);
            if (ov > v || (ov == v && oi < idx && oi >= 0) || (idx < 0 && oi >= 0)) {
                v = ov;
                idx = oi;
            }
        }
        if (lane == 0) {
            sv[0] = v;
            si[0] = idx;
        }
    }
    __syncthreads();
    out_v = sv[0];
    out_i = si[0];
    __syncthreads();
}

/// In-place Cholesky of the lower triangle (Eigen LLT semantics: fails when a
/// pivot is <= 0). Returns false on failure.
__device__ bool dev_llt(double* W, int ldw, int m) {
    __shared__ int s_ok;
    for (int k = 0; k < m; ++k) {
        if (threadIdx.x == 0) {
            const double x = W[k + i64(k) * ldw];
            if (x <= 0.0) {
                s_ok = 0;
            } else {
                W[k + i64(k) * ldw] = sqrt(x);
                s_ok = 1;
            }
        }
        __syncthreads();
        if (!s_ok) return false;
        const double d = W[k + i64(k) * ldw];
        for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) W[i + i64(k) * ldw] /= d;
        __syncthreads();
        // trailing update of the lower triangle: warp per column, lanes down the rows
        const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        for (int j = k + 1 + int(threadIdx.x >> 5); j < m; j += nw) {
            const double wjk = W[j + i64(k) * ldw];
            for (int i = j + lane; i < m; i += 32) W[i + i64(j) * ldw] -= W[i + i64(k) * ldw] * wjk;
        }
        __syncthreads();
    }
    return true;
}

/// dev_llt on the packed lower triangle: column j holds rows [j, m) at
/// Wp[i + cb(j)], cb(j) = j m - j (j + 1) / 2 (half the shared memory of the
/// square layout, so three factorizations share an SM instead of one).
__device__ __forceinline__ int ll_cb(int j, int m) { return j * m - j * (j + 1) / 2; }

__device__ bool dev_llt_packed(double* Wp, int m) {
    __shared__ int s_ok;
    for (int k = 0; k < m; ++k) {
        const int ck = ll_cb(k, m);
        if (threadIdx.x == 0) {
            const double x = Wp[k + ck];
            if (x <= 0.0) {
                s_ok = 0;
            } else {
                Wp[k + ck] = sqrt(x);
                s_ok = 1;
            }
        }
        __syncthreads();
        if (!s_ok) return false;
        const double d = Wp[k + ck];
        for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) Wp[i + ck] /= d;
        __syncthreads();
        const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
        for (int j = k + 1 + int(threadIdx.x >> 5); j < m; j += nw) {
            const double wjk = Wp[j + ck];
            double* cj = Wp + ll_cb(j, m);
            for (int i = j + lane; i < m; i += 32) cj[i] -= Wp[i + ck] * wjk;
        }
        __syncthreads();
    }
    return true;
}

/// In-place LU with partial pivoting (Eigen PartialPivLU: first max-abs
/// pivot; zero pivots leave the column unscaled). Row swaps -> piv[k].
__device__ int dev_lu(double* W, int ldw, int m, int* piv) {
    int nswap = 0;
    for (int k = 0; k < m; ++k) {
        double bv = -1.0;
        int bi = -1;
        for (int i = k + threadIdx.x; i < m; i += blockDim.x) {
            const double a = fabs(W[i + i64(k) * ldw]);
            if (a > bv) {
                bv = a;
                bi = i;
            }
        }
        double mv;
        int p;
        block_argmax(bv, bi, mv, p);
        if (p < 0) p = k;
        if (threadIdx.x == 0) piv[k] = p;
        if (p != k) {
            ++nswap;
            for (int j = threadIdx.x; j < m; j += blockDim.x) {
                const double t = W[k + i64(j) * ldw];
                W[k + i64(j) * ldw] = W[p + i64(j) * ldw];
                W[p + i64(j) * ldw] = t;
            }
        }
        __syncthreads();
        const double pv = W[k + i64(k) * ldw];
        if (pv != 0.0)
            for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) W[i + i64(k) * ldw] /= pv;
        __syncthreads();
        const int rem = m - k - 1;
        for (int e = threadIdx.x; e < rem * rem; e += blockDim.x) {
            const int i = k + 1 + e % rem, j = k + 1 + e / rem;
            W[i + i64(j) * ldw] -= W[i + i64(k) * ldw] * W[k + i64(j) * ldw];
        }
        __syncthreads();
    }
    return nswap;
}

// ------------------------------------------------------------ leaf factor
struct LeafFacArgs {
    const int* bounds;
    int bmax;
    const double* orig;
    double* fac;
    int prefer_llt;
    int use_smem;
    int* kind;
    int* piv;
    double* ld;
    int* sign;
};

__global__ void __launch_bounds__(FNT) k_leaf_factor(LeafFacArgs g) {
    extern __shared__ double sm[];
    const int b = blockIdx.x;
    const int m = g.bounds[b + 1] - g.bounds[b];
    const i64 ls = i64(g.bmax) * g.bmax;
    const double* A = g.orig + b * ls;
    if (g.use_smem == 2) {  // packed lower-triangle Cholesky in shared memory
        for (int j = 0; j < m; ++j)
            for (int i = j + threadIdx.x; i < m; i += blockDim.x) sm[i + ll_cb(j, m)] = A[i + i64(j) * g.bmax];
        __syncthreads();
        if (dev_llt_packed(sm, m)) {
            double* F = g.fac + b * ls;
            for (int j = 0; j < m; ++j)
                for (int i = j + threadIdx.x; i < m; i += blockDim.x) F[i + i64(j) * g.bmax] = sm[i + ll_cb(j, m)];
            if (threadIdx.x == 0) {
                double ld = 0.0;
                for (int i = 0; i < m; ++i) ld += log(sm[i + ll_cb(i, m)]);
                g.kind[b] = 1;
                g.ld[b] = 2.0 * ld;
                g.sign[b] = 1;
            }
            return;
        }
        // not SPD: PartialPivLU in global memory (factorization.cpp:10-17 fallback)
        double* W = g.fac + b * ls;
        for (int j = 0; j < m; ++j)
            for (int i = threadIdx.x; i < m; i += blockDim.x) W[i + i64(j) * g.bmax] = A[i + i64(j) * g.bmax];
        __syncthreads();
        const int nswap = dev_lu(W, g.bmax, m, g.piv + i64(b) * g.bmax);
        if (threadIdx.x == 0) {
            double ld = 0.0;
            int sign = (nswap & 1) ? -1 : 1;
            for (int i = 0; i < m; ++i) {
                const double d = W[i + i64(i) * g.bmax];
                if (d < 0) sign = -sign;
                ld += log(fabs(d));
            }
            g.kind[b] = 0;
            g.ld[b] = ld;
            g.sign[b] = sign;
        }
        return;
    }
    double* W = g.use_smem ? sm : g.fac + b * ls;
    const int ldw = g.use_smem ? m : g.bmax;
    int* piv = g.piv + i64(b) * g.bmax;
    for (int j = 0; j < m; ++j)
        for (int i = threadIdx.x; i < m; i += blockDim.x) W[i + i64(j) * ldw] = A[i + i64(j) * g.bmax];
    __syncthreads();
    bool llt = false;
    if (g.prefer_llt) llt = dev_llt(W, ldw, m);
    int nswap = 0;
    if (!llt) {
        for (int j = 0; j < m; ++j)
            for (int i = threadIdx.x; i < m; i += blockDim.x) W[i + i64(j) * ldw] = A[i + i64(j) * g.bmax];
        __syncthreads();
        nswap = dev_lu(W, ldw, m, piv);
    }
    if (threadIdx.x == 0) {
        double ld = 0.0;
        int sign = 1;
        if (llt) {
            for (int i = 0; i < m; ++i) ld += log(W[i + i64(i) * ldw]);
            ld *= 2.0;
        } else {
            sign = (nswap & 1) ? -1 : 1;
            for (int i = 0; i < m; ++i) {
                const double d = W[i + i64(i) * ldw];
                if (d < 0) sign = -sign;
                ld += log(fabs(d));
            }
        }
        g.kind[b] = llt ? 1 : 0;
        g.ld[b] = ld;
        g.sign[b] = sign;
    }
    if (g.use_smem) {
        __syncthreads();
        double* F = g.fac + b * ls;
        for (int j = 0; j < m; ++j)
            for (int i = threadIdx.x; i < m; i += blockDim.x) F[i + i64(j) * g.bmax] = W[i + i64(j) * ldw];
    }
}

// -------------------------------------------------------------- leaf solve
struct LeafSolveArgs {
    const int* bounds;
    int bmax;
    const double* fac;
    const int* kind;
    const int* piv;
    double* Y;
    i64 ldy;
    int w;
};

/// Blocked substitution on one leaf x 64 RHS columns held in shared memory.
/// LLT: L y = b, L^T x = y. LU: P b, unit-lower L, upper U.
__global__ void __launch_bounds__(FNT) k_leaf_solve(LeafSolveArgs g) {
    extern __shared__ double sm[];
    const int b = blockIdx.x;
    const int lo = g.bounds[b], m = g.bounds[b + 1] - lo;
    const int c0 = blockIdx.y * SOLVE_COLS;
    const int nc = min(SOLVE_COLS, g.w - c0);
    const double* F = g.fac + i64(b) * g.bmax * g.bmax;
    const int ldf = g.bmax;
    const bool llt = g.kind[b] != 0;
    constexpr int YS = SOLVE_COLS + 1;
    double* Ys = sm;                 // m x YS (row-major: Ys[r*YS + c])
    double* Ls = sm + i64(m) * YS;   // 16 x (m + 1)
    const int LS = m + 1;
    const int tid = threadIdx.x;
    for (int e = tid; e < m * SOLVE_COLS; e += blockDim.x) {
        const int r = e % m, c = e / m;
        Ys[r * YS + c] = c < nc ? g.Y[i64(lo + r) + i64(c0 + c) * g.ldy] : 0.0;
    }
    __syncthreads();
    if (!llt) {  // P b
        const int* piv = g.piv + i64(b) * g.bmax;
        for (int k = 0; k < m; ++k) {
            const int p = piv[k];
            if (p != k && tid < SOLVE_COLS) {
                const double t = Ys[k * YS + tid];
                Ys[k * YS + tid] = Ys[p * YS + tid];
                Ys[p * YS + tid] = t;
            }
            __syncthreads();
        }
    }
    const int c = tid & 63, r4 = tid >> 6;
    // forward: lower triangle (L for LLT, unit L for LU)
    for (int ib = 0; ib < m; ib += 16) {
        const int nb = min(16, m - ib);
        for (int e = tid; e < nb * (ib + nb); e += blockDim.x) {
            const int q = e % nb, p = e / nb;
            Ls[q * LS + p] = F[(ib + q) + i64(p) * ldf];
        }
        __syncthreads();
        double acc[4] = {0, 0, 0, 0};
        for (int p = 0; p < ib; ++p) {
            const double y = Ys[p * YS + c];
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (r4 * 4 + t < nb) acc[t] = fma(Ls[(r4 * 4 + t) * LS + p], y, acc[t]);
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (r4 * 4 + t < nb) Ys[(ib + r4 * 4 + t) * YS + c] -= acc[t];
        __syncthreads();
        if (tid < SOLVE_COLS) {
            for (int q = 0; q < nb; ++q) {
                double s = Ys[(ib + q) * YS + tid];
                for (int p = 0; p < q; ++p) s -= Ls[q * LS + ib + p] * Ys[(ib + p) * YS + tid];
                Ys[(ib + q) * YS + tid] = llt ? s / Ls[q * LS + ib + q] : s;
            }
        }
        __syncthreads();
    }
    // backward: upper triangle (L^T for LLT, U for LU); Ls[q][p] = T(ib+q, p)
    for (int ib = ((m - 1) / 16) * 16; ib >= 0; ib -= 16) {
        const int nb = min(16, m - ib);
        const int rest = m - ib;
        for (int e = tid; e < nb * rest; e += blockDim.x) {
            int q, pp;
            double v;
            if (llt) {  // T(ib+q, ib+pp) = L(ib+pp, ib+q): contiguous in pp
                pp = e % rest;
                q = e / rest;
                v = F[(ib + pp) + i64(ib + q) * ldf];
            } else {  // T(ib+q, ib+pp) = U(ib+q, ib+pp): contiguous in q
                q = e % nb;
                pp = e / nb;
                v = F[(ib + q) + i64(ib + pp) * ldf];
            }
            Ls[q * LS + pp] = v;
        }
        __syncthreads();
        double acc[4] = {0, 0, 0, 0};
        for (int pp = nb; pp < rest; ++pp) {
            const double y = Ys[(ib + pp) * YS + c];
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (r4 * 4 + t < nb) acc[t] = fma(Ls[(r4 * 4 + t) * LS + pp], y, acc[t]);
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (r4 * 4 + t < nb) Ys[(ib + r4 * 4 + t) * YS + c] -= acc[t];
        __syncthreads();
        if (tid < SOLVE_COLS) {
            for (int q = nb - 1; q >= 0; --q) {
                double s = Ys[(ib + q) * YS + tid];
                for (int pp = q + 1; pp < nb; ++pp) s -= Ls[q * LS + pp] * Ys[(ib + pp) * YS + tid];
                Ys[(ib + q) * YS + tid] = s / Ls[q * LS + q];
            }
        }
        __syncthreads();
    }
    for (int e = tid; e < m * nc; e += blockDim.x) {
        const int r = e % m, cc = e / m;
        g.Y[i64(lo + r) + i64(c0 + cc) * g.ldy] = Ys[r * YS + cc];
    }
}

#include "leafsolve_tc.cuh"

// --------------------------------------------------------------- capacitance
struct CapLuArgs {
    int R;
    const double* P;  // per child R x R (ld R)
    double* lu;       // per node 2R x 2R
    int* piv;
    double* ld;
    int* sign;
    int use_smem;
};

__global__ void __launch_bounds__(FNT) k_cap_lu(CapLuArgs g) {
    extern __shared__ double sm[];
    const int j = blockIdx.x, R = g.R, m = 2 * R;
    double* W = g.use_smem ? sm : g.lu + i64(j) * m * m;
    const double* Pl = g.P + i64(2 * j) * R * R;      // w^T wbar (left child)
    const double* Pr = g.P + i64(2 * j + 1) * R * R;  // x^T xbar (right child)
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int r = e % m, c = e / m;
        double v;
        if (r < R && c < R)
            v = r == c ? 1.0 : 0.0;
        else if (r < R)
            v = Pr[r + (c - R) * R];
        else if (c < R)
            v = Pl[(r - R) + c * R];
        else
            v = r == c ? 1.0 : 0.0;
        W[r + i64(c) * m] = v;
    }
    __syncthreads();
    const int nswap = dev_lu(W, m, m, g.piv + i64(j) * m);
    if (threadIdx.x == 0) {
        double ld = 0.0;
        int sign = (nswap & 1) ? -1 : 1;
        for (int i = 0; i < m; ++i) {
            const double d = W[i + i64(i) * m];
            if (d < 0) sign = -sign;
            ld += log(fabs(d));
        }
        g.ld[j] = ld;
        g.sign[j] = sign;
    }
    if (g.use_smem) {
        __syncthreads();
        double* O = g.lu + i64(j) * m * m;
        for (int e = threadIdx.x; e < m * m; e += blockDim.x) O[e] = W[e];
    }
}

struct CapSolveArgs {
    int R, w;
    const double* lu;
    const int* piv;
    const double* Q;  // per child R x w (ld R, stride R*w); null => identity RHS
    int top_odd;
    int trans;
    double* T;  // per node 2R x w (ld 2R)
    int stage_lu;
};

/// One thread per RHS column; LU in global memory (L1/L2 broadcast reads).
__global__ void k_cap_solve(CapSolveArgs g) {
    extern __shared__ double sm[];
    const int j = blockIdx.x, R = g.R, m = 2 * R;
    const int c = threadIdx.x, col = blockIdx.y * blockDim.x + c;
    const int nthr = blockDim.x;
    double* x = sm;  // x[r * nthr + c]
    const double* A = g.lu + i64(j) * m * m;
    if (g.stage_lu) {  // the LU in shared memory: every substitution step reads it
        double* As = sm + m * nthr;
        for (int e = threadIdx.x; e < m * m; e += nthr) As[e] = A[e];
        __syncthreads();
        A = As;
    }
    const int* piv = g.piv + i64(j) * m;
    const bool active = col < g.w;
    if (active) {
        const double* Qt = g.Q ? g.Q + i64(2 * j + (g.top_odd ? 1 : 0)) * R * g.w : nullptr;
        const double* Qb = g.Q ? g.Q + i64(2 * j + (g.top_odd ? 0 : 1)) * R * g.w : nullptr;
        for (int r = 0; r < m; ++r) {
            double v;
            if (!g.Q)
                v = (r == col) ? 1.0 : 0.0;
            else
                v = r < R ? Qt[r + i64(col) * R] : Qb[(r - R) + i64(col) * R];
            x[r * nthr + c] = v;
        }
        if (!g.trans) {
            for (int k = 0; k < m; ++k) {
                const int p = piv[k];
                if (p != k) {
                    const double t = x[k * nthr + c];
                    x[k * nthr + c] = x[p * nthr + c];
                    x[p * nthr + c] = t;
                }
            }
            for (int i = 0; i < m; ++i) {  // unit lower
                double s = x[i * nthr + c];
                for (int p = 0; p < i; ++p) s -= A[i + i64(p) * m] * x[p * nthr + c];
                x[i * nthr + c] = s;
            }
            for (int i = m - 1; i >= 0; --i) {  // upper
                double s = x[i * nthr + c];
                for (int p = i + 1; p < m; ++p) s -= A[i + i64(p) * m] * x[p * nthr + c];
                x[i * nthr + c] = s / A[i + i64(i) * m];
            }
        } else {
            for (int i = 0; i < m; ++i) {  // U^T y = b
                double s = x[i * nthr + c];
                for (int p = 0; p < i; ++p) s -= A[p + i64(i) * m] * x[p * nthr + c];
                x[i * nthr + c] = s / A[i + i64(i) * m];
            }
            for (int i = m - 1; i >= 0; --i) {  // L^T z = y (unit)
                double s = x[i * nthr + c];
                for (int p = i + 1; p < m; ++p) s -= A[p + i64(i) * m] * x[p * nthr + c];
                x[i * nthr + c] = s;
            }
            for (int k = m - 1; k >= 0; --k) {  // x = P^T z
                const int p = piv[k];
                if (p != k) {
                    const double t = x[k * nthr + c];
                    x[k * nthr + c] = x[p * nthr + c];
                    x[p * nthr + c] = t;
                }
            }
        }
        double* out = g.T + i64(j) * m * g.w;
        for (int r = 0; r < m; ++r) out[r + i64(col) * m] = x[r * nthr + c];
    }
}

void set_smem(const void* fn, size_t bytes) {
    if (bytes > 48 * 1024) HG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

constexpr size_t SMEM_CAP = 220 * 1024;

void cap_solve(const DFactor& f, int i, const double* Q, bool top_odd, bool trans, double* T, int w) {
    const int R = f.Rl(i), m = 2 * R;
    const int nodes = 1 << (i - 1);
    int thr = 64;
    while (thr > 8 && static_cast<size_t>(m) * thr * sizeof(double) > SMEM_CAP) thr >>= 1;
    size_t smem = static_cast<size_t>(m) * thr * sizeof(double);
    if (smem > SMEM_CAP) throw std::length_error("cap_solve: capacitance too large for shared memory");
    const bool stage = smem + static_cast<size_t>(m) * m * sizeof(double) <= SMEM_CAP;
    if (stage) smem += static_cast<size_t>(m) * m * sizeof(double);
    ProfScope prof(PROF_CAP_SOLVE, 2.0 * nodes * double(m) * m * w, 8.0 * nodes * (double(m) * m + 2.0 * m * w));
    set_smem(reinterpret_cast<const void*>(k_cap_solve), smem);
    CapSolveArgs g{R, w, f.cap[static_cast<size_t>(i - 1)]->get(), f.cap_piv[static_cast<size_t>(i - 1)]->get(), Q, top_odd ? 1 : 0,
                   trans ? 1 : 0, T, stage ? 1 : 0};
    dim3 grid(unsigned(nodes), unsigned(cdiv(w, thr)));
    k_cap_solve<<<grid, thr, smem, current().stream>>>(g);
    HG_LAUNCH();
    count_launch();
}

/// p = -v cap^{-T} of every level-i node by LU substitution per row of v
/// (product_rep.cpp:74-78: p = -(cap.solve(v^T))^T), the reference's own
/// association; v = [0 w; x 0] from the source panel F. One thread per row.
__global__ void k_cap_p_rows(int R, const int* bounds, const double* lu, const int* piv_all, const double* F, i64 n,
                             double* P) {
    extern __shared__ double sm[];
    const int j = blockIdx.x, m = 2 * R, nthr = blockDim.x, c = threadIdx.x;
    const int lo = bounds[2 * j], mid = bounds[2 * j + 1], hi = bounds[2 * j + 2];
    const int row = lo + blockIdx.y * nthr + c;
    if (row >= hi) return;
    const double* A = lu + i64(j) * m * m;
    const int* piv = piv_all + i64(j) * m;
    double* x = sm;  // x[r * nthr + c]
    const bool left = row < mid;
    for (int r = 0; r < m; ++r) {
        const bool src = left ? r >= R : r < R;
        x[r * nthr + c] = src ? F[row + i64(left ? r - R : r) * n] : 0.0;
    }
    for (int k = 0; k < m; ++k) {
        const int p = piv[k];
        if (p != k) {
            const double t = x[k * nthr + c];
            x[k * nthr + c] = x[p * nthr + c];
            x[p * nthr + c] = t;
        }
    }
    for (int i = 0; i < m; ++i) {  // unit lower
        double s = x[i * nthr + c];
        for (int p = 0; p < i; ++p) s -= A[i + i64(p) * m] * x[p * nthr + c];
        x[i * nthr + c] = s;
    }
    for (int i = m - 1; i >= 0; --i) {  // upper
        double s = x[i * nthr + c];
        for (int p = i + 1; p < m; ++p) s -= A[i + i64(p) * m] * x[p * nthr + c];
        x[i * nthr + c] = s / A[i + i64(i) * m];
    }
    for (int r = 0; r < m; ++r) P[row + i64(r) * n] = -x[r * nthr + c];
}

void form_p_reference_impl(const DFactor& f, int i, double* P) {
    const int R = f.Rl(i), m = 2 * R;
    if (R == 0) return;
    const Partition& p = f.tree->part(i);
    const int nodes = p.nseg() / 2;
    int maxrows = 0;
    for (int j = 0; j < nodes; ++j) maxrows = std::max(maxrows, p.hbounds()[2 * j + 2] - p.hbounds()[2 * j]);
    int thr = 64;
    while (thr > 8 && static_cast<size_t>(m) * thr * sizeof(double) > SMEM_CAP) thr >>= 1;
    const size_t smem = static_cast<size_t>(m) * thr * sizeof(double);
    if (smem > SMEM_CAP) throw std::length_error("form_p_reference: capacitance too large for shared memory");
    ProfScope prof(PROF_CAP_SOLVE, 2.0 * double(f.n()) * m * m, 8.0 * nodes * double(m) * m + 16.0 * f.n() * m);
    set_smem(reinterpret_cast<const void*>(k_cap_p_rows), smem);
    dim3 grid(unsigned(nodes), unsigned(cdiv(maxrows, thr)));
    k_cap_p_rows<<<grid, thr, smem, current().stream>>>(R, p.dbounds(), f.cap[static_cast<size_t>(i - 1)]->get(),
                                                       f.cap_piv[static_cast<size_t>(i - 1)]->get(), f.Fl(i), f.n(), P);
    HG_LAUNCH();
    count_launch();
}

/// Node panels (nodes*m rows, ld L = nodes*m) of the capacitance operators,
/// with Pi the half swap so that node j's right-hand side is the contiguous
/// block [Q_{2j}; Q_{2j+1}]:
///   Right solve  (cap^{-1} [Q_{2j+1}; Q_{2j}]):  SR = cap^{-1} Pi, AR = Pi cap
///   Left solve   (cap^{-T} [Q_{2j}; Q_{2j+1}]):  SL = cap^{-T},    AL = cap^T
/// from E_j = cap_j^{-T} (m x m, ld m) and the blocks P of cap (k_cap_lu).
__global__ void k_cap_panels(const double* E, const double* P, int R, i64 L, double* SR, double* AR, double* SL,
                             double* AL) {
    const int j = blockIdx.x, m = 2 * R;
    const double* Ej = E + i64(j) * m * m;
    const double* Pl = P + i64(2 * j) * R * R;
    const double* Pr = P + i64(2 * j + 1) * R * R;
    auto cap = [&](int r, int c) -> double {
        if ((r < R) == (c < R)) return r == c ? 1.0 : 0.0;
        return r < R ? Pr[r + (c - R) * R] : Pl[(r - R) + c * R];
    };
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int r = e % m, c = e / m;
        const int swc = c < R ? c + R : c - R, swr = r < R ? r + R : r - R;
        const i64 o = i64(j) * m + r + i64(c) * L;
        SL[o] = Ej[r + i64(c) * m];
        SR[o] = Ej[swc + i64(r) * m];
        AR[o] = cap(swr, c);
        AL[o] = cap(c, r);
    }
}

/// Y <- Abar^{-1} Y by blocked substitution with the leaf factors. (An
/// explicit-inverse GEMM path was tried and dropped: with refinement it is
/// slower, without it the leaves' conditioning costs parity.)
void leaf_solve_subst(const DFactor& f, double* Y, i64 ldy, int w) {
    if (w <= 0) return;
    const Partition& lv = f.tree->leaves();
    const int m = lv.max_seg();
    const size_t smem = (static_cast<size_t>(m) * (SOLVE_COLS + 1) + 16 * static_cast<size_t>(m + 1)) * sizeof(double);
    const double rows = double(f.n());
    ProfScope prof(PROF_LEAF_SOLVE, 2.0 * rows * m * w, 8.0 * (rows * m + 2.0 * rows * w));
    if (prof_enabled()) prof.key(prof_tag("leafsolve w=%d", w));
    if (f.all_llt && f.bmax() <= TS_MAX) {
        static DeviceOnce attr;
        if (attr.first()) set_smem(reinterpret_cast<const void*>(k_leaf_solve_tc<TS_S>), TS_SMEM);
        // Column tiles per CTA: enough CTAs for ~4 waves, the factor loaded once per CTA.
        const int ct = cdiv(w, TS_NC);
        const int groups = std::max(1, std::min(ct, cdiv(4 * 2 * current().num_sms, lv.nseg())));
        const int cpt = cdiv(ct, groups);
        LeafSolveTcArgs a{lv.dbounds(), f.bmax(), f.leaf_fac->get(), Y, ldy, w, ct, cpt};
        k_leaf_solve_tc<TS_S>
            <<<unsigned(lv.nseg()) * unsigned(cdiv(ct, cpt)), TS_NC * 4 / TS_S, TS_SMEM, current().stream>>>(a);
        HG_LAUNCH();
        count_launch();
        return;
    }
    if (f.all_llt && f.bmax() <= TS2_MAX) {  // 129..256-row leaves: 2 x 2 blocks
        static DeviceOnce attr2;
        if (attr2.first()) set_smem(reinterpret_cast<const void*>(k_leaf_solve_tc2), TS2_SMEM);
        const int ct = cdiv(w, TS_NC);
        const int groups = std::max(1, std::min(ct, cdiv(4 * current().num_sms, lv.nseg())));
        const int cpt = cdiv(ct, groups);
        LeafSolveTcArgs a{lv.dbounds(), f.bmax(), f.leaf_fac->get(), Y, ldy, w, ct, cpt};
        k_leaf_solve_tc2<<<unsigned(lv.nseg()) * unsigned(cdiv(ct, cpt)), TS_THREADS, TS2_SMEM, current().stream>>>(a);
        HG_LAUNCH();
        count_launch();
        return;
    }
    set_smem(reinterpret_cast<const void*>(k_leaf_solve), smem);
    LeafSolveArgs g{lv.dbounds(), f.bmax(), f.leaf_fac->get(), f.leaf_kind->get(), f.leaf_piv->get(), Y, ldy, w};
    dim3 grid(unsigned(lv.nseg()), unsigned(cdiv(w, SOLVE_COLS)));
    k_leaf_solve<<<grid, FNT, smem, current().stream>>>(g);
    HG_LAUNCH();
    count_launch();
}

}  // namespace

void leaf_solve(const DFactor& f, double* Y, i64 ldy, int w) { leaf_solve_subst(f, Y, ldy, w); }

void form_p_reference(const DFactor& f, int i, double* P) { form_p_reference_impl(f, i, P); }

void level_inverse(const DFactor& f, int i, bool transposed, double* Y, i64 ldy, int w) {
    const int R = f.Rl(i);
    if (R == 0 || w <= 0) return;
    const Partition& p = f.tree->part(i);
    const i64 n = f.n();
    const int m = 2 * R, nodes = p.nseg() / 2;
    const i64 L = i64(p.nseg()) * R;
    // Q panel: rows s*R.. hold the projection of child s, so node j's
    // [Q_{2j}; Q_{2j+1}] is one contiguous 2R-row block.
    DVec Q(static_cast<size_t>(L) * static_cast<size_t>(w));
    DVec T(static_cast<size_t>(L) * static_cast<size_t>(w));
    const Partition& up = uniform_partition(nodes, m);
    const size_t li = static_cast<size_t>(i - 1);
    const double* S = transposed ? f.capinvT[li]->get() : f.capinv[li]->get();
    const double* A = transposed ? f.capT[li]->get() : f.capR[li]->get();
    seg_tn(p, transposed ? f.Wl(i) : f.Fl(i), n, R, Y, ldy, w, Q.get(), R, int(L));
    // Capacitance solve as three batched GEMMs: T = S Q, then one step of
    // refinement Q <- Q - A T, T += S Q. Without the refinement the explicit
    // inverse loses ~2 digits on the C1 parity case (cond(cap) ~ 1e7); with
    // it the result matches the LU substitution of the reference.
    static const int refine = [] {  // HG_CAP_REFINE: refinement steps (tuning/diagnostic knob)
        const char* e = std::getenv("HG_CAP_REFINE");
        return e ? std::max(0, std::atoi(e)) : 1;
    }();
    seg_nn(up, S, L, m, Q.get(), m, int(L), TMap::same(), T.get(), L, w);
    if (refine > 1) {  // keep the right-hand side: every step needs its residual
        DVec Q0(static_cast<size_t>(L) * static_cast<size_t>(w));
        panel_axpby(L, w, 1.0, Q.get(), L, 0.0, Q0.get(), L);
        for (int it = 0; it < refine; ++it) {
            panel_axpby(L, w, 1.0, Q0.get(), L, 0.0, Q.get(), L);
            seg_nn(up, A, L, m, T.get(), m, int(L), TMap::same(), Q.get(), L, w, -1.0, 1.0);
            seg_nn(up, S, L, m, Q.get(), m, int(L), TMap::same(), T.get(), L, w, 1.0, 1.0);
        }
    } else if (refine == 1) {
        seg_nn(up, A, L, m, T.get(), m, int(L), TMap::same(), Q.get(), L, w, -1.0, 1.0);
        seg_nn(up, S, L, m, Q.get(), m, int(L), TMap::same(), T.get(), L, w, 1.0, 1.0);
    }
    if (!transposed)
        seg_nn(p, f.Wl(i), n, R, T.get(), m, int(L), TMap::parent(0, R), Y, ldy, w, -1.0, 1.0);
    else
        seg_nn(p, f.Fl(i), n, R, T.get(), m, int(L), TMap::parent(R, 0), Y, ldy, w, -1.0, 1.0);
}

DFactor factorize(const DHodlr& h, int orient) {
    DFactor f;
    f.tree = h.tree;
    f.orient = orient;
    const int tau = h.tau();
    const i64 n = h.n();
    f.R = h.R;
    f.off.assign(static_cast<size_t>(tau), 0);
    for (int l = 1; l <= tau; ++l) {
        f.off[static_cast<size_t>(l - 1)] = f.sumR;
        f.sumR += f.R[static_cast<size_t>(l - 1)];
    }
    // Source factors (factorization.cpp:75-96): w = upper.left on left-child
    // rows, x = upper.right on right-child rows.
    f.F.assign(static_cast<size_t>(tau), nullptr);
    for (int l = 1; l <= tau; ++l) {
        const int R = f.Rl(l);
        if (!R) continue;
        if (h.sym) {
            f.F[static_cast<size_t>(l - 1)] = h.U[static_cast<size_t>(l - 1)];
        } else {
            auto P = make_dvec(static_cast<size_t>(n) * static_cast<size_t>(R), false);
            const Partition& p = h.tree->part(l);
            panel_parity_select(p, R, h.Ul(l), n, 1.0, h.Vl(l), n, 1.0, P->get(), n);
            f.F[static_cast<size_t>(l - 1)] = P;
        }
    }
    // Leaves (factorization.cpp:68-72).
    const Partition& lv = h.tree->leaves();
    const int nl = lv.nseg(), bm = h.bmax();
    if (bm > MAX_LEAF) throw std::length_error("factorize: leaf size above 320 not supported");
    f.leaf_mat = h.leaves;
    f.leaf_fac = make_dvec(h.leaves->size(), true);
    f.leaf_kind = std::make_shared<DBuf<int>>(static_cast<size_t>(nl));
    f.leaf_piv = std::make_shared<DBuf<int>>(static_cast<size_t>(nl) * static_cast<size_t>(bm));
    f.leaf_ld = make_dvec(static_cast<size_t>(nl), false);
    f.leaf_sign = std::make_shared<DBuf<int>>(static_cast<size_t>(nl));
    {
        const size_t psmem = static_cast<size_t>(bm) * (bm + 1) / 2 * sizeof(double);
        const size_t smem = h.sym && psmem <= SMEM_CAP ? psmem : static_cast<size_t>(bm) * bm * sizeof(double);
        const int use = h.sym && psmem <= SMEM_CAP ? 2 : (smem <= SMEM_CAP ? 1 : 0);
        if (use) set_smem(reinterpret_cast<const void*>(k_leaf_factor), smem);
        LeafFacArgs g{lv.dbounds(), bm, h.leaves->get(), f.leaf_fac->get(), h.sym ? 1 : 0, use,
                      f.leaf_kind->get(), f.leaf_piv->get(), f.leaf_ld->get(), f.leaf_sign->get()};
        k_leaf_factor<<<unsigned(nl), FNT, use ? smem : 0, current().stream>>>(g);
        HG_LAUNCH();
        count_launch();
        const std::vector<int> kinds = f.leaf_kind->download();
        f.all_llt = std::all_of(kinds.begin(), kinds.end(), [](int k) { return k == 1; });
        if (f.all_llt && bm <= TS2_MAX) {  // tensor-core solve path: invert diagonal blocks once
            k_leaf_diag_inv<<<unsigned(nl), 16 * ((bm + 15) / 16), 0, current().stream>>>(lv.dbounds(), bm,
                                                                                          f.leaf_fac->get());
            HG_LAUNCH();
            count_launch();
        }
    }
    // Working left factors (factorization.cpp:75-119): Wbar = Abar^{-1} F.
    f.Wbar = make_dvec(static_cast<size_t>(n) * static_cast<size_t>(std::max(f.sumR, 1)), false);
    for (int l = 1; l <= tau; ++l)
        if (f.Rl(l)) panel_axpby(n, f.Rl(l), 1.0, f.Fl(l), n, 0.0, f.Wl(l), n);
    leaf_solve(f, f.Wbar->get(), n, f.sumR);
    // Levels tau..1 (factorization.cpp:121-166).
    f.cap.assign(static_cast<size_t>(tau), nullptr);
    f.cap_piv.assign(static_cast<size_t>(tau), nullptr);
    f.cap_ld.assign(static_cast<size_t>(tau), nullptr);
    f.cap_sign.assign(static_cast<size_t>(tau), nullptr);
    f.capinv.assign(static_cast<size_t>(tau), nullptr);
    f.capinvT.assign(static_cast<size_t>(tau), nullptr);
    f.capR.assign(static_cast<size_t>(tau), nullptr);
    f.capT.assign(static_cast<size_t>(tau), nullptr);
    for (int i = tau; i >= 1; --i) {
        const int R = f.Rl(i), m = 2 * R, nodes = 1 << (i - 1);
        if (R == 0) continue;
        const Partition& p = h.tree->part(i);
        DVec P(static_cast<size_t>(p.nseg()) * static_cast<size_t>(R) * static_cast<size_t>(R));
        seg_tn(p, f.Fl(i), n, R, f.Wl(i), n, R, P.get(), i64(R) * R, R);
        f.cap[static_cast<size_t>(i - 1)] = make_dvec(static_cast<size_t>(nodes) * static_cast<size_t>(m) * static_cast<size_t>(m), false);
        f.cap_piv[static_cast<size_t>(i - 1)] = std::make_shared<DBuf<int>>(static_cast<size_t>(nodes) * static_cast<size_t>(m));
        f.cap_ld[static_cast<size_t>(i - 1)] = make_dvec(static_cast<size_t>(nodes), false);
        f.cap_sign[static_cast<size_t>(i - 1)] = std::make_shared<DBuf<int>>(static_cast<size_t>(nodes));
        const size_t smem = static_cast<size_t>(m) * m * sizeof(double);
        const int use = smem <= SMEM_CAP ? 1 : 0;
        if (use) set_smem(reinterpret_cast<const void*>(k_cap_lu), smem);
        CapLuArgs g{R, P.get(), f.cap[static_cast<size_t>(i - 1)]->get(), f.cap_piv[static_cast<size_t>(i - 1)]->get(),
                    f.cap_ld[static_cast<size_t>(i - 1)]->get(), f.cap_sign[static_cast<size_t>(i - 1)]->get(), use};
        k_cap_lu<<<unsigned(nodes), FNT, use ? smem : 0, current().stream>>>(g);
        HG_LAUNCH();
        count_launch();
        {  // explicit cap^{-T} by substitution on identity columns, then both panels
            DVec E(static_cast<size_t>(nodes) * static_cast<size_t>(m) * static_cast<size_t>(m));
            cap_solve(f, i, nullptr, false, true, E.get(), m);
            const size_t ps = static_cast<size_t>(nodes) * static_cast<size_t>(m) * static_cast<size_t>(m);
            const size_t li = static_cast<size_t>(i - 1);
            f.capinvT[li] = make_dvec(ps, false);
            f.capinv[li] = make_dvec(ps, false);
            f.capR[li] = make_dvec(ps, false);
            f.capT[li] = make_dvec(ps, false);
            k_cap_panels<<<unsigned(nodes), 256, 0, current().stream>>>(E.get(), P.get(), R, i64(nodes) * m,
                                                                       f.capinv[li]->get(), f.capR[li]->get(),
                                                                       f.capinvT[li]->get(), f.capT[li]->get());
            HG_LAUNCH();
            count_launch();
        }
        if (i > 1 && f.off[static_cast<size_t>(i - 1)] > 0) level_inverse(f, i, false, f.Wbar->get(), n, f.off[static_cast<size_t>(i - 1)]);
    }
    return f;
}

void factor_solve(const DFactor& f, double* Y, i64 ldy, int w) {
    if (f.orient == 0) {
        leaf_solve(f, Y, ldy, w);
        for (int i = f.tau(); i >= 1; --i) level_inverse(f, i, false, Y, ldy, w);
    } else {
        for (int i = 1; i <= f.tau(); ++i) level_inverse(f, i, true, Y, ldy, w);
        leaf_solve(f, Y, ldy, w);
    }
}

double factor_logdet(const DFactor& f) {
    // every (log|det|, sign) array copied back asynchronously, one stream sync
    auto& c = current();
    const int tau = f.tau();
    std::vector<double> lld(f.leaf_ld->size());
    std::vector<int> lsg(f.leaf_sign->size());
    std::vector<std::vector<double>> cl(static_cast<size_t>(tau));
    std::vector<std::vector<int>> cs(static_cast<size_t>(tau));
    auto get = [&](auto& h, const auto& d) {
        if (!h.empty())
            HG_CUDA(cudaMemcpyAsync(h.data(), d.get(), h.size() * sizeof(h[0]), cudaMemcpyDeviceToHost, c.stream));
    };
    get(lld, *f.leaf_ld);
    get(lsg, *f.leaf_sign);
    for (int i = 1; i <= tau; ++i) {
        const size_t li = static_cast<size_t>(i - 1);
        if (!f.cap[li]) continue;
        cl[li].resize(f.cap_ld[li]->size());
        cs[li].resize(f.cap_sign[li]->size());
        get(cl[li], *f.cap_ld[li]);
        get(cs[li], *f.cap_sign[li]);
    }
    HG_CUDA(cudaStreamSynchronize(c.stream));
    double ld = 0.0;
    for (size_t b = 0; b < lld.size(); ++b) {
        if (lsg[b] <= 0) throw NotPositiveDefinite("leaf block has non-positive determinant");
        ld += lld[b];
    }
    for (int i = 1; i <= tau; ++i) {
        const size_t li = static_cast<size_t>(i - 1);
        if (!f.cap[li]) continue;
        for (size_t j = 0; j < cl[li].size(); ++j) {
            if (cs[li][j] <= 0) throw NotPositiveDefinite("capacitance has non-positive determinant");
            ld += cl[li][j];
        }
    }
    return ld;
}

std::vector<int> leaf_kinds(const DFactor& f) { return f.leaf_kind->download(); }

}  // namespace hg
