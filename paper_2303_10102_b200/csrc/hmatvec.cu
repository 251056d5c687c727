// Streaming H-matvec for narrow blocks (s <= 4): Y = beta Y + alpha H_sel X.
//
// Reference: HodlrMatrix::matvec (hodlr_matrix.cpp:198-226); same product as
// hodlr_apply (mlapply.cu), which stays the path for wide blocks where the
// FP64 tensor pipe bounds the work. For s <= 4 the apply is a pure HBM stream
// (arithmetic intensity < 1 flop/B), and the two-pass structure of the
// general path (all projections, then all updates) reads every level panel
// twice. This path reads each panel once plus the LEFT-child half of it a
// second time:
//
//   pass 1 (k_mv_sweep)  one CTA per leaf. For every level l the CTA projects
//       its rows, t = V_l[rows]^T x[rows], and publishes the partial; the
//       last CTA of each group / child folds the partials in a fixed order
//       into T_l[child] (deterministic) and raises the child's ready flag.
//       A leaf in the RIGHT child of its level-l node also needs
//       T_l[left sibling]: it applies U_l[rows] T_l[left] from the same
//       registers the projection used (one read of the rows). Levels are
//       visited in phases — the levels where the leaf is a LEFT child (no
//       waits: publish only), then the leaf block y = L_b x_b, then the
//       levels where it is a RIGHT child (wait for the sibling's flag). A
//       wait therefore only ever depends on other CTAs' first phase, which
//       never waits; leaves are assigned in CTA start order (atomic ticket),
//       so every CTA waited on is resident or retired: no deadlock.
//   pass 2 (k_mv_left)   left-child rows of every level: Y += U_l[rows] T_l[right].
//
// HBM traffic: leaves + panels + half the panels (vs leaves + 2 x panels).
// Every sum runs in an order fixed by the tree, so results are bitwise
// reproducible and independent of the column count s (column c of a batched
// apply equals the apply of that column alone).
#include <cstdint>
#include <type_traits>

#include "hodlr.cuh"
#include "prof.cuh"

namespace hg {

namespace {

constexpr int MV_T = 128;     // threads per CTA
constexpr int MV_MAXL = 24;
constexpr int MV_RMAX = 256;  // widest level the path takes
constexpr int MV_G = 32;      // tier-1 fan-in (chunks folded per group)

struct MvLevel {
    const double* P;  // projection panel (V_l), n x R
    const double* Q;  // update panel (U_l), n x R
    double* ws1;      // nleaves x RS   chunk partials
    double* ws2;      // nleaves/G x RS group partials (children wider than G chunks)
    double* T;        // 2^l x RS       child projections (ld R, S columns)
    int* cnt1;        // nleaves       group counters
    int* cnt2;        // 2^l           child counters
    int* ready;       // 2^l           child flags
    int R, depth;
};

struct MvArgs {
    MvLevel L[MV_MAXL];
    int nl, tau, s;
    i64 n;
    const int* lb;  // leaf bounds (nleaves + 1)
    const double* leaves;  // null => no leaf term
    i64 lstride;
    int bmax;
    const double* X;
    i64 ldx;
    double* Y;
    i64 ldy;
    double alpha, beta;
    int* ticket;
    int dleft;  // pass 2 covers levels of depth <= dleft (deeper ones finish inside a CTA)
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

/// Butterfly transpose-reduce of V values per lane over the warp: V - 1
/// shuffles fold the V independent warp sums into one value per lane; the
/// lane holds the sum of value index lane >> (5 - log2 V) (every lane of the
/// group holds it). Fixed exchange pattern => deterministic.
template <int V>
__device__ __forceinline__ double tr_reduce(double (&v)[V], int lane) {
#pragma unroll
    for (int h = V / 2, m = 16; h >= 1; h >>= 1, m >>= 1) {
        const bool up = (lane & m) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? v[i] : v[i + h];
            const double keep = up ? v[i + h] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, m);
        }
    }
    constexpr int lg = V == 8 ? 3 : V == 16 ? 4 : 5;
#pragma unroll
    for (int m = 16 >> lg; m >= 1; m >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], m);
    return v[0];
}

/// Row k of this thread within the leaf. NT = 64 threads own row pairs
/// (2t, 2t+1: 16-byte loads, half the instructions per byte; t = thread
/// index within its 64-thread leaf group); otherwise rows t + k NT.
template <int NT, int RPT>
__device__ __forceinline__ int mv_row(int k) {
    return NT == 64 ? 2 * int(threadIdx.x & 63) + k : int(threadIdx.x) + k * NT;
}

/// v[k][jj] = P[row_k, j0 + jj] (0 outside the leaf / past R).
template <int NT, int RPT>
__device__ __forceinline__ void load_blk(double (&v)[RPT][8], const double* P, i64 n, int lo, int m, int j0, int R) {
    if constexpr (NT == 64) {
        static_assert(RPT == 2, "row pairs");
        const int r = 2 * int(threadIdx.x & 63);  // 64-thread group per leaf (multi-leaf CTAs)
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const double* p = P + i64(lo) + r + i64(j0 + jj) * n;
            if (j0 + jj < R && r + 1 < m) {
                const double2 d = *reinterpret_cast<const double2*>(p);
                v[0][jj] = d.x;
                v[1][jj] = d.y;
            } else {
                v[0][jj] = (j0 + jj < R && r < m) ? p[0] : 0.0;
                v[1][jj] = 0.0;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const int r = mv_row<NT, RPT>(k);
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
                v[k][jj] = (r < m && j0 + jj < R) ? P[i64(lo) + r + i64(j0 + jj) * n] : 0.0;
        }
    }
}

/// yacc[k][c] += sum_j Q[row_k, j] t[c*R + j]  (t in shared memory).
template <int S, int RPT, int NT>
__device__ __forceinline__ void update(const double* Q, i64 n, int lo, int m, int R, const double* t,
                                       double (&yacc)[RPT][S]) {
    const int nblk = (R + 7) >> 3;
    double a[RPT][8];
    load_blk<NT, RPT>(a, Q, n, lo, m, 0, R);
#pragma unroll 1
    for (int jb = 0; jb < nblk; ++jb) {
        double cur[RPT][8];
#pragma unroll
        for (int k = 0; k < RPT; ++k)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) cur[k][jj] = a[k][jj];
        if (jb + 1 < nblk) load_blk<NT, RPT>(a, Q, n, lo, m, (jb + 1) * 8, R);
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int j = jb * 8 + jj;
            if (j < R) {
#pragma unroll
                for (int c = 0; c < S; ++c) {
                    const double tv = t[c * R + j];
#pragma unroll
                    for (int k = 0; k < RPT; ++k) yacc[k][c] = fma(cur[k][jj], tv, yacc[k][c]);
                }
            }
        }
    }
}

/// Warp-level publish (lanes of one warp; the rest of the CTA runs on): the
/// partial p (RS values, lane-strided in registers of the caller via pv) is
/// stored, and the warp completing a group / the child folds and releases.
template <int S>
__device__ void publish_warp(const MvLevel& L, int tau, int b, int anc, const double* part) {
    const int lane = threadIdx.x & 31;
    const int RS = L.R * S;
    const int nch = 1 << (tau - L.depth);
    auto fold_w = [&](const double* src, int cnt, double* dst) {
        for (int i = lane; i < RS; i += 32) {
            double acc = __ldcg(src + i);
            for (int c = 1; c < cnt; ++c) acc += __ldcg(src + i64(c) * RS + i);
            dst[i] = acc;
        }
    };
    auto release = [&]() {
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release(L.ready + anc, 1);
    };
    if (nch == 1) {
        for (int i = lane; i < RS; i += 32) L.T[i64(anc) * RS + i] = part[i];
        release();
        return;
    }
    const int G = nch < MV_G ? nch : MV_G;
    for (int i = lane; i < RS; i += 32) L.ws1[i64(b) * RS + i] = part[i];
    __threadfence();
    __syncwarp();
    const int grp = b / G;
    int last = lane == 0 ? atomicAdd(L.cnt1 + grp, 1) == G - 1 : 0;
    if (!__shfl_sync(0xffffffffu, last, 0)) return;
    __threadfence();
    if (nch == G) {
        fold_w(L.ws1 + i64(grp) * G * RS, G, L.T + i64(anc) * RS);
        release();
        return;
    }
    fold_w(L.ws1 + i64(grp) * G * RS, G, L.ws2 + i64(grp) * RS);
    __threadfence();
    __syncwarp();
    const int ng = nch / G;
    last = lane == 0 ? atomicAdd(L.cnt2 + anc, 1) == ng - 1 : 0;
    if (!__shfl_sync(0xffffffffu, last, 0)) return;
    __threadfence();
    fold_w(L.ws2 + i64(anc) * ng * RS, ng, L.T + i64(anc) * RS);
    release();
}

/// One level of the sweep for this CTA's rows: projection partial into
/// red (per warp), and for a right child the update with T_l[left sibling]
/// (tv, per-warp shared copy) from the same registers.
template <int S, int RPT, int NT, bool RIGHT>
__device__ __forceinline__ void sweep_level(const MvLevel& L, i64 n, int lo, int m, const double (&x)[RPT][S],
                                            const double* tv, double* red, double (&yacc)[RPT][S]) {
    constexpr int V = 8 * S;
    constexpr int lg = V == 8 ? 3 : V == 16 ? 4 : 5;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int R = L.R, nblk = (R + 7) >> 3;
    double a[RPT][8];
    load_blk<NT, RPT>(a, L.P, n, lo, m, 0, R);
#pragma unroll 1
    for (int jb = 0; jb < nblk; ++jb) {
        double cur[RPT][8];
#pragma unroll
        for (int k = 0; k < RPT; ++k)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) cur[k][jj] = a[k][jj];
        if (jb + 1 < nblk) load_blk<NT, RPT>(a, L.P, n, lo, m, (jb + 1) * 8, R);
        double v[V];
#pragma unroll
        for (int c = 0; c < S; ++c)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                double acc = cur[0][jj] * x[0][c];
#pragma unroll
                for (int k = 1; k < RPT; ++k) acc = fma(cur[k][jj], x[k][c], acc);
                v[c * 8 + jj] = acc;
            }
        if (RIGHT) {  // symmetric storage: U_l rows == V_l rows
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const int j = jb * 8 + jj;
                if (j < R) {
#pragma unroll
                    for (int c = 0; c < S; ++c) {
                        const double tj = tv[c * R + j];
#pragma unroll
                        for (int k = 0; k < RPT; ++k) yacc[k][c] = fma(cur[k][jj], tj, yacc[k][c]);
                    }
                }
            }
        }
        const double sum = tr_reduce<V>(v, lane);
        if ((lane & ((1 << (5 - lg)) - 1)) == 0) {
            const int idx = lane >> (5 - lg), c = idx >> 3, j = jb * 8 + (idx & 7);
            if (j < R) red[warp * (R * S) + c * R + j] = sum;
        }
    }
}

template <int S, int RPT, int NT>
__global__ void __launch_bounds__(NT) k_mv_sweep(const __grid_constant__ MvArgs g) {
    constexpr int NW = NT / 32;
    extern __shared__ double sm[];
    __shared__ int s_ord[MV_MAXL], s_nleft, s_b;
    // leaf = start-order ticket: a CTA only waits on lower tickets, which are resident or retired
    if (threadIdx.x == 0) s_b = atomicAdd(g.ticket, 1);
    __syncthreads();
    const int b = s_b;
    const int lo = g.lb[b], m = g.lb[b + 1] - lo;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int rmax = 0;
    for (int li = 0; li < g.nl; ++li) rmax = max(rmax, g.L[li].R);
    const int RSM = rmax * S;
    double* red = sm;                   // 2 x NW x RSM (double-buffered by level sequence)
    double* part = red + 2 * NW * RSM;  // RSM (warp 0)
    double* tw = part + RSM;            // NW x RSM
    double* xs = tw + NW * RSM;         // bmax x S
    if (threadIdx.x == 0) {  // phase order: left-child levels, then right-child levels
        int k = 0;
        for (int li = 0; li < g.nl; ++li)
            if (!((b >> (g.tau - g.L[li].depth)) & 1)) s_ord[k++] = li;
        s_nleft = k;
        for (int li = 0; li < g.nl; ++li)
            if ((b >> (g.tau - g.L[li].depth)) & 1) s_ord[k++] = li;
    }
    double x[RPT][S], yacc[RPT][S];
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const int r = mv_row<NT, RPT>(k);
#pragma unroll
        for (int c = 0; c < S; ++c) {
            x[k][c] = (r < m && c < g.s) ? g.X[i64(lo) + r + i64(c) * g.ldx] : 0.0;
            yacc[k][c] = 0.0;
            if (r < m) xs[r * S + c] = x[k][c];
        }
    }
    __syncthreads();
    const int nleft = s_nleft;
    for (int i = 0; i <= g.nl; ++i) {
        if (i == nleft && g.leaves) {  // between the phases: y += L_b x_b (leaf column-major, ld bmax)
            const double* Lb = g.leaves + i64(b) * g.lstride;
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                const int r = mv_row<NT, RPT>(k);
                if (r >= m) continue;
                double acc[S];  // (row pairs: the second row's loads hit the first's sectors)
#pragma unroll
                for (int c = 0; c < S; ++c) acc[c] = 0.0;
#pragma unroll 16
                for (int q = 0; q < m; ++q) {
                    const double lv = Lb[r + i64(q) * g.bmax];
#pragma unroll
                    for (int c = 0; c < S; ++c) acc[c] = fma(lv, xs[q * S + c], acc[c]);
                }
#pragma unroll
                for (int c = 0; c < S; ++c) yacc[k][c] += acc[c];
            }
        }
        if (i == g.nl) break;
        const MvLevel& L = g.L[s_ord[i]];
        const int RS = L.R * S;
        const int anc = b >> (g.tau - L.depth);
        double* rb = red + (i & 1) * NW * RSM;
        if (anc & 1) {
            double* tv = tw + warp * RSM;
            if (lane == 0)
                while (ld_acquire(L.ready + (anc ^ 1)) == 0) __nanosleep(32);
            __syncwarp();
            const double* t = L.T + i64(anc ^ 1) * RS;
            for (int q = lane; q < RS; q += 32) tv[q] = __ldcg(t + q);
            __syncwarp();
            sweep_level<S, RPT, NT, true>(L, g.n, lo, m, x, tv, rb, yacc);
        } else {
            sweep_level<S, RPT, NT, false>(L, g.n, lo, m, x, nullptr, rb, yacc);
        }
        __syncthreads();  // rb complete; warp 0 folds and publishes while the others stream on
        if (warp == 0) {
            for (int q = lane; q < RS; q += 32) {
                double acc = rb[q];
#pragma unroll
                for (int w = 1; w < NW; ++w) acc += rb[w * RS + q];
                part[q] = acc;
            }
            __syncwarp();
            publish_warp<S>(L, g.tau, b, anc, part);
        }
    }
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const int r = mv_row<NT, RPT>(k);
        if (r >= m) continue;
#pragma unroll
        for (int c = 0; c < S; ++c) {
            if (c >= g.s) continue;
            double* yp = g.Y + i64(lo) + r + i64(c) * g.ldy;
            *yp = g.beta == 0.0 ? g.alpha * yacc[k][c] : fma(g.alpha, yacc[k][c], g.beta * *yp);
        }
    }
}

/// Multi-leaf sweep (row pairs, LPC leaves per CTA = one node of depth
/// tau - log2 LPC): the levels below that node finish inside the CTA —
/// both children's projections are folded in shared memory and both halves
/// updated (rows re-read from L2) — so neither publication nor the second
/// pass touches them; the levels above behave as in k_mv_sweep with the CTA
/// node as the chunk.
template <int S, int LPC>
__global__ void __launch_bounds__(64 * LPC) k_mv_sweep_multi(const __grid_constant__ MvArgs g) {
    constexpr int NTH = 64 * LPC, NW = NTH / 32;
    constexpr int J = LPC == 2 ? 1 : LPC == 4 ? 2 : 3;
    extern __shared__ double sm[];
    __shared__ int s_ord[MV_MAXL], s_nleft, s_nin, s_b;
    if (threadIdx.x == 0) s_b = atomicAdd(g.ticket, 1);
    __syncthreads();
    const int cta = s_b, tc = g.tau - J;
    const int slot = threadIdx.x >> 6;
    const int b = cta * LPC + slot;
    const int lo = g.lb[b], m = g.lb[b + 1] - lo;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int rmax = 0;
    for (int li = 0; li < g.nl; ++li) rmax = max(rmax, g.L[li].R);
    const int RSM = rmax * S;
    double* red = sm;                    // 2 x NW x RSM
    double* part = red + 2 * NW * RSM;   // RSM (warp 0)
    double* tw = part + RSM;             // NW x RSM
    double* tloc = tw + NW * RSM;        // LPC x RSM (children inside the CTA)
    double* xs = tloc + LPC * RSM;       // LPC x 128 x S
    if (threadIdx.x == 0) {  // order: cross levels as left child, in-CTA levels, cross levels as right child
        int k = 0;
        for (int li = 0; li < g.nl; ++li)
            if (g.L[li].depth <= tc && !((cta >> (tc - g.L[li].depth)) & 1)) s_ord[k++] = li;
        s_nleft = k;
        for (int li = 0; li < g.nl; ++li)
            if (g.L[li].depth > tc) s_ord[k++] = li;
        s_nin = k;
        for (int li = 0; li < g.nl; ++li)
            if (g.L[li].depth <= tc && ((cta >> (tc - g.L[li].depth)) & 1)) s_ord[k++] = li;
    }
    double x[2][S], yacc[2][S];
    double* xl = xs + slot * 128 * S;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int r = mv_row<64, 2>(k);
#pragma unroll
        for (int c = 0; c < S; ++c) {
            x[k][c] = (r < m && c < g.s) ? g.X[i64(lo) + r + i64(c) * g.ldx] : 0.0;
            yacc[k][c] = 0.0;
            if (r < m) xl[r * S + c] = x[k][c];
        }
    }
    __syncthreads();
    const int nleft = s_nleft, nin = s_nin;
    for (int i = 0; i <= g.nl; ++i) {
        if (i == nin && g.leaves) {  // leaf block of this thread's leaf
            const double* Lb = g.leaves + i64(b) * g.lstride;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const int r = mv_row<64, 2>(k);
                if (r >= m) continue;
                double acc[S];
#pragma unroll
                for (int c = 0; c < S; ++c) acc[c] = 0.0;
#pragma unroll 16
                for (int q = 0; q < m; ++q) {
                    const double lv = Lb[r + i64(q) * g.bmax];
#pragma unroll
                    for (int c = 0; c < S; ++c) acc[c] = fma(lv, xl[q * S + c], acc[c]);
                }
#pragma unroll
                for (int c = 0; c < S; ++c) yacc[k][c] += acc[c];
            }
        }
        if (i == g.nl) break;
        const MvLevel& L = g.L[s_ord[i]];
        const int R = L.R, RS = R * S;
        double* rb = red + (i & 1) * NW * RSM;
        if (i >= nleft && i < nin) {  // level inside the CTA node
            sweep_level<S, 2, 64, false>(L, g.n, lo, m, x, nullptr, rb, yacc);
            __syncthreads();
            const int sh = g.tau - L.depth, nch = LPC >> sh, wpc = 2 << sh;  // children, warps per child
            for (int q = threadIdx.x; q < nch * RS; q += NTH) {
                const int c = q / RS, e = q - c * RS;
                double acc = rb[(c * wpc) * RS + e];
                for (int w = 1; w < wpc; ++w) acc += rb[(c * wpc + w) * RS + e];
                tloc[c * RS + e] = acc;
            }
            __syncthreads();
            update<S, 2, 64>(L.Q, g.n, lo, m, R, tloc + ((slot >> sh) ^ 1) * RS, yacc);
            continue;
        }
        const int anc = cta >> (tc - L.depth);
        if (anc & 1) {
            double* tv = tw + warp * RSM;
            if (lane == 0)
                while (ld_acquire(L.ready + (anc ^ 1)) == 0) __nanosleep(32);
            __syncwarp();
            const double* t = L.T + i64(anc ^ 1) * RS;
            for (int q = lane; q < RS; q += 32) tv[q] = __ldcg(t + q);
            __syncwarp();
            sweep_level<S, 2, 64, true>(L, g.n, lo, m, x, tv, rb, yacc);
        } else {
            sweep_level<S, 2, 64, false>(L, g.n, lo, m, x, nullptr, rb, yacc);
        }
        __syncthreads();
        if (warp == 0) {
            for (int q = lane; q < RS; q += 32) {
                double acc = rb[q];
#pragma unroll
                for (int w = 1; w < NW; ++w) acc += rb[w * RS + q];
                part[q] = acc;
            }
            __syncwarp();
            publish_warp<S>(L, tc, cta, anc, part);
        }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int r = mv_row<64, 2>(k);
        if (r >= m) continue;
#pragma unroll
        for (int c = 0; c < S; ++c) {
            if (c >= g.s) continue;
            double* yp = g.Y + i64(lo) + r + i64(c) * g.ldy;
            *yp = g.beta == 0.0 ? g.alpha * yacc[k][c] : fma(g.alpha, yacc[k][c], g.beta * *yp);
        }
    }
}

template <int S, int RPT, int NT>
__global__ void __launch_bounds__(NT) k_mv_left(const __grid_constant__ MvArgs g) {
    extern __shared__ double sm[];
    const int b = blockIdx.x;
    const int lo = g.lb[b], m = g.lb[b + 1] - lo;
    double yacc[RPT][S];
#pragma unroll
    for (int k = 0; k < RPT; ++k)
#pragma unroll
        for (int c = 0; c < S; ++c) yacc[k][c] = 0.0;
    bool any = false;
    for (int li = 0; li < g.nl; ++li) {
        const MvLevel& L = g.L[li];
        const int anc = b >> (g.tau - L.depth);
        if ((anc & 1) || L.depth > g.dleft) continue;
        any = true;
        const int R = L.R;
        const double* t = L.T + i64(anc ^ 1) * R * S;
        for (int i = threadIdx.x; i < R * S; i += NT) sm[i] = t[i];
        __syncthreads();
        update<S, RPT, NT>(L.Q, g.n, lo, m, R, sm, yacc);
        __syncthreads();
    }
    if (!any) return;
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const int r = mv_row<NT, RPT>(k);
        if (r >= m) continue;
#pragma unroll
        for (int c = 0; c < S; ++c)
            if (c < g.s) {
                double* yp = g.Y + i64(lo) + r + i64(c) * g.ldy;
                *yp = fma(g.alpha, yacc[k][c], *yp);
            }
    }
}

/// Pass 2 for the register sweep's shapes: each left level's rows are loaded
/// at once; T of the right sibling is read with warp-uniform (broadcast) loads.
template <int S, int RPT, int NT>
void launch(MvArgs& a, int nleaves, int rmax, int bmax) {
    auto& c = current();
    constexpr int NW = NT / 32;
    const int sm2 = int(sizeof(double)) * (rmax * S > 0 ? rmax * S : 1);
    constexpr int LPC = 4;
    if (NT == 64 && a.tau >= 2) {  // row pairs: 4 leaves per CTA, the two deepest levels finish in-CTA
        constexpr int NTH = 64 * LPC, NWM = NTH / 32;
        const int sm1 = int(sizeof(double)) * ((3 * NWM + 1 + LPC) * rmax * S + LPC * 128 * S);
        static DeviceOnce once;
        if (once.first())
            HG_CUDA(cudaFuncSetAttribute(k_mv_sweep_multi<S, LPC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         100 * 1024));
        a.dleft = a.tau - 2;
        k_mv_sweep_multi<S, LPC><<<unsigned(nleaves / LPC), NTH, size_t(sm1), c.stream>>>(a);
    } else {
        const int sm1 = int(sizeof(double)) * ((3 * NW + 1) * rmax * S + bmax * S);
        static DeviceOnce once;
        if (once.first())
            HG_CUDA(cudaFuncSetAttribute(k_mv_sweep<S, RPT, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         100 * 1024));
        a.dleft = a.tau;
        k_mv_sweep<S, RPT, NT><<<unsigned(nleaves), NT, size_t(sm1), c.stream>>>(a);
    }
    HG_LAUNCH();
    ++c.launches;
    if (a.nl > 0) {
        k_mv_left<S, RPT, NT><<<unsigned(nleaves), NT, size_t(sm2), c.stream>>>(a);
        HG_LAUNCH();
        ++c.launches;
    }
}

}  // namespace

bool hodlr_apply_narrow(const DHodlr& h, const double* X, i64 ldx, int s, double* Y, i64 ldy, int lmin, int lmax,
                        bool with_leaves, bool transpose, double beta, double alpha, ZeroRows zero) {
    if (s < 1 || s > 4 || transpose || zero.bounds) return false;
    const DTree& t = *h.tree;
    const int tau = t.tau();
    const i64 n = h.n();
    if (t.bmax > 2 * MV_T || n >= (i64(1) << 31)) return false;
    lmin = std::max(lmin, 1);
    lmax = std::min(lmax, tau);
    std::vector<int> lv;
    int rmax = 0;
    for (int l = lmin; l <= lmax; ++l)
        if (h.Rl(l) > 0) {
            if (h.Rl(l) > MV_RMAX) return false;
            lv.push_back(l);
            rmax = std::max(rmax, h.Rl(l));
        }
    if (int(lv.size()) > MV_MAXL) return false;
    for (int l : lv)  // the right-child update reuses the projection's rows
        if (h.Ul(l) != h.Vl(l)) return false;
    const int S = s == 1 ? 1 : s == 2 ? 2 : 4;
    const int nleaves = 1 << tau;
    const int nl = int(lv.size());
    // workspaces: counters (zeroed per call) and partial / projection buffers
    DBuf<int> cnt(static_cast<size_t>(1 + 3 * std::max(nl, 1) * nleaves));
    cnt.zero();
    size_t w1 = 0, w2 = 0, wt = 0;
    for (int l : lv) {
        const size_t RS = size_t(h.Rl(l)) * S;
        const int nch = 1 << (tau - l);
        if (nch > 1) w1 += RS * nleaves;
        if (nch > MV_G) w2 += RS * size_t(nleaves / MV_G);
        wt += RS * (size_t(1) << l);
    }
    DVec ws(w1 + w2 + wt);
    MvArgs a{};
    a.nl = nl;
    a.tau = tau;
    a.s = s;
    a.n = n;
    a.lb = t.leaves().dbounds();
    a.leaves = with_leaves && !h.leaves_zero ? h.leaves->get() : nullptr;
    a.lstride = h.lstride();
    a.bmax = t.bmax;
    a.X = X;
    a.ldx = ldx;
    a.Y = Y;
    a.ldy = ldy;
    a.alpha = alpha;
    a.beta = beta;
    a.ticket = cnt.get();

    double* p = ws.get();
    int* ci = cnt.get() + 1;
    double bytes = 8.0 * double(n) * s * (beta != 0.0 ? 3.0 : 2.0), flops = 0;
    if (a.leaves) {
        bytes += 8.0 * double(n) * t.bmax;
        flops += 2.0 * double(n) * s * t.bmax;
    }
    for (int i = 0; i < nl; ++i) {
        const int l = lv[static_cast<size_t>(i)], R = h.Rl(l);
        const size_t RS = size_t(R) * S;
        const int nch = 1 << (tau - l);
        MvLevel& L = a.L[i];
        L.P = h.Vl(l);
        L.Q = h.Ul(l);
        L.R = R;
        L.depth = l;
        L.ws1 = nch > 1 ? p : nullptr;
        p += nch > 1 ? RS * nleaves : 0;
        L.ws2 = nch > MV_G ? p : nullptr;
        p += nch > MV_G ? RS * size_t(nleaves / MV_G) : 0;
        L.T = p;
        p += RS * (size_t(1) << l);
        L.cnt1 = ci;
        L.cnt2 = ci + nleaves;
        L.ready = ci + 2 * nleaves;
        ci += 3 * nleaves;
        bytes += 8.0 * double(n) * R * (h.sym ? 1.0 : 2.0);
        flops += 4.0 * double(n) * R * s;
    }
    ProfScope prof(PROF_MATVEC, flops, bytes);
    if (prof_enabled()) prof.key(prof_tag("hmatvec s=%d Rmax=%d", s, rmax));
    // row pairs (16-byte loads) when every column run is 16-byte aligned
    bool pair = t.bmax <= MV_T && n % 2 == 0;
    for (int v : t.leaves().hbounds()) pair = pair && v % 2 == 0;
    const int mode = t.bmax > MV_T ? 2 : pair ? 1 : 0;
    auto go = [&](auto SS) {
        constexpr int SC = decltype(SS)::value;
        if (mode == 0) launch<SC, 1, 128>(a, nleaves, rmax, t.bmax);
        else if (mode == 1) launch<SC, 2, 64>(a, nleaves, rmax, t.bmax);
        else launch<SC, 2, 128>(a, nleaves, rmax, t.bmax);
    };
    if (S == 1) go(std::integral_constant<int, 1>{});
    else if (S == 2) go(std::integral_constant<int, 2>{});
    else go(std::integral_constant<int, 4>{});
    return true;
}

}  // namespace hg
