// Strong-admissibility H-matrix for grid-stationary covariances (hstrong.cuh).
#include <algorithm>
#include <array>
#include <tuple>
#include <cmath>
#include <cstdlib>
#include <limits>

#include "hstrong.cuh"
#include "prof.cuh"
#include "tile.cuh"

namespace hg {

// ------------------------------------------------------------------ plan
namespace {

struct Box {
    int x0, x1, y0, y1;
};

double periodic_gap(int a0, int a1, int b0, int b1, int N) {
    double best = std::numeric_limits<double>::infinity();
    for (int sh = -N; sh <= N; sh += N) {
        const int g = std::max(0, std::max(b0 + sh - a1, a0 - (b1 + sh)));
        best = std::min(best, double(g));
    }
    return best;
}

}  // namespace

HsPlan hs_plan(const std::int64_t* order, int nside, int tau, double eta, int k) {
    require(nside >= 2, "hstrong: grid side must be >= 2");
    require(eta > 0.0, "hstrong: eta must be positive");
    require(k >= 1 && k <= 64, "hstrong: rank must be in [1, 64]");
    HsPlan P;
    P.n = i64(nside) * nside;
    P.tau = tau;
    P.nside = nside;
    P.eta = eta;
    P.k = k;
    P.tree = ClusterTree(P.n, tau);
    const i64 n = P.n;
    {
        std::vector<char> seen(static_cast<size_t>(n), 0);
        for (i64 i = 0; i < n; ++i) {
            require(order[i] >= 0 && order[i] < n && !seen[static_cast<size_t>(order[i])],
                    "hstrong: order must be a permutation of the grid");
            seen[static_cast<size_t>(order[i])] = 1;
        }
    }
    // bounding boxes of every node (grid-index rectangles of its points)
    std::vector<std::vector<Box>> boxes(static_cast<size_t>(tau) + 1);
    std::vector<std::vector<double>> diam(static_cast<size_t>(tau) + 1);
    for (int d = 0; d <= tau; ++d) {
        const auto& lv = P.tree.level(d);
        auto& bx = boxes[static_cast<size_t>(d)];
        auto& dm = diam[static_cast<size_t>(d)];
        bx.resize(lv.size());
        dm.resize(lv.size());
        for (size_t t = 0; t < lv.size(); ++t) {
            Box b{nside, -1, nside, -1};
            for (i64 i = lv[t].lo; i < lv[t].hi; ++i) {
                const int x = int(order[i] % nside), y = int(order[i] / nside);
                b.x0 = std::min(b.x0, x), b.x1 = std::max(b.x1, x);
                b.y0 = std::min(b.y0, y), b.y1 = std::max(b.y1, y);
            }
            bx[t] = b;
            dm[t] = std::hypot(double(b.x1 - b.x0), double(b.y1 - b.y0));
        }
    }
    auto admissible = [&](int d, int t, int s) {
        const Box& a = boxes[static_cast<size_t>(d)][static_cast<size_t>(t)];
        const Box& b = boxes[static_cast<size_t>(d)][static_cast<size_t>(s)];
        const double dist = std::hypot(periodic_gap(a.x0, a.x1, b.x0, b.x1, nside),
                                       periodic_gap(a.y0, a.y1, b.y0, b.y1, nside));
        const auto& lv = P.tree.level(d);
        const i64 mmin = std::min(lv[static_cast<size_t>(t)].size(), lv[static_cast<size_t>(s)].size());
        return dist > 0.0 && mmin > k &&
               std::min(diam[static_cast<size_t>(d)][static_cast<size_t>(t)],
                        diam[static_cast<size_t>(d)][static_cast<size_t>(s)]) <= eta * dist;
    };
    // recursion over (t, s), t <= s, from (root, root)
    std::vector<std::array<int, 3>> stack{{0, 0, 0}};
    std::vector<HsPlan::Lr> lr;
    std::vector<HsPlan::Dn> dn;
    while (!stack.empty()) {
        const auto [d, t, s] = stack.back();
        stack.pop_back();
        if (t != s && admissible(d, t, s)) {
            lr.push_back({d, t, s});
        } else if (d == tau) {
            dn.push_back({t, s});
        } else if (t == s) {
            stack.push_back({d + 1, 2 * t + 1, 2 * t + 1});
            stack.push_back({d + 1, 2 * t, 2 * t + 1});
            stack.push_back({d + 1, 2 * t, 2 * t});
        } else {
            stack.push_back({d + 1, 2 * t + 1, 2 * s + 1});
            stack.push_back({d + 1, 2 * t + 1, 2 * s});
            stack.push_back({d + 1, 2 * t, 2 * s + 1});
            stack.push_back({d + 1, 2 * t, 2 * s});
        }
    }
    // canonical order: by depth, then (t, s)
    std::sort(lr.begin(), lr.end(), [](const HsPlan::Lr& a, const HsPlan::Lr& b) {
        return std::tie(a.d, a.t, a.s) < std::tie(b.d, b.t, b.s);
    });
    std::sort(dn.begin(), dn.end(),
              [](const HsPlan::Dn& a, const HsPlan::Dn& b) { return std::tie(a.t, a.s) < std::tie(b.t, b.s); });
    P.lr = std::move(lr);
    P.dn = std::move(dn);
    return P;
}

// --------------------------------------------------------------- kernels
namespace {

constexpr int EG_THREADS = 256;

struct EgItem {
    int r_lo, r_m, c_lo, c_m;
    int row0, pad;
    const double* X;  // c_m x k, ld ldx
    i64 ldx;
    double* Y;  // r_m x k, ld ldy
    i64 ldy;
};

__device__ __forceinline__ double grid_entry(const GridEntries& E, int rx, int ry, int cx, int cy) {
    int dx = rx - cx, dy = ry - cy;
    dx += dx < 0 ? E.N : 0;
    dy += dy < 0 ? E.N : 0;
    return __ldg(E.c + i64(dy) * E.N + dx);
}

/// Y[rows row0..row0+TR) = A(r block, c block) X with A's entries generated in
/// shared memory from the generating column (never stored). FP64 FMA,
/// register tile (TR/16) x (KC/16) per thread.
template <int TR, int KC, int KS>
__global__ void __launch_bounds__(EG_THREADS) k_hs_egemm(const EgItem* items, GridEntries E, int k) {
    constexpr int RPT = TR / 16, CPT = KC / 16;
    __shared__ double As[KS][TR];
    __shared__ double Xs[KS][KC];
    __shared__ int Cx[KS], Cy[KS];
    const EgItem it = items[blockIdx.x];
    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    // generation mapping: this thread's row is fixed
    const int grow = tid % TR, jstep = EG_THREADS / TR;
    const bool rvalid = it.row0 + grow < it.r_m;
    const int gi = it.r_lo + it.row0 + (rvalid ? grow : 0);
    const int rx = __ldg(E.gx + gi), ry = __ldg(E.gy + gi);
    double acc[RPT][CPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int c = 0; c < CPT; ++c) acc[r][c] = 0.0;
    for (int j0 = 0; j0 < it.c_m; j0 += KS) {
        if (tid < KS) {
            const int col = it.c_lo + min(j0 + tid, it.c_m - 1);
            Cx[tid] = __ldg(E.gx + col);
            Cy[tid] = __ldg(E.gy + col);
        }
        for (int e = tid; e < KS * KC; e += EG_THREADS) {
            const int jj = e & (KS - 1), cc = e / KS;
            Xs[jj][cc] = (j0 + jj < it.c_m && cc < k) ? it.X[i64(j0 + jj) + i64(cc) * it.ldx] : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int jj = tid / TR; jj < KS; jj += jstep)
            As[jj][grow] = (rvalid && j0 + jj < it.c_m) ? grid_entry(E, rx, ry, Cx[jj], Cy[jj]) : 0.0;
        __syncthreads();
#pragma unroll 4
        for (int jj = 0; jj < KS; ++jj) {
            double a[RPT], b[CPT];
#pragma unroll
            for (int r = 0; r < RPT; ++r) a[r] = As[jj][ty + 16 * r];
#pragma unroll
            for (int c = 0; c < CPT; ++c) b[c] = Xs[jj][tx + 16 * c];
#pragma unroll
            for (int r = 0; r < RPT; ++r)
#pragma unroll
                for (int c = 0; c < CPT; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int row = it.row0 + ty + 16 * r;
        if (row >= it.r_m) continue;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            const int col = tx + 16 * c;
            if (col < k) it.Y[i64(row) + i64(col) * it.ldy] = acc[r][c];
        }
    }
}

/// The same product on the FP64 tensor cores: a 64 x TBN tile per CTA (4
/// warps, tile.cuh), K = the block's columns in slices of 16. The A slice
/// (64 rows x 16 generated entries) is produced one slice ahead: the gathers
/// from the generating column are issued before the current slice's DMMA work
/// and stored to the other shared buffer after it; X slices arrive by
/// cp.async. (The FMA kernel above is bound by shared-memory bandwidth:
/// 11 loads per 24 FMAs; a DMMA fragment feeds 16x more FMAs per load.)
template <int TBN>
__global__ void __launch_bounds__(tile::THREADS) k_hs_egemm_tc(const EgItem* items, GridEntries E, int k) {
    constexpr int TBM = 64, BK = tile::BK, AE = tile::stage_elems(TBM), BE = tile::stage_elems(TBN);
    constexpr int LDA = TBM + 4;  // MC layout: element (m, kk) at [kk * LDA + m]
    constexpr int EPT = TBM * BK / tile::THREADS;  // generated entries per thread and slice (8)
    __shared__ double As[2][AE];
    __shared__ double Xs[2][BE];
    const EgItem it = items[blockIdx.x];
    const int tid = threadIdx.x, m = tid % TBM, kk0 = tid / TBM;  // this thread's row, first slice column
    const bool rvalid = it.row0 + m < it.r_m;
    const int gi = it.r_lo + it.row0 + (rvalid ? m : 0);
    const int rx = __ldg(E.gx + gi), ry = __ldg(E.gy + gi);
    const int ktiles = (it.c_m + BK - 1) / BK;
    double ent[EPT];
    auto gen = [&](int kt) {
#pragma unroll
        for (int q = 0; q < EPT; ++q) {
            const int j = kt * BK + kk0 + (tile::THREADS / TBM) * q;
            double v = 0.0;
            if (rvalid && j < it.c_m) {
                const int col = it.c_lo + j;
                v = grid_entry(E, rx, ry, __ldg(E.gx + col), __ldg(E.gy + col));
            }
            ent[q] = v;
        }
    };
    auto put = [&](int buf) {
#pragma unroll
        for (int q = 0; q < EPT; ++q) As[buf][(kk0 + (tile::THREADS / TBM) * q) * LDA + m] = ent[q];
    };
    tile::LoadKCT<TBN> lx{it.X, it.ldx, it.c_m, k};
    typename tile::Shape<TBM, TBN>::Acc acc;
    acc.zero();
    gen(0);
    lx.issue(Xs[0], 0);
    tile::cp_commit();
    put(0);
    for (int kt = 0; kt < ktiles; ++kt) {
        const int buf = kt & 1;
        if (kt + 1 < ktiles) {
            lx.issue(Xs[buf ^ 1], kt + 1);  // the other buffers were last read in slice kt - 1 (barrier below)
            gen(kt + 1);                    // gathers in flight during this slice's DMMA work
        }
        tile::cp_commit();
        tile::cp_wait<1>();
        __syncthreads();  // slice kt: X landed, A stored by every thread
        tile::mma_stage<false, true, TBM, TBN>(As[buf], Xs[buf], acc);
        if (kt + 1 < ktiles) put(buf ^ 1);
        __syncthreads();  // every warp is done with slice kt's buffers; slice kt + 1's A is stored
    }
    tile::cp_wait<0>();
    tile::for_each_t<TBM, TBN>(acc, [&](int mi, int ci, double v) {
        const int row = it.row0 + mi;
        if (row < it.r_m && ci < k) it.Y[i64(row) + i64(ci) * it.ldy] = v;
    });
}

struct DnItem {
    int t_lo, t_m, s_lo, s_m;
    double* D;   // t_m x s_m
    double* DT;  // s_m x t_m exact transpose (off-diagonal blocks), or null
};

/// Dense near-field blocks from the generating column; off-diagonal blocks
/// also get their exact transpose (so every matvec read is coalesced).
__global__ void __launch_bounds__(256) k_hs_dense_fill(const DnItem* items, GridEntries E) {
    __shared__ double S[32][33];
    const DnItem it = items[blockIdx.x];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int tj = 0; tj < it.s_m; tj += 32)
        for (int ti = 0; ti < it.t_m; ti += 32) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int i = ti + tx, j = tj + ty + 8 * r;
                double v = 0.0;
                if (i < it.t_m && j < it.s_m) {
                    const int a = it.t_lo + i, b = it.s_lo + j;
                    v = grid_entry(E, __ldg(E.gx + a), __ldg(E.gy + a), __ldg(E.gx + b), __ldg(E.gy + b));
                    it.D[i + i64(j) * it.t_m] = v;
                }
                S[ty + 8 * r][tx] = v;
            }
            if (!it.DT) continue;
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int jj = tj + tx, ii = ti + ty + 8 * r;  // DT(jj, ii) = D(ii, jj)
                if (jj < it.s_m && ii < it.t_m) it.DT[jj + i64(ii) * it.s_m] = S[tx][ty + 8 * r];
            }
            __syncthreads();
        }
}

__device__ __forceinline__ std::uint64_t splitmix64(std::uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/// Gaussian sketch entries, a pure function of (seed, flat index).
__global__ void k_hs_gauss(double* O, i64 total, std::uint64_t seed) {
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) {
        const std::uint64_t h1 = splitmix64(seed ^ (std::uint64_t(e) * 2 + 0x5851F42D4C957F2Dull));
        const std::uint64_t h2 = splitmix64(h1 ^ 0xD1B54A32D192ED03ull);
        const double u1 = (double(h1 >> 11) + 1.0) * 0x1.0p-53, u2 = double(h2 >> 11) * 0x1.0p-53;
        O[e] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
}

constexpr int PJ_ROWS = 32, PJ_CS = 16;

/// partials[part] (k x s, ld k; columns of this CTA's 16-column chunk) = M[rows]^T X[rows].
__global__ void __launch_bounds__(256) k_hs_proj(const DHStrong::ProjItem* items, const double* Xc, i64 ldxc, int k,
                                                 int s, double* partials) {
    __shared__ double Ms[PJ_ROWS][65];
    __shared__ double Xs[PJ_ROWS][PJ_CS];
    const DHStrong::ProjItem it = items[blockIdx.x];
    const int c0 = blockIdx.y * PJ_CS, tid = threadIdx.x, a = tid & 63, cg = tid >> 6;
    const double* X = it.X ? it.X : Xc;
    const i64 ldx = it.X ? it.ldx : ldxc;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r0 = 0; r0 < it.rows; r0 += PJ_ROWS) {
        for (int e = tid; e < PJ_ROWS * 64; e += 256) {
            const int rr = e & (PJ_ROWS - 1), aa = e / PJ_ROWS;
            Ms[rr][aa] = (r0 + rr < it.rows && aa < k) ? it.M[i64(r0 + rr) + i64(aa) * it.ldm] : 0.0;
        }
        for (int e = tid; e < PJ_ROWS * PJ_CS; e += 256) {
            const int rr = e & (PJ_ROWS - 1), cc = e / PJ_ROWS;
            Xs[rr][cc] = (r0 + rr < it.rows && c0 + cc < s) ? X[it.xoff + r0 + rr + i64(c0 + cc) * ldx] : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int rr = 0; rr < PJ_ROWS; ++rr) {
            const double m = Ms[rr][a];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] = fma(m, Xs[rr][cg * 4 + j], acc[j]);
        }
        __syncthreads();
    }
    if (a < k)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = c0 + cg * 4 + j;
            if (col < s) partials[i64(it.part) * k * s + a + i64(col) * k] = acc[j];
        }
}

/// P[slot] = sum of its partials, in order (deterministic).
__global__ void k_hs_reduce(const int* first, int nslots, const double* partials, int k, int s, double* P) {
    const i64 ks = i64(k) * s, tot = i64(nslots) * ks;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += i64(gridDim.x) * blockDim.x) {
        const int slot = int(e / ks);
        const i64 w = e % ks;
        double acc = 0.0;
        for (int p = first[slot]; p < first[slot + 1]; ++p) acc += partials[i64(p) * ks + w];
        P[e] = acc;
    }
}

constexpr int UP_ROWS = 64;

/// Y[tile rows, c0 .. c0+CS) = sum over the tile's contributions of
/// M(rows, :) R, R a projection slot (k x s) or rows of X (dense blocks).
/// One CTA per (64-row tile, CS-column chunk); the contributions are dealt
/// round-robin to the 8 warps, each warp streams its panels with no barrier
/// (lane = rows l and l + 32; R broadcast), and the warps' partial sums are
/// combined in a fixed tree order at the end (deterministic, no atomics).
template <int CS>
__global__ void __launch_bounds__(256) k_hs_update(const DHStrong::Tile* tiles, const DHStrong::Contrib* contrib,
                                                   const double* P, const double* X, i64 ldx, int k, int s, double* Y,
                                                   i64 ldy) {
    __shared__ double red[4][UP_ROWS][CS];
    const DHStrong::Tile tl = tiles[blockIdx.x];
    const int c0 = blockIdx.y * CS, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nc = min(CS, s - c0);
    const bool v0 = lane < tl.rows, v1 = lane + 32 < tl.rows;
    double acc0[CS], acc1[CS];
#pragma unroll
    for (int c = 0; c < CS; ++c) acc0[c] = acc1[c] = 0.0;
    for (int ci = tl.cfirst + w; ci < tl.clast; ci += 8) {
        const DHStrong::Contrib C = contrib[ci];
        const double* M0 = C.M + C.moff + tl.rin + lane;
        const double* R = C.rkind == 0 ? P + (C.ridx * s + c0) * i64(k) : X + C.ridx + i64(c0) * ldx;
        const i64 ldr = C.rkind == 0 ? i64(k) : ldx;
#pragma unroll 4
        for (int kk = 0; kk < C.K; ++kk) {
            const double m0 = v0 ? __ldcs(M0 + i64(kk) * C.ldm) : 0.0;
            const double m1 = v1 ? __ldcs(M0 + 32 + i64(kk) * C.ldm) : 0.0;
#pragma unroll
            for (int c = 0; c < CS; ++c) {
                const double r = c < nc ? __ldg(R + kk + c * ldr) : 0.0;
                acc0[c] = fma(m0, r, acc0[c]);
                acc1[c] = fma(m1, r, acc1[c]);
            }
        }
    }
    // fixed-order tree over the warps: 4..7 -> 0..3, 2..3 -> 0..1, 1 -> 0
    for (int half = 4; half >= 1; half >>= 1) {
        if (w >= half && w < 2 * half)
#pragma unroll
            for (int c = 0; c < CS; ++c) {
                red[w - half][lane][c] = acc0[c];
                red[w - half][lane + 32][c] = acc1[c];
            }
        __syncthreads();
        if (w < half)
#pragma unroll
            for (int c = 0; c < CS; ++c) {
                acc0[c] += red[w][lane][c];
                acc1[c] += red[w][lane + 32][c];
            }
        __syncthreads();
    }
    if (w == 0)
#pragma unroll
        for (int c = 0; c < CS; ++c) {
            if (c >= nc) break;
            if (v0) Y[tl.row0 + lane + i64(c0 + c) * ldy] = acc0[c];
            if (v1) Y[tl.row0 + lane + 32 + i64(c0 + c) * ldy] = acc1[c];
        }
}

constexpr int UT_K = 32, UT_CS = 16;

/// Wide blocks (s > 4): the same sum with the panels staged through shared
/// memory, a 64 x 16 output tile per CTA (one thread per row and 4 columns).
__global__ void __launch_bounds__(256) k_hs_update_tiled(const DHStrong::Tile* tiles, const DHStrong::Contrib* contrib,
                                                         const double* P, const double* X, i64 ldx, int k, int s,
                                                         double* Y, i64 ldy) {
    __shared__ double Ms[UP_ROWS][UT_K + 1];
    __shared__ double Rs[UT_K][UT_CS];
    const DHStrong::Tile tl = tiles[blockIdx.x];
    const int c0 = blockIdx.y * UT_CS, tid = threadIdx.x, r = tid & 63, cg = tid >> 6;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int ci = tl.cfirst; ci < tl.clast; ++ci) {
        const DHStrong::Contrib C = contrib[ci];
        for (int kk0 = 0; kk0 < C.K; kk0 += UT_K) {
            const int kc = min(UT_K, C.K - kk0);
            for (int e = tid; e < UP_ROWS * UT_K; e += 256) {
                const int rr = e & 63, kk = e >> 6;
                Ms[rr][kk] = (rr < tl.rows && kk < kc) ? C.M[C.moff + tl.rin + rr + i64(kk0 + kk) * C.ldm] : 0.0;
            }
            for (int e = tid; e < UT_K * UT_CS; e += 256) {
                const int kk = e & 31, cc = e >> 5;
                double v = 0.0;
                if (kk < kc && c0 + cc < s)
                    v = C.rkind == 0 ? P[(C.ridx * s + (c0 + cc)) * i64(k) + kk0 + kk]
                                     : X[C.ridx + kk0 + kk + i64(c0 + cc) * ldx];
                Rs[kk][cc] = v;
            }
            __syncthreads();
            for (int kk = 0; kk < kc; ++kk) {
                const double m = Ms[r][kk];
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[j] = fma(m, Rs[kk][cg * 4 + j], acc[j]);
            }
            __syncthreads();
        }
    }
    if (r < tl.rows)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int col = c0 + cg * 4 + j;
            if (col < s) Y[tl.row0 + r + i64(col) * ldy] = acc[j];
        }
}

// ---- wide blocks (s > 4): both passes on the FP64 tensor cores (tile.cuh)

/// partials[part] (k x s, ld k) = M[rows]^T X[rows]: one TBM x TBN DMMA tile
/// per (projection chunk, column chunk); both operands k-contiguous (rows are
/// the reduction index).
template <int TBM, int TBN>
__global__ void __launch_bounds__(tile::THREADS) k_hs_proj_tc(const DHStrong::ProjItem* items, const double* Xc,
                                                              i64 ldxc, int k, int s, double* partials) {
    extern __shared__ double smem[];
    const DHStrong::ProjItem it = items[blockIdx.x];
    const int c0 = blockIdx.y * TBN;
    const double* X = it.X ? it.X : Xc;
    const i64 ldx = it.X ? it.ldx : ldxc;
    tile::LoadKCT<TBM> la{it.M, it.ldm, it.rows, k};
    tile::LoadKCT<TBN> lb{X + it.xoff + i64(c0) * ldx, ldx, it.rows, s - c0};
    typename tile::Shape<TBM, TBN>::Acc acc;
    acc.zero();
    tile::run_t<tile::STAGES, TBM, TBN>(la, lb, (it.rows + tile::BK - 1) / tile::BK, smem, acc);
    double* o = partials + i64(it.part) * k * s;
    tile::for_each_t<TBM, TBN>(acc, [&](int a, int ci, double v) {
        const int col = c0 + ci;
        if (a < k && col < s) o[a + i64(col) * k] = v;
    });
}

constexpr int UTC_MAXC = 1024;  // contributions of one leaf staged in shared memory

/// Y[64-row tile, TBN columns] = sum over the tile's contributions of
/// M(rows, :) R: ONE GEMM whose K runs over the concatenated contributions
/// (each padded to whole 16-slices by the loaders' zero fill), the panels
/// streamed through the cp.async pipeline; fixed order (deterministic).
template <int TBN>
__global__ void __launch_bounds__(tile::THREADS) k_hs_update_tc(const DHStrong::Tile* tiles,
                                                                const DHStrong::Contrib* contrib, const double* P,
                                                                const double* X, i64 ldx, int k, int s, double* Y,
                                                                i64 ldy) {
    constexpr int TBM = UP_ROWS, NS = tile::STAGES, BK = tile::BK;
    constexpr int AE = tile::stage_elems(TBM), BE = tile::stage_elems(TBN);
    extern __shared__ double smem[];
    __shared__ int pref[UTC_MAXC + 1];
    const DHStrong::Tile tl = tiles[blockIdx.x];
    const int c0 = blockIdx.y * TBN, nc = tl.clast - tl.cfirst;
    if (threadIdx.x == 0) {  // K-slice prefix of the contributions
        int acc = 0;
        for (int i = 0; i < nc; ++i) {
            pref[i] = acc;
            acc += (contrib[tl.cfirst + i].K + BK - 1) / BK;
        }
        pref[nc] = acc;
    }
    __syncthreads();
    const int ktiles = pref[nc];
    double* As = smem;
    double* Bs = smem + NS * AE;
    int cur = 0;
    auto issue = [&](int stage, int vt) {  // vt increases from call to call
        while (vt >= pref[cur + 1]) ++cur;
        const DHStrong::Contrib C = contrib[tl.cfirst + cur];
        const int kt = vt - pref[cur];
        tile::LoadMCT<TBM> la{C.M + C.moff + tl.rin, C.ldm, tl.rows, C.K};
        la.issue(As + stage * AE, kt);
        const bool lowrank = C.rkind == 0;
        tile::LoadKCT<TBN> lb{lowrank ? P + (C.ridx * s + c0) * i64(k) : X + C.ridx + i64(c0) * ldx,
                              lowrank ? i64(k) : ldx, C.K, s - c0};
        lb.issue(Bs + stage * BE, kt);
    };
    typename tile::Shape<TBM, TBN>::Acc acc;
    acc.zero();
#pragma unroll
    for (int st = 0; st < NS - 1; ++st) {
        if (st < ktiles) issue(st, st);
        tile::cp_commit();
    }
    for (int kt = 0; kt < ktiles; ++kt) {
        tile::cp_wait<NS - 2>();
        __syncthreads();
        const int nk = kt + NS - 1;
        if (nk < ktiles) issue(nk % NS, nk);
        tile::cp_commit();
        const int st = kt % NS;
        tile::mma_stage<false, true, TBM, TBN>(As + st * AE, Bs + st * BE, acc);
    }
    tile::cp_wait<0>();
    tile::for_each_t<TBM, TBN>(acc, [&](int r, int ci, double v) {
        const int col = c0 + ci;
        if (r < tl.rows && col < s) Y[tl.row0 + r + i64(col) * ldy] = v;
    });
}

struct DotItem {
    const double* A;
    const double* B;
    i64 len;
    double w;
};

/// partial[b] = w_b sum(A_b .* B_b), fixed-order block reduction.
__global__ void k_hs_block_dot(const DotItem* items, double* partial) {
    __shared__ double red[256];
    const DotItem it = items[blockIdx.x];
    double acc = 0.0;
    for (i64 e = threadIdx.x; e < it.len; e += blockDim.x) acc = fma(it.A[e], it.B[e], acc);
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if (int(threadIdx.x) < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = it.w * red[0];
}

__global__ void k_hs_sum(const double* partial, int m, double* out) {
    __shared__ double red[256];
    double acc = 0.0;
    for (int e = threadIdx.x; e < m; e += blockDim.x) acc += partial[e];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
        if (int(threadIdx.x) < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = red[0];
}

int blocks_for(i64 tot) { return int(std::max<i64>(1, std::min<i64>((tot + 255) / 256, 148 * 16))); }

/// Launch the entry-generated products Y_b = A(r_b, c_b) X_b of a batch.
void egemm(const std::vector<EgItem>& blocks, const GridEntries& E, int k, double flops_per_entry) {
    if (blocks.empty()) return;
    auto& c = current();
    static const bool use_tc = [] {  // HG_HS_EGEMM_TC=0: the FMA kernel
        const char* e = std::getenv("HG_HS_EGEMM_TC");
        return !(e && e[0] == '0');
    }();
    int minrows = 1 << 30;
    for (const auto& b : blocks) minrows = std::min(minrows, b.r_m);
    const int TR = (!use_tc && minrows >= 128) ? 128 : 64;
    std::vector<EgItem> items;
    double entries = 0.0;
    for (const auto& b : blocks) {
        for (int r0 = 0; r0 < b.r_m; r0 += TR) {
            EgItem it = b;
            it.row0 = r0;
            items.push_back(it);
        }
        entries += double(b.r_m) * b.c_m;
    }
    DBuf<EgItem> d;
    d.upload(items);
    const int KC = k <= 48 ? 48 : 64;
    ProfScope prof(PROF_ORACLE, 2.0 * entries * k * flops_per_entry, 8.0 * entries / TR * KC);
    if (prof_enabled()) prof.key(prof_tag("hs_egemm k=%d items=%d", k, int(items.size())));
    const unsigned g = unsigned(items.size());
    if (use_tc) {
        if (k <= 32)
            k_hs_egemm_tc<32><<<g, tile::THREADS, 0, c.stream>>>(d.get(), E, k);
        else if (k <= 48)
            k_hs_egemm_tc<48><<<g, tile::THREADS, 0, c.stream>>>(d.get(), E, k);
        else
            k_hs_egemm_tc<64><<<g, tile::THREADS, 0, c.stream>>>(d.get(), E, k);
        HG_LAUNCH();
        ++c.launches;
        return;
    }
    // inner slice KS: 32 columns, 16 where 32 would exceed 48 KB of static shared memory
    if (TR == 128 && KC == 48) k_hs_egemm<128, 48, 32><<<g, EG_THREADS, 0, c.stream>>>(d.get(), E, k);
    else if (TR == 128) k_hs_egemm<128, 64, 16><<<g, EG_THREADS, 0, c.stream>>>(d.get(), E, k);
    else if (KC == 48) k_hs_egemm<64, 48, 32><<<g, EG_THREADS, 0, c.stream>>>(d.get(), E, k);
    else k_hs_egemm<64, 64, 32><<<g, EG_THREADS, 0, c.stream>>>(d.get(), E, k);
    HG_LAUNCH();
    ++c.launches;
}

/// Orthonormal basis (thin Q, k columns) of every Y_b, written to Q_b.
void orth(const std::vector<double*>& Y, const std::vector<int>& rows, const std::vector<double*>& Q, int k) {
    std::vector<BatchedQR::Block> blocks;
    std::vector<i64> ldq;
    for (size_t b = 0; b < Y.size(); ++b) {
        blocks.push_back({Y[b], i64(rows[b]), rows[b]});
        ldq.push_back(rows[b]);
    }
    BatchedQR qr(blocks, k, false);
    qr.form_q(k, nullptr, 0, 0, Q, ldq);
}

}  // namespace

// ------------------------------------------------------------------ build
DHStrong hs_build(const DOracle& o, int param, const std::int64_t* order, int nside, int tau, double eta, int k,
                  int power_iters, std::uint64_t seed) {
    require(power_iters >= 0 && power_iters <= 8, "hstrong: power_iters must be in [0, 8]");
    DHStrong h;
    h.plan = hs_plan(order, nside, tau, eta, k);
    const HsPlan& P = h.plan;
    const i64 n = P.n;
    require(o.dim() == n, "hstrong: oracle dimension does not match the grid");
    require(param >= -1 && param < o.num_params(), "hstrong: parameter index");
    auto& c = current();
    // grid coordinates per row
    std::vector<int> hx(static_cast<size_t>(n)), hy(static_cast<size_t>(n));
    std::vector<i64> row_of(static_cast<size_t>(n));
    for (i64 i = 0; i < n; ++i) {
        hx[static_cast<size_t>(i)] = int(order[i] % nside);
        hy[static_cast<size_t>(i)] = int(order[i] / nside);
        row_of[static_cast<size_t>(order[i])] = i;
    }
    DBuf<int> gx, gy;
    gx.upload(hx);
    gy.upload(hy);
    // generating column: one apply of the operator to two unit vectors (grid
    // points 0 and g1); the second checks translation invariance
    const int g1x = nside / 2 + 1 < nside ? nside / 2 + 1 : 0, g1y = nside / 3;
    const i64 i0 = row_of[0], i1 = row_of[static_cast<size_t>(i64(g1y) * nside + g1x)];
    std::vector<double> he(static_cast<size_t>(2 * n), 0.0);
    he[static_cast<size_t>(i0)] = 1.0;
    he[static_cast<size_t>(n + i1)] = 1.0;
    DVec e, y(static_cast<size_t>(2 * n));
    e.upload(he);
    o.apply(param, e.get(), n, 2, y.get(), n);
    const std::vector<double> hy2 = y.download();
    std::vector<double> cg(static_cast<size_t>(n));
    double cmax = 0.0;
    for (i64 i = 0; i < n; ++i) {
        cg[static_cast<size_t>(order[i])] = hy2[static_cast<size_t>(i)];
        cmax = std::max(cmax, std::fabs(hy2[static_cast<size_t>(i)]));
    }
    double dev = 0.0;
    for (i64 i = 0; i < n; ++i) {
        int dx = hx[static_cast<size_t>(i)] - g1x, dy = hy[static_cast<size_t>(i)] - g1y;
        dx += dx < 0 ? nside : 0;
        dy += dy < 0 ? nside : 0;
        dev = std::max(dev, std::fabs(hy2[static_cast<size_t>(n + i)] - cg[static_cast<size_t>(i64(dy) * nside + dx)]));
    }
    if (!(dev <= 1e-10 * cmax + 1e-300))
        throw std::invalid_argument("hstrong: the oracle is not translation invariant on the grid (max deviation " +
                                    std::to_string(dev / std::max(cmax, 1e-300)) + " of max|c|)");
    DVec cgrid;
    cgrid.upload(cg);
    const GridEntries E{cgrid.get(), gx.get(), gy.get(), nside};
    // storage
    const auto range = [&](int d, int t) { return P.tree.level(d)[static_cast<size_t>(t)]; };
    i64 nu = 0, nv = 0, nd = 0;
    for (const auto& b : P.lr) {
        h.uoff.push_back(nu);
        h.voff.push_back(nv);
        nu += range(b.d, b.t).size() * k;
        nv += range(b.d, b.s).size() * k;
    }
    for (const auto& b : P.dn) {  // D, then (off-diagonal) its transpose
        h.doff.push_back(nd);
        nd += range(P.tau, b.t).size() * range(P.tau, b.s).size() * (b.t == b.s ? 1 : 2);
    }
    h.U.alloc(static_cast<size_t>(nu));
    h.V.alloc(static_cast<size_t>(nv));
    h.D.alloc(static_cast<size_t>(nd));
    // dense blocks
    if (!P.dn.empty()) {
        std::vector<DnItem> di;
        for (size_t b = 0; b < P.dn.size(); ++b) {
            const Range t = range(P.tau, P.dn[b].t), s = range(P.tau, P.dn[b].s);
            double* D = h.D.get() + h.doff[b];
            di.push_back({int(t.lo), int(t.size()), int(s.lo), int(s.size()), D,
                          P.dn[b].t == P.dn[b].s ? nullptr : D + t.size() * s.size()});
        }
        DBuf<DnItem> dd;
        dd.upload(di);
        ProfScope prof(PROF_ORACLE, 0.0, 8.0 * double(nd));
        k_hs_dense_fill<<<unsigned(di.size()), 256, 0, c.stream>>>(dd.get(), E);
        HG_LAUNCH();
        ++c.launches;
    }
    // low-rank blocks: batched randomized range finder over every admissible pair
    if (!P.lr.empty()) {
        DVec Om(static_cast<size_t>(nv)), Yb(static_cast<size_t>(nu));
        k_hs_gauss<<<blocks_for(nv), 256, 0, c.stream>>>(Om.get(), nv, seed);
        HG_LAUNCH();
        ++c.launches;
        std::vector<EgItem> fwd, bwd;  // A X (rows t) and A^T X (rows s)
        std::vector<double*> yb, ub, ob, vb;
        std::vector<int> tr, sr;
        for (size_t b = 0; b < P.lr.size(); ++b) {
            const Range t = range(P.lr[b].d, P.lr[b].t), s = range(P.lr[b].d, P.lr[b].s);
            yb.push_back(Yb.get() + h.uoff[b]);
            ub.push_back(h.U.get() + h.uoff[b]);
            ob.push_back(Om.get() + h.voff[b]);
            vb.push_back(h.V.get() + h.voff[b]);
            tr.push_back(int(t.size()));
            sr.push_back(int(s.size()));
        }
        auto products = [&](bool forward, const std::vector<double*>& X, const std::vector<double*>& Yo) {
            std::vector<EgItem> it;
            for (size_t b = 0; b < P.lr.size(); ++b) {
                const Range t = range(P.lr[b].d, P.lr[b].t), s = range(P.lr[b].d, P.lr[b].s);
                const Range r = forward ? t : s, q = forward ? s : t;
                it.push_back({int(r.lo), int(r.size()), int(q.lo), int(q.size()), 0, 0, X[b], q.size(), Yo[b],
                              r.size()});
            }
            egemm(it, E, k, 1.0);
        };
        products(true, ob, yb);  // Y = A Omega
        for (int q = 0; q < power_iters; ++q) {
            orth(yb, tr, ub, k);       // U <- orth(Y)
            products(false, ub, ob);   // Z = A^T U (into Omega)
            orth(ob, sr, vb, k);       // V <- orth(Z)
            products(true, vb, yb);    // Y = A V
        }
        orth(yb, tr, ub, k);       // U = orth(Y)
        products(false, ub, vb);   // V = A^T U: block = U V^T
    }
    // ---- apply work lists
    const int nlr = int(P.lr.size());
    std::vector<DHStrong::ProjItem> pj;
    constexpr int PCH = 2048;
    h.slot_first.assign(static_cast<size_t>(2 * nlr + 1), 0);
    int part = 0;
    for (int b = 0; b < nlr; ++b) {
        const Range t = range(P.lr[b].d, P.lr[b].t), s = range(P.lr[b].d, P.lr[b].s);
        for (int side = 0; side < 2; ++side) {  // slot 2b: U^T X_t, slot 2b+1: V^T X_s
            h.slot_first[static_cast<size_t>(2 * b + side)] = part;
            const Range r = side == 0 ? t : s;
            const double* M = side == 0 ? h.U.get() + h.uoff[b] : h.V.get() + h.voff[b];
            for (i64 r0 = 0; r0 < r.size(); r0 += PCH)
                pj.push_back({M + r0, r.size(), nullptr, r.lo + r0, 0, int(std::min<i64>(PCH, r.size() - r0)), part++});
        }
    }
    h.slot_first[static_cast<size_t>(2 * nlr)] = part;
    h.nparts = part;
    h.proj.upload(pj);
    h.dslot_first.upload(h.slot_first);
    const int nleaves = int(P.tree.num_leaves());
    std::vector<std::vector<DHStrong::Contrib>> per(static_cast<size_t>(nleaves));
    for (int b = 0; b < nlr; ++b) {
        const int d = P.lr[b].d, sh = P.tau - d;
        const Range t = range(d, P.lr[b].t), s = range(d, P.lr[b].s);
        for (int l = P.lr[b].t << sh; l < (P.lr[b].t + 1) << sh; ++l)
            per[static_cast<size_t>(l)].push_back(
                {h.U.get() + h.uoff[b], t.size(), range(P.tau, l).lo - t.lo, i64(2 * b + 1), 0, k, 0, 0});
        for (int l = P.lr[b].s << sh; l < (P.lr[b].s + 1) << sh; ++l)
            per[static_cast<size_t>(l)].push_back(
                {h.V.get() + h.voff[b], s.size(), range(P.tau, l).lo - s.lo, i64(2 * b), 0, k, 0, 0});
    }
    for (size_t b = 0; b < P.dn.size(); ++b) {
        const Range t = range(P.tau, P.dn[b].t), s = range(P.tau, P.dn[b].s);
        double* D = h.D.get() + h.doff[b];
        per[static_cast<size_t>(P.dn[b].t)].push_back({D, t.size(), 0, s.lo, 0, int(s.size()), 1, 0});
        if (P.dn[b].s != P.dn[b].t)  // mirrored block from the stored transpose
            per[static_cast<size_t>(P.dn[b].s)].push_back({D + t.size() * s.size(), s.size(), 0, t.lo, 0,
                                                           int(t.size()), 1, 0});
    }
    std::vector<DHStrong::Contrib> cl;
    std::vector<DHStrong::Tile> tl;
    for (int l = 0; l < nleaves; ++l) {
        const int first = int(cl.size());
        cl.insert(cl.end(), per[static_cast<size_t>(l)].begin(), per[static_cast<size_t>(l)].end());
        h.max_contrib = std::max(h.max_contrib, int(per[static_cast<size_t>(l)].size()));
        const Range lr = range(P.tau, l);
        for (i64 r0 = 0; r0 < lr.size(); r0 += UP_ROWS)
            tl.push_back({int(lr.lo + r0), int(r0), int(std::min<i64>(UP_ROWS, lr.size() - r0)), first, int(cl.size()), 0});
    }
    h.contrib.upload(cl);
    h.tiles.upload(tl);
    h.ntiles = int(tl.size());
    sync();  // host vectors of the lists go out of scope
    return h;
}

namespace {

void proj_tc(const DHStrong::ProjItem* items, int nitems, const double* X, i64 ldx, int k, int s, double* partials) {
    auto& c = current();
    with_tile(tile::tile_for(k), [&](auto TM) {
        constexpr int M = decltype(TM)::value;
        if constexpr (!tile::shape_ok(M, 16) || !tile::shape_ok(M, 64)) {
            throw std::logic_error("hstrong proj_tc: tile extent");
        } else if (s <= 16) {
            constexpr int bytes = tile::smem_bytes_t(tile::STAGES, M, 16);
            attr_once<k_hs_proj_tc<M, 16>>(bytes);
            k_hs_proj_tc<M, 16><<<dim3(unsigned(nitems), unsigned(cdiv(s, 16))), tile::THREADS, bytes, c.stream>>>(
                items, X, ldx, k, s, partials);
        } else {
            constexpr int bytes = tile::smem_bytes_t(tile::STAGES, M, 64);
            attr_once<k_hs_proj_tc<M, 64>>(bytes);
            k_hs_proj_tc<M, 64><<<dim3(unsigned(nitems), unsigned(cdiv(s, 64))), tile::THREADS, bytes, c.stream>>>(
                items, X, ldx, k, s, partials);
        }
    });
}

}  // namespace

// ------------------------------------------------------------------ apply
void hs_apply(const DHStrong& h, const double* X, i64 ldx, int s, double* Y, i64 ldy) {
    if (s <= 0) return;
    auto& c = current();
    const int k = h.k(), nslots = 2 * int(h.plan.lr.size());
    const unsigned cy = unsigned(cdiv(s, 16));
    // wide blocks on the tensor cores (one M tile covers k; a leaf's contributions fit the staged prefix)
    const bool tc = s > 4 && k <= 96 && h.max_contrib <= UTC_MAXC;
    DVec partials, P;
    if (nslots) {
        partials.alloc(static_cast<size_t>(h.nparts) * k * s);
        P.alloc(static_cast<size_t>(nslots) * k * s);
        {
            ProfScope prof(PROF_MATVEC, 2.0 * double(h.U.size() + h.V.size()) * s, 8.0 * double(h.U.size() + h.V.size()));
            if (tc || k <= 96)  // narrow blocks too: the DMMA tile streams the panels at ~5.5 TB/s (the FMA kernel: 1.3)
                proj_tc(h.proj.get(), int(h.proj.size()), X, ldx, k, s, partials.get());
            else
                k_hs_proj<<<dim3(unsigned(h.proj.size()), cy), 256, 0, c.stream>>>(h.proj.get(), X, ldx, k, s,
                                                                                     partials.get());
            HG_LAUNCH();
            k_hs_reduce<<<blocks_for(i64(nslots) * k * s), 256, 0, c.stream>>>(h.dslot_first.get(), nslots,
                                                                                partials.get(), k, s, P.get());
            HG_LAUNCH();
        }
        c.launches += 2;
    }
    ProfScope prof(PROF_MATVEC, 2.0 * double(h.U.size() + h.V.size() + h.D.size()) * s,
                   8.0 * double(h.U.size() + h.V.size() + h.D.size()) + 16.0 * double(h.n()) * s);
    if (s == 1)
        k_hs_update<1><<<h.ntiles, 256, 0, c.stream>>>(h.tiles.get(), h.contrib.get(), P.get(), X, ldx, k, s, Y, ldy);
    else if (s <= 4)
        k_hs_update<4><<<h.ntiles, 256, 0, c.stream>>>(h.tiles.get(), h.contrib.get(), P.get(), X, ldx, k, s, Y, ldy);
    else if (tc && s <= 16) {
        constexpr int bytes = tile::smem_bytes_t(tile::STAGES, UP_ROWS, 16);
        attr_once<k_hs_update_tc<16>>(bytes);
        k_hs_update_tc<16><<<dim3(unsigned(h.ntiles), unsigned(cdiv(s, 16))), tile::THREADS, bytes, c.stream>>>(
            h.tiles.get(), h.contrib.get(), P.get(), X, ldx, k, s, Y, ldy);
    } else if (tc) {
        constexpr int bytes = tile::smem_bytes_t(tile::STAGES, UP_ROWS, 64);
        attr_once<k_hs_update_tc<64>>(bytes);
        k_hs_update_tc<64><<<dim3(unsigned(h.ntiles), unsigned(cdiv(s, 64))), tile::THREADS, bytes, c.stream>>>(
            h.tiles.get(), h.contrib.get(), P.get(), X, ldx, k, s, Y, ldy);
    } else
        k_hs_update_tiled<<<dim3(unsigned(h.ntiles), cy), 256, 0, c.stream>>>(h.tiles.get(), h.contrib.get(), P.get(),
                                                                              X, ldx, k, s, Y, ldy);
    HG_LAUNCH();
    ++c.launches;
}

// ------------------------------------------------------------------ trace
void hs_trace_product(const DHStrong& a, const DHStrong& b, double* out) {
    require(a.plan.n == b.plan.n && a.plan.tau == b.plan.tau && a.plan.k == b.plan.k &&
                a.plan.lr.size() == b.plan.lr.size() && a.plan.dn.size() == b.plan.dn.size() && a.plan.eta == b.plan.eta,
            "hstrong trace_product: different block structures");
    auto& c = current();
    const HsPlan& P = a.plan;
    const int k = P.k, nlr = int(P.lr.size());
    const auto range = [&](int d, int t) { return P.tree.level(d)[static_cast<size_t>(t)]; };
    std::vector<DotItem> dots;
    DVec G;
    if (nlr) {
        // Grams U_A^T U_B (slot 2b) and V_A^T V_B (slot 2b+1)
        std::vector<DHStrong::ProjItem> pj;
        std::vector<int> first(static_cast<size_t>(2 * nlr + 1), 0);
        int part = 0;
        constexpr int PCH = 2048;
        for (int bl = 0; bl < nlr; ++bl) {
            const Range t = range(P.lr[bl].d, P.lr[bl].t), s = range(P.lr[bl].d, P.lr[bl].s);
            for (int side = 0; side < 2; ++side) {
                first[static_cast<size_t>(2 * bl + side)] = part;
                const Range r = side == 0 ? t : s;
                const double* MA = side == 0 ? a.U.get() + a.uoff[bl] : a.V.get() + a.voff[bl];
                const double* MB = side == 0 ? b.U.get() + b.uoff[bl] : b.V.get() + b.voff[bl];
                for (i64 r0 = 0; r0 < r.size(); r0 += PCH)
                    pj.push_back({MA + r0, r.size(), MB, r0, r.size(), int(std::min<i64>(PCH, r.size() - r0)), part++});
            }
        }
        first[static_cast<size_t>(2 * nlr)] = part;
        DBuf<DHStrong::ProjItem> dpj;
        dpj.upload(pj);
        DBuf<int> df;
        df.upload(first);
        DVec partials(static_cast<size_t>(part) * k * k);
        G.alloc(static_cast<size_t>(2 * nlr) * k * k);
        ProfScope prof(PROF_REDUCE, 2.0 * double(a.U.size() + a.V.size()) * k, 16.0 * double(a.U.size() + a.V.size()));
        k_hs_proj<<<dim3(unsigned(pj.size()), unsigned(cdiv(k, 16))), 256, 0, c.stream>>>(dpj.get(), nullptr, 0, k, k,
                                                                                          partials.get());
        HG_LAUNCH();
        k_hs_reduce<<<blocks_for(i64(2 * nlr) * k * k), 256, 0, c.stream>>>(df.get(), 2 * nlr, partials.get(), k, k,
                                                                           G.get());
        HG_LAUNCH();
        c.launches += 2;
        for (int bl = 0; bl < nlr; ++bl)  // <U_A V_A^T, U_B V_B^T> = sum(G1 .* G2), mirrored block: x2
            dots.push_back({G.get() + i64(2 * bl) * k * k, G.get() + i64(2 * bl + 1) * k * k, i64(k) * k, 2.0});
    }
    for (size_t bl = 0; bl < P.dn.size(); ++bl) {
        const Range t = range(P.tau, P.dn[bl].t), s = range(P.tau, P.dn[bl].s);
        dots.push_back({a.D.get() + a.doff[bl], b.D.get() + b.doff[bl], t.size() * s.size(),
                        P.dn[bl].t == P.dn[bl].s ? 1.0 : 2.0});
    }
    DBuf<DotItem> dd;
    dd.upload(dots);
    DVec partial(dots.size());
    ProfScope prof(PROF_REDUCE, 2.0 * double(a.D.size()), 16.0 * double(a.D.size()));
    k_hs_block_dot<<<unsigned(dots.size()), 256, 0, c.stream>>>(dd.get(), partial.get());
    HG_LAUNCH();
    k_hs_sum<<<1, 256, 0, c.stream>>>(partial.get(), int(dots.size()), out);
    HG_LAUNCH();
    c.launches += 2;
}

}  // namespace hg
