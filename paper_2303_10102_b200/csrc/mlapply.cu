// Level-fused HODLR apply: Y = beta Y + alpha H_sel X with H_sel the levels
// [lmin, lmax] (+ leaves), in three launches whatever the number of levels:
//   1. k_ml_proj   T_l[s] = V_l[s]^T X[s] for every level at once (work items
//                  ordered chunk-major so X stays L2-resident across levels);
//   2. k_ml_reduce deterministic sum of the split-K partials (coarse levels);
//   3. k_ml_update Y[tile] (+)= sum_l U_l[tile] T_l[sib(s_l)] — one GEMM whose
//                  K runs over the concatenated level ranks, so Y is read and
//                  written once.
// Reference: HodlrMatrix::matvec / sub_matvec (hodlr_matrix.cpp:198-265).
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "hodlr.cuh"
#include "prof.cuh"
#include "tile.cuh"

namespace hg {

namespace {

using tile::Acc;
using tile::BK;
using tile::BM;
using tile::BN;
using tile::THREADS;

constexpr int MAXL = 24;
constexpr int ML_CHUNK = 512;

struct MlLevels {
    int nl;
    int depth[MAXL];        // partition depth of level l (= l)
    int R[MAXL];            // rank capacity
    int ktoff[MAXL + 1];    // prefix of ceil(R/BK) (update kernel K tiles)
    int coff[MAXL + 1];     // prefix of R (packed update K: levels back to back)
    const double* P[MAXL];  // projection operand (V_l, or U_l when transposed)
    const double* Q[MAXL];  // update operand (U_l, or V_l when transposed)
    double* T[MAXL];        // per-level projections: nseg_l x R_l x s (ld R_l)
    double* ws[MAXL];       // split-K partial workspace (null when one chunk per segment)
    int item_off[MAXL + 1]; // first projection work item of each level
    int ncol[MAXL];         // columns of X the level's projection needs (<= s)
};

struct MlItem {  // projection work item
    int level, seg, row0, rows, chunk;  // chunk = index within the level's partial workspace
};

struct ProjArgs {
    MlLevels L;
    const MlItem* items;
    const double* X;
    i64 ldx, n;
    int s, tiles_n;
    ZeroRows zero;
};

/// Segment (of the hint's partition) holding row r.
__device__ __forceinline__ int seg_of(const int* b, int nseg, int r) {
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (b[mid] <= r)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ int cdiv_i(int a, int b) { return (a + b - 1) / b; }

template <int TBM, int TBN>
__global__ void __launch_bounds__(THREADS) k_ml_proj(ProjArgs g) {
    extern __shared__ double smem[];
    const MlItem it = g.items[blockIdx.x];
    const int l = it.level, R = g.L.R[l];
    const int m0 = (blockIdx.y / g.tiles_n) * TBM, n0 = (blockIdx.y % g.tiles_n) * TBN;
    if (m0 >= R || n0 >= g.L.ncol[l]) return;
    tile::LoadKCT<TBM> la{g.L.P[l] + it.row0 + i64(m0) * g.n, g.n, it.rows, R - m0};
    tile::LoadKCT<TBN> lb{g.X + it.row0 + i64(n0) * g.ldx, g.ldx, it.rows, g.s - n0};
    typename tile::Shape<TBM, TBN>::Acc acc;
    acc.zero();
    int kt = cdiv_i(it.rows, BK);
    if (g.zero.bounds && it.rows > 0) {  // chunk inside a known-zero segment of X: T tile = 0
        const int s0 = seg_of(g.zero.bounds, g.zero.nseg, it.row0);
        const int s1 = seg_of(g.zero.bounds, g.zero.nseg, it.row0 + it.rows - 1);
        if (s0 == s1 && (s0 & 1) == g.zero.parity) kt = 0;
    }
    tile::run_t<tile::STAGES, TBM, TBN>(la, lb, kt, smem, acc);
    const i64 blk = i64(R) * g.s;
    double* o = g.L.ws[l] ? g.L.ws[l] + i64(it.chunk) * blk : g.L.T[l] + i64(it.seg) * blk;
    tile::for_each_t<TBM, TBN>(acc, [&](int mi, int ni, double v) {
        const int m = m0 + mi, c = n0 + ni;
        if (m < R && c < g.s) o[m + i64(c) * R] = v;
    });
}

struct ReduceArgs {
    MlLevels L;
    const int* seg_level;  // per reduce segment: level
    const int* seg_index;  // segment index within the level
    const int* first;      // partial range [first, first+count) in that level's ws
    const int* count;
    int s;
};

__global__ void k_ml_reduce(ReduceArgs g) {
    const int r = blockIdx.y;
    const int l = g.seg_level[r], R = g.L.R[l];
    const i64 blk = i64(R) * g.s;
    const i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= blk || e / R >= g.L.ncol[l]) return;
    const double* w = g.L.ws[l];
    double sum = 0.0;
    for (int c = g.first[r]; c < g.first[r] + g.count[r]; ++c) sum += w[i64(c) * blk + e];
    g.L.T[l][i64(g.seg_index[r]) * blk + e] = sum;
}

struct UpdArgs {
    MlLevels L;
    const WorkItem* items;  // row tiles of the finest partition (depth tau)
    int tau;
    i64 n;
    double* Y;
    i64 ldy;
    int s;
    double alpha, beta;
    int out_depth, out_parity;  // rows read by the caller (ZeroRows::out_depth)
};

/// A operand: rows of the update panels, K = concatenated level columns.
struct LoadUpdA {
    static constexpr bool KC = false;
    static constexpr int ROWS = BM;
    const MlLevels* L;
    int row0, rows;
    i64 n;
    __device__ __forceinline__ void issue(double* S, int kt) const {
        int l = 0;
        while (kt >= L->ktoff[l + 1]) ++l;
        const int kb = (kt - L->ktoff[l]) * BK, R = L->R[l];
        const double* base = L->Q[l] + row0;
        if (tile::pairs_aligned(base, n)) {  // row pairs as 16-byte copies
            const int m2 = 2 * (threadIdx.x & 31);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = (threadIdx.x >> 5) + 4 * q, kk = kb + k;
                const int bytes = kk < R ? (m2 + 1 < rows ? 16 : (m2 < rows ? 8 : 0)) : 0;
                tile::cp_async16(S + k * tile::LD_MC + m2, bytes ? base + m2 + kk * n : base, bytes);
            }
            return;
        }
        const int m = threadIdx.x & 63;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int k = (threadIdx.x >> 6) + 2 * q, kk = kb + k;
            const bool v = m < rows && kk < R;
            tile::cp_async8(S + k * tile::LD_MC + m, v ? base + m + kk * n : base, v);
        }
    }
};

/// B operand: T_l of the sibling segment at each level (k-contiguous, ld R_l).
template <int TBN>
struct LoadUpdB {
    static constexpr bool KC = true;
    static constexpr int ROWS = TBN;
    const MlLevels* L;
    int leaf, tau, s, n0;
    __device__ __forceinline__ void issue(double* S, int kt) const {
        int l = 0;
        while (kt >= L->ktoff[l + 1]) ++l;
        const int kb = (kt - L->ktoff[l]) * BK, R = L->R[l];
        const int seg = (leaf >> (tau - L->depth[l])) ^ 1;
        const double* base = L->T[l] + i64(seg) * R * s + i64(n0) * R;
        const int k = threadIdx.x & 15, kk = kb + k;
#pragma unroll
        for (int q = 0; q < TBN / 8; ++q) {
            const int c = (threadIdx.x >> 4) + 8 * q;
            const bool v = kk < R && n0 + c < s;
            tile::cp_async8(S + c * tile::LD_KC + k, v ? base + kk + i64(c) * R : base, v);
        }
    }
};

constexpr int PACK_MAX = 2048;  // packed update K held as a (level, column) table in shared memory
#ifndef HG_UPD_NS
#define HG_UPD_NS 2
#endif
constexpr int UPD_NS = HG_UPD_NS;  // cp.async stages of the packed update (3 measured slower: occupancy)

/// Packed A operand: K runs over the levels' columns back to back (no
/// per-level padding to BK); tab[c] = level << 16 | column for c < coff[nl].
struct LoadUpdAPacked {
    static constexpr bool KC = false;
    static constexpr int ROWS = BM;
    const MlLevels* L;
    const int* tab;
    int row0, rows;
    i64 n;
    __device__ __forceinline__ void issue(double* S, int kt) const {
        const int ktot = L->coff[L->nl];
        if (((row0 | n) & 1) == 0) {  // row pairs as 16-byte copies (panels are 16-byte aligned)
            const int m2 = 2 * (threadIdx.x & 31);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = (threadIdx.x >> 5) + 4 * q, cc = kt * BK + k;
                const int bytes = cc < ktot ? (m2 + 1 < rows ? 16 : (m2 < rows ? 8 : 0)) : 0;
                const int e = cc < ktot ? tab[cc] : 0, l = e >> 16, j = e & 0xffff;
                const double* src = L->Q[l] + row0 + m2 + i64(j) * n;
                if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
                    tile::cp_async16(S + k * tile::LD_MC + m2, bytes ? src : L->Q[0], bytes);
                } else {  // a panel view at an odd offset
                    tile::cp_async8(S + k * tile::LD_MC + m2, bytes >= 8 ? src : L->Q[0], bytes >= 8);
                    tile::cp_async8(S + k * tile::LD_MC + m2 + 1, bytes == 16 ? src + 1 : L->Q[0], bytes == 16);
                }
            }
            return;
        }
        const int m = threadIdx.x & 63;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int k = (threadIdx.x >> 6) + 2 * q, cc = kt * BK + k;
            const bool v = m < rows && cc < ktot;
            const int e = v ? tab[cc] : 0, l = e >> 16, j = e & 0xffff;
            const double* src = L->Q[l] + row0 + m + i64(j) * n;
            tile::cp_async8(S + k * tile::LD_MC + m, v ? src : L->Q[0], v);
        }
    }
};

template <int TBN>
struct LoadUpdBPacked {
    static constexpr bool KC = true;
    static constexpr int ROWS = TBN;
    const MlLevels* L;
    const int* tab;
    int leaf, tau, s, n0;
    __device__ __forceinline__ void issue(double* S, int kt) const {
        const int k = threadIdx.x & 15, cc = kt * BK + k, ktot = L->coff[L->nl];
        const bool kv = cc < ktot;
        const int e = kv ? tab[cc] : 0, l = e >> 16, j = e & 0xffff, R = L->R[l];
        const int seg = (leaf >> (tau - L->depth[l])) ^ 1;
        const double* base = L->T[l] + i64(seg) * R * s + i64(n0) * R + j;
#pragma unroll
        for (int q = 0; q < TBN / 8; ++q) {
            const int c = (threadIdx.x >> 4) + 8 * q;
            const bool v = kv && n0 + c < s;
            tile::cp_async8(S + c * tile::LD_KC + k, v ? base + i64(c) * R : L->T[0], v);
        }
    }
};

template <int TBN>
__global__ void __launch_bounds__(THREADS) k_ml_update_packed(UpdArgs g) {
    extern __shared__ double smem[];
    __shared__ MlLevels L;
    __shared__ int tab[PACK_MAX];
    if (g.out_depth >= 0 && ((g.items[blockIdx.x].seg >> (g.tau - g.out_depth)) & 1) != g.out_parity) return;
    for (int i = threadIdx.x; i < int(sizeof(MlLevels) / sizeof(int)); i += blockDim.x)
        reinterpret_cast<int*>(&L)[i] = reinterpret_cast<const int*>(&g.L)[i];
    __syncthreads();
    const int ktot = L.coff[L.nl];
    for (int c = threadIdx.x; c < ktot; c += blockDim.x) {
        int l = 0;
        while (c >= L.coff[l + 1]) ++l;
        tab[c] = (l << 16) | (c - L.coff[l]);
    }
    __syncthreads();
    const WorkItem it = g.items[blockIdx.x];
    const int n0 = blockIdx.y * TBN;
    LoadUpdAPacked la{&L, tab, it.row0, it.rows, g.n};
    LoadUpdBPacked<TBN> lb{&L, tab, it.seg, g.tau, g.s, n0};
    typename tile::Shape<BM, TBN>::Acc acc, yv;
    acc.zero();
    yv.zero();
    if (g.beta != 0.0)
        tile::for_each_slot<BM, TBN>(yv, [&](double& y, int m, int ni) {
            const int c = n0 + ni;
            if (c < g.s && m < it.rows) y = g.Y[i64(it.row0 + m) + i64(c) * g.ldy];
        });
    tile::run_t<UPD_NS, BM, TBN>(la, lb, (ktot + BK - 1) / BK, smem, acc);
    tile::for_each_slot2<BM, TBN>(acc, yv, [&](double v, double y, int m, int ni) {
        const int c = n0 + ni;
        if (c >= g.s || m >= it.rows) return;
        g.Y[i64(it.row0 + m) + i64(c) * g.ldy] = g.alpha * v + g.beta * y;
    });
}

template <int TBN>
__global__ void __launch_bounds__(THREADS) k_ml_update(UpdArgs g) {
    extern __shared__ double smem[];
    __shared__ MlLevels L;
    if (g.out_depth >= 0 && ((g.items[blockIdx.x].seg >> (g.tau - g.out_depth)) & 1) != g.out_parity) return;
    for (int i = threadIdx.x; i < int(sizeof(MlLevels) / sizeof(int)); i += blockDim.x)
        reinterpret_cast<int*>(&L)[i] = reinterpret_cast<const int*>(&g.L)[i];
    __syncthreads();
    const WorkItem it = g.items[blockIdx.x];
    const int n0 = blockIdx.y * TBN;
    LoadUpdA la{&L, it.row0, it.rows, g.n};
    LoadUpdB<TBN> lb{&L, it.seg, g.tau, g.s, n0};
    typename tile::Shape<BM, TBN>::Acc acc, yv;
    acc.zero();
    yv.zero();
    if (g.beta != 0.0)  // fetch the accumulated Y before the main loop (latency overlap)
        tile::for_each_slot<BM, TBN>(yv, [&](double& y, int m, int ni) {
            const int c = n0 + ni;
            if (c < g.s && m < it.rows) y = g.Y[i64(it.row0 + m) + i64(c) * g.ldy];
        });
    tile::run_t<2, BM, TBN>(la, lb, L.ktoff[L.nl], smem, acc);
    tile::for_each_slot2<BM, TBN>(acc, yv, [&](double v, double y, int m, int ni) {
        const int c = n0 + ni;
        if (c >= g.s || m >= it.rows) return;
        g.Y[i64(it.row0 + m) + i64(c) * g.ldy] = g.alpha * v + g.beta * y;
    });
}

/// Projection work items of levels [lmin, lmax] (chunk-major), cached per tree.
struct ItemPlan {
    DBuf<MlItem> items;
    int count = 0;
    std::vector<int> item_off;           // per level (relative to lmin)
    std::vector<int> nchunks;            // per level: partial count (0 => direct)
    DBuf<int> rl, ri, rf, rc;            // reduce segments
    int nred = 0;
};

const ItemPlan& item_plan(const DTree& t, int lmin, int lmax, int chunk_rows) {
    static std::mutex mu;
    static std::map<std::tuple<const DTree*, int, int, int>, std::unique_ptr<ItemPlan>> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(&t, lmin, lmax, chunk_rows);
    auto itc = cache.find(key);
    if (itc != cache.end()) return *itc->second;
    auto p = std::make_unique<ItemPlan>();
    const int nl = lmax - lmin + 1;
    // Per level: chunks of at most chunk_rows rows that never cross a segment.
    std::vector<std::vector<MlItem>> per(static_cast<size_t>(nl));
    std::vector<int> rl, ri, rf, rc;
    p->nchunks.assign(static_cast<size_t>(nl), 0);
    for (int i = 0; i < nl; ++i) {
        const Partition& pt = t.part(lmin + i);
        const auto& hb = pt.hbounds();
        bool multi = false;
        for (int sgi = 0; sgi < pt.nseg(); ++sgi)
            if (hb[static_cast<size_t>(sgi + 1)] - hb[static_cast<size_t>(sgi)] > chunk_rows) multi = true;
        int chunk = 0;
        for (int sgi = 0; sgi < pt.nseg(); ++sgi) {
            const int lo = hb[static_cast<size_t>(sgi)], hi = hb[static_cast<size_t>(sgi + 1)];
            const int first = chunk;
            for (int r = lo; r < hi || r == lo; r += chunk_rows) {
                per[static_cast<size_t>(i)].push_back(MlItem{i, sgi, r, std::min(chunk_rows, hi - r), chunk++});
                if (hi == lo) break;
            }
            if (multi) {
                rl.push_back(i);
                ri.push_back(sgi);
                rf.push_back(first);
                rc.push_back(chunk - first);
            }
        }
        p->nchunks[static_cast<size_t>(i)] = multi ? chunk : 0;
    }
    // Chunk-major interleave: items touching the same rows run back to back.
    std::vector<MlItem> all;
    std::vector<size_t> pos(static_cast<size_t>(nl), 0);
    p->item_off.assign(static_cast<size_t>(nl + 1), 0);
    bool left = true;
    while (left) {
        left = false;
        // advance every level up to the same row position
        int row = 1 << 30;
        for (int i = 0; i < nl; ++i)
            if (pos[static_cast<size_t>(i)] < per[static_cast<size_t>(i)].size())
                row = std::min(row, per[static_cast<size_t>(i)][pos[static_cast<size_t>(i)]].row0);
        for (int i = 0; i < nl; ++i) {
            auto& v = per[static_cast<size_t>(i)];
            while (pos[static_cast<size_t>(i)] < v.size() && v[pos[static_cast<size_t>(i)]].row0 <= row) {
                all.push_back(v[pos[static_cast<size_t>(i)]++]);
            }
            if (pos[static_cast<size_t>(i)] < v.size()) left = true;
        }
    }
    p->count = int(all.size());
    p->items.upload(all);
    p->nred = int(rl.size());
    if (p->nred) {
        p->rl.upload(rl);
        p->ri.upload(ri);
        p->rf.upload(rf);
        p->rc.upload(rc);
    }
    auto& ref = *p;
    cache[key] = std::move(p);
    return ref;
}

// ------------------------------------------------ concatenated thin projections
// hodlr_project for thin bases (sum of the level ranks <= CAT_MAX): instead of
// one GEMM per level over the same rows of X (13 re-reads of every X chunk
// through L2, which bounded the cross terms of the sigma^2 derivative), one
// GEMM per row span with N = all levels' columns side by side, so each CTA
// reads its X tile once. A level's accumulators are flushed whenever the
// K loop crosses one of its segment boundaries (uniform trees: segments of
// n >> depth rows); levels wider than the span leave per-span partials that
// a fixed-order reduction folds.
constexpr int CAT_MAX = 96;

struct CatArgs {
    const double* X;
    i64 ldx, n;
    int s, nl, ncat, span;
    int tiles_m, tau, leaf;
    const double* P[MAXL];
    int R[MAXL], coff[MAXL + 1], ncol[MAXL], depth[MAXL];
    double* T[MAXL];
    double* ws[MAXL];
};

template <int TBN>
struct LoadCat {
    static constexpr bool KC = true;
    static constexpr int ROWS = TBN;
    const double* const* colp;  // per concatenated column: panel column base (null = absent)
    const double* dummy;
    int row0, kmax;
    __device__ __forceinline__ void issue(double* S, int kt) const {
        const int k = threadIdx.x & 15, kk = kt * BK + k;
#pragma unroll
        for (int q = 0; q < TBN / 8; ++q) {
            const int c = (threadIdx.x >> 4) + 8 * q;
            const double* p = colp[c];
            const bool v = p != nullptr && kk < kmax;
            tile::cp_async8(S + c * tile::LD_KC + k, v ? p + row0 + kk : dummy, v);
        }
    }
};

template <int TBM, int TBN>
__global__ void __launch_bounds__(THREADS) k_proj_cat(const __grid_constant__ CatArgs g) {
    extern __shared__ double smem[];
    __shared__ const double* colp[TBN];
    __shared__ int collev[TBN];
    const int sp = blockIdx.x, row0 = sp * g.span;
    const int m0 = blockIdx.y * TBM;
    for (int j = threadIdx.x; j < TBN; j += blockDim.x) {
        int l = -1;
        const double* p = nullptr;
        if (j < g.ncat) {
            l = 0;
            while (j >= g.coff[l + 1]) ++l;
            if (m0 < g.ncol[l]) p = g.P[l] + i64(j - g.coff[l]) * g.n;
        }
        collev[j] = l;
        colp[j] = p;
    }
    __syncthreads();
    tile::LoadKCT<TBM> la{g.X + row0 + i64(m0) * g.ldx, g.ldx, g.span, g.s - m0};
    LoadCat<TBN> lb{colp, g.X, row0, g.span};
    typename tile::Shape<TBM, TBN>::Acc acc;
    acc.zero();
    const int ktiles = g.span / BK;
    auto flush = [&](int li, int seg, bool direct) {
        const int R = g.R[li], c0 = g.coff[li], nc = g.ncol[li];
        double* o = direct ? g.T[li] + i64(seg) * R * g.s : g.ws[li] + i64(sp) * R * g.s;
        tile::for_each_slot<TBM, TBN>(acc, [&](double& v, int m, int j) {
            if (collev[j] != li) return;
            const int c = m0 + m;
            if (c < nc) o[(j - c0) + i64(c) * R] = v;
            v = 0.0;
        });
    };
    // flush schedule in leaf units (bit tests only): a depth-d segment spans
    // 2^(tau - d) leaves of g.leaf rows
    const int leaf_kt = g.leaf / BK, leaf0 = row0 / g.leaf;
    int kc = 0, ld = 0;
    tile::run_t_hook<tile::STAGES, TBM, TBN>(la, lb, ktiles, smem, acc, [&](int kt) {
        if (++kc < leaf_kt) return;
        kc = 0;
        ++ld;
        for (int li = 0; li < g.nl; ++li) {
            if (g.R[li] == 0 || m0 >= g.ncol[li]) continue;
            const int sh = g.tau - g.depth[li];
            if ((i64(g.leaf) << sh) <= g.span) {
                if ((ld & ((1 << sh) - 1)) == 0) flush(li, ((leaf0 + ld) >> sh) - 1, true);
            } else if (kt + 1 == ktiles) {
                flush(li, 0, false);
            }
        }
    });
}

/// T_l[seg] = sum of the per-span partials of levels wider than the span.
__global__ void k_cat_reduce(const __grid_constant__ CatArgs g, int li) {
    const int seg = blockIdx.y;
    const int R = g.R[li];
    const i64 blk = i64(R) * g.s;
    const i64 S = g.n >> g.depth[li];
    const int cps = int(S / g.span);
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < blk; e += i64(gridDim.x) * blockDim.x) {
        if (e / R >= g.ncol[li]) continue;
        double acc = 0.0;
        for (int c = 0; c < cps; ++c) acc += g.ws[li][i64(seg * cps + c) * blk + e];
        g.T[li][i64(seg) * blk + e] = acc;
    }
}

/// k_proj_cat applies: uniform tree (leaves of n >> tau rows, a multiple of
/// BK), levels [l0, l1] with at most CAT_MAX columns side by side.
bool proj_cat_ok(const DHodlr& h, int l0, int l1, const int* nc, int ncat) {
    const i64 n = h.n();
    const int tau = h.tau();
    if (ncat <= 0 || ncat > CAT_MAX || tau < 1 || l1 - l0 + 1 > MAXL || n >= (i64(1) << 31)) return false;
    if (n % (i64(1) << tau) != 0 || (n >> tau) % BK != 0 || std::getenv("HG_NO_PROJ_CAT")) return false;
    (void)nc;
    return true;
}

/// T_l[seg] (R_l x nc_l, ld R_l, segment stride R_l s) = P_l[seg]^T X[seg] for
/// l in [l0, l1] in one pass over X (P = U when transpose, else V).
void proj_cat(const DHodlr& h, const double* X, i64 ldx, int s, bool transpose, int l0, int l1, const int* nc,
              double* const* tout) {
    auto& c = current();
    const i64 n = h.n();
    const int tau = h.tau(), nl = l1 - l0 + 1;
    const i64 leaf = n >> tau;
    int ncat = 0, cmax = 0;
    for (int i = 0; i < nl; ++i)
        if (nc[i] > 0) {
            ncat += h.Rl(l0 + i);
            cmax = std::max(cmax, nc[i]);
        }
    const int tbm = tile::tile_for(cmax), tbn = tile::tile_for(ncat);
    const int tiles_m = cdiv(cmax, tbm);
    i64 span = n;
    while (span > leaf && (n / span) * tiles_m < 4 * c.num_sms) span /= 2;
    CatArgs a{};
    a.X = X;
    a.ldx = ldx;
    a.n = n;
    a.s = s;
    a.nl = nl;
    a.ncat = ncat;
    a.span = int(span);
    a.tiles_m = tiles_m;
    a.tau = tau;
    a.leaf = int(leaf);
    a.coff[0] = 0;
    std::vector<DVec> wsb(static_cast<size_t>(nl));
    double flops = 0;
    for (int i = 0; i < nl; ++i) {
        const int l = l0 + i;
        const int R = nc[i] > 0 ? h.Rl(l) : 0;
        a.P[i] = transpose ? h.Ul(l) : h.Vl(l);
        a.R[i] = R;
        a.coff[i + 1] = a.coff[i] + R;
        a.ncol[i] = nc[i];
        a.depth[i] = l;
        a.T[i] = tout[i];
        if (R > 0 && (n >> l) > span) {
            wsb[static_cast<size_t>(i)].alloc(static_cast<size_t>(n / span) * R * s);
            a.ws[i] = wsb[static_cast<size_t>(i)].get();
        }
        flops += 2.0 * double(n) * R * nc[i];
    }
    ProfScope prof(PROF_SEG_TN, flops, 8.0 * double(n) * (cmax + ncat));
    if (prof_enabled()) prof.key(prof_tag("projcat l=%d..%d s=%d ncat=%d span=%d", l0, l1, s, ncat, int(span)));
    with_tile(tbm, [&](auto TM) {
        with_tile(tbn, [&](auto TN) {
            constexpr int M = decltype(TM)::value, N = decltype(TN)::value;
            if constexpr (tile::shape_ok(M, N)) {
                constexpr int bytes = tile::smem_bytes_t(tile::STAGES, M, N);
                static DeviceOnce once;
                if (once.first())
                    HG_CUDA(cudaFuncSetAttribute(k_proj_cat<M, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
                k_proj_cat<M, N><<<dim3(unsigned(n / span), unsigned(tiles_m)), THREADS, bytes, c.stream>>>(a);
            } else {
                throw std::logic_error("proj_cat: unsupported tile shape");
            }
        });
    });
    HG_LAUNCH();
    ++c.launches;
    for (int i = 0; i < nl; ++i)
        if (a.ws[i]) {
            const int nseg = int(i64(1) << (l0 + i));
            k_cat_reduce<<<dim3(unsigned(cdiv(i64(a.R[i]) * s, 256 * 4)), unsigned(nseg)), 256, 0, c.stream>>>(a, i);
            HG_LAUNCH();
            ++c.launches;
        }
}

// ------------------------------------------------ leaf-sampler projections
constexpr int LID_GL = 32;  // leaves per CTA
constexpr int LID_J = 8;    // panel columns per CTA (independent accumulators per thread)

struct LeafIdArgs {
    const int* lb;  // leaf bounds
    i64 n;
    int tau, nl, s;
    const double* P[MAXL];
    int R[MAXL], depth[MAXL];
    double* T[MAXL];
    double* ws[MAXL];  // levels whose segments exceed LID_GL leaves: per-group partials
};

/// T_l[seg](j, c) = sum over the leaves b of seg of P_l[lo_b + c, j] (c < m_b).
/// Thread = column c of the leaf block, LID_J panel columns per CTA.
__global__ void __launch_bounds__(256) k_leafid_proj(const __grid_constant__ LeafIdArgs a) {
    const int li = blockIdx.y, R = a.R[li];
    const int j0 = blockIdx.z * LID_J;
    if (j0 >= R) return;
    const int g = blockIdx.x, b0 = g * LID_GL, nleaves = 1 << a.tau;
    const int Ls = 1 << (a.tau - a.depth[li]);  // leaves per segment
    const i64 blk = i64(R) * a.s;
    const int c = threadIdx.x;
    const double* P = a.P[li] + i64(j0) * a.n + c;
    const int b1 = min(b0 + LID_GL, nleaves);
    const int seglen = Ls < LID_GL ? Ls : LID_GL;
    for (int s0 = b0; s0 < b1; s0 += seglen) {
        double acc[LID_J];
#pragma unroll
        for (int q = 0; q < LID_J; ++q) acc[q] = 0.0;
        for (int b = s0; b < min(s0 + seglen, b1); ++b) {
            const int lo = a.lb[b], m = a.lb[b + 1] - lo;
            if (c >= m || c >= a.s) continue;
#pragma unroll
            for (int q = 0; q < LID_J; ++q)
                if (j0 + q < R) acc[q] += P[lo + i64(q) * a.n];
        }
        if (c >= a.s) continue;
        double* o = Ls <= LID_GL ? a.T[li] + i64(s0 / Ls) * blk : a.ws[li] + i64(g) * blk;
#pragma unroll
        for (int q = 0; q < LID_J; ++q)
            if (j0 + q < R) o[(j0 + q) + i64(c) * R] = acc[q];
    }
}

__global__ void k_leafid_fold(const __grid_constant__ LeafIdArgs a, int li) {
    const int seg = blockIdx.y, R = a.R[li];
    const i64 blk = i64(R) * a.s;
    const int gps = (1 << (a.tau - a.depth[li])) / LID_GL;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < blk; e += i64(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int q = 0; q < gps; ++q) acc += a.ws[li][i64(seg * gps + q) * blk + e];
        a.T[li][i64(seg) * blk + e] = acc;
    }
}

/// Projections of the leaf sampler for levels [l0, l0 + nl) into T[] (one
/// streaming pass over each panel instead of a GEMM with an identity stack).
void leafid_proj(const DHodlr& h, bool transpose, int l0, int nl, int s, double* const* T) {
    auto& c = current();
    const DTree& t = *h.tree;
    const int tau = t.tau(), nleaves = 1 << tau;
    LeafIdArgs a{};
    a.lb = t.leaves().dbounds();
    a.n = h.n();
    a.tau = tau;
    a.nl = nl;
    a.s = s;
    std::vector<DVec> wsb(static_cast<size_t>(nl));
    for (int i = 0; i < nl; ++i) {
        const int l = l0 + i;
        a.P[i] = transpose ? h.Ul(l) : h.Vl(l);
        a.R[i] = h.Rl(l);
        a.depth[i] = l;
        a.T[i] = T[i];
        if (a.R[i] > 0 && (nleaves >> l) > LID_GL) {
            wsb[static_cast<size_t>(i)].alloc(static_cast<size_t>(cdiv(nleaves, LID_GL)) * a.R[i] * s);
            a.ws[i] = wsb[static_cast<size_t>(i)].get();
        }
    }
    int rmax = 1;
    for (int i = 0; i < nl; ++i) rmax = std::max(rmax, a.R[i]);
    if (s > 256) throw std::logic_error("leafid_proj: leaves wider than 256 rows");
    const int nt = (s + 31) / 32 * 32;  // thread = column of the leaf block
    k_leafid_proj<<<dim3(unsigned(cdiv(nleaves, LID_GL)), unsigned(nl), unsigned(cdiv(rmax, LID_J))), nt, 0,
                    c.stream>>>(a);
    HG_LAUNCH();
    ++c.launches;
    for (int i = 0; i < nl; ++i)
        if (a.ws[i]) {
            k_leafid_fold<<<dim3(unsigned(cdiv(i64(a.R[i]) * s, 1024)), unsigned(1 << (l0 + i))), 256, 0, c.stream>>>(
                a, i);
            HG_LAUNCH();
            ++c.launches;
        }
}

/// Projection chunk: from ML_CHUNK rows, doubled while >= 8 CTAs per SM remain
/// (fewer split-K partials to write and fold).
int proj_chunk(const DTree& t, int nl, int tiles) {
    int chunk = ML_CHUNK;
    const i64 n = t.n();
    // beyond ~1024 rows an item's X chunk stops being L2-resident across the
    // level items that share it (s = 64 matvec: 6.68 -> 6.31 ms at 1024)
    const char* e = std::getenv("HG_PROJ_CHUNK_MAX");
    const int cmax = e ? std::atoi(e) : 1024;
    while (chunk < t.part(1).max_seg() && chunk < cmax && (n / (2 * chunk)) * nl * tiles >= 8 * current().num_sms)
        chunk *= 2;
    return chunk;
}

}  // namespace

void hodlr_apply(const DHodlr& h, const double* X, i64 ldx, int s, double* Y, i64 ldy, int lmin, int lmax,
                 bool with_leaves, bool transpose, double beta, double alpha, ZeroRows zero) {
    if (s <= 0) return;
    if (hodlr_apply_narrow(h, X, ldx, s, Y, ldy, lmin, lmax, with_leaves, transpose, beta, alpha, zero)) return;
    const i64 n = h.n();
    const DTree& t = *h.tree;
    if (with_leaves && !h.leaves_zero) {
        leaf_mm(t.leaves(), h.leaves->get(), h.lstride(), h.bmax(), transpose, X, ldx, Y, ldy, s, alpha, beta);
        beta = 1.0;
    }
    lmin = std::max(lmin, 1);
    lmax = std::min(lmax, h.tau());
    // levels with nonzero rank
    std::vector<int> lv;
    for (int l = lmin; l <= lmax; ++l)
        if (h.Rl(l) > 0) lv.push_back(l);
    if (lv.empty()) {
        if (beta != 1.0) panel_axpby(n, s, 0.0, nullptr, 0, beta, Y, ldy);
        return;
    }
    if (int(lv.size()) > MAXL) throw std::length_error("hodlr_apply: too many levels");
    auto& c = current();
    MlLevels L{};
    L.nl = lmax - lmin + 1;
    std::vector<DVec> Tbuf(static_cast<size_t>(L.nl)), Wbuf(static_cast<size_t>(L.nl));
    double flops = 0, bytes = 8.0 * double(n) * (s + 2.0 * s);
    L.ktoff[0] = 0;
    L.coff[0] = 0;
    for (int i = 0; i < L.nl; ++i) {
        const int l = lmin + i, R = h.Rl(l);
        const Partition& pt = t.part(l);
        L.depth[i] = l;
        L.R[i] = R;
        L.ktoff[i + 1] = L.ktoff[i] + (R + BK - 1) / BK;
        L.coff[i + 1] = L.coff[i] + R;
        L.P[i] = transpose ? h.Ul(l) : h.Vl(l);
        L.Q[i] = transpose ? h.Vl(l) : h.Ul(l);
        if (R > 0) Tbuf[static_cast<size_t>(i)].alloc(static_cast<size_t>(pt.nseg()) * R * s);
        L.T[i] = Tbuf[static_cast<size_t>(i)].get();
        L.ws[i] = nullptr;
        L.ncol[i] = s;
        // algorithmic flops: the projection reads only the nonzero half of X
        // under a ZeroRows hint, the update writes only the rows the caller reads
        const double f = 2.0 * double(n) * R * s;
        if (!(zero.leaf_identity && s == h.bmax() && s <= 256))  // leaf sampler: the projection is a sum, not a GEMM
            flops += zero.bounds ? 0.5 * f : f;
        flops += (zero.bounds && zero.out_depth >= 0) ? 0.5 * f : f;
        bytes += 16.0 * double(n) * R;
    }
    ProfScope prof(PROF_SEG_TN, flops, bytes);
    if (prof_enabled()) {
        int rmax = 0;
        for (int l = lmin; l <= lmax; ++l) rmax = std::max(rmax, h.Rl(l));
        prof.key(prof_tag("mlapply l=%d..%d s=%d Rmax=%d tr=%d", lmin, lmax, s, rmax, int(transpose)));
    }
    const bool zero_was_leafid = zero.leaf_identity && s == h.bmax() && s <= 256;
    if (zero_was_leafid) {
        leafid_proj(h, transpose, lmin, L.nl, s, L.T);
        zero = ZeroRows{};
    }
    // Projections in runs of consecutive levels sharing an M tile (a derivative
    // HODLR has ranks 4..8 on most levels and ~45 on the deepest two: one tile
    // for all would pad the thin levels up to 12x).
    auto proj_tile = [&](int R) { return tile::tile_for(std::max(R, 1)); };
    for (int a = (zero_was_leafid ? L.nl : 0); a < L.nl;) {
        int e = a, tb = -1;  // run [a, e): levels with one projection tile (empty levels join any run)
        for (; e < L.nl; ++e) {
            if (L.R[e] == 0) continue;
            if (tb < 0)
                tb = proj_tile(L.R[e]);
            else if (proj_tile(L.R[e]) != tb)
                break;
        }
        const int b = e - 1;
        int rmax = 1, ncat = 0;
        for (int i = a; i <= b; ++i) {
            rmax = std::max(rmax, L.R[i]);
            ncat += L.R[i];
        }
        if (!zero.bounds && rmax <= 16) {  // thin run: all its levels in one pass over X
            std::vector<int> nc(static_cast<size_t>(b - a + 1), s);
            if (proj_cat_ok(h, lmin + a, lmin + b, nc.data(), ncat)) {
                proj_cat(h, X, ldx, s, transpose, lmin + a, lmin + b, nc.data(), L.T + a);
                a = e;
                continue;
            }
        }
        int tbm = tile::tile_for(rmax);
        const int tbn = tile::tile_for_n(s, tbm);
        if (rmax > 32 && rmax <= 40 && tbn % 32 == 0) tbm = 40;  // 1 x 4 warp grid: no padding of rank-40 levels
        const int max_tiles_m = (rmax + tbm - 1) / tbm;
        const int tiles_n = (s + tbn - 1) / tbn;
        int chunk = proj_chunk(t, b - a + 1, max_tiles_m * tiles_n);
        if (zero.bounds)  // keep chunks inside the hint's segments so zero chunks are still skipped
            while (chunk > ML_CHUNK && chunk > n / std::max(zero.nseg, 1)) chunk /= 2;
        const ItemPlan& ip = item_plan(t, lmin + a, lmin + b, chunk);
        MlLevels Ls{};
        Ls.nl = b - a + 1;
        for (int i = 0; i < Ls.nl; ++i) {
            const int j = a + i;
            Ls.depth[i] = L.depth[j];
            Ls.R[i] = L.R[j];
            Ls.P[i] = L.P[j];
            Ls.Q[i] = L.Q[j];
            Ls.T[i] = L.T[j];
            Ls.ncol[i] = s;
            if (L.R[j] > 0 && ip.nchunks[static_cast<size_t>(i)])
                Wbuf[static_cast<size_t>(j)].alloc(static_cast<size_t>(ip.nchunks[static_cast<size_t>(i)]) * L.R[j] * s);
            Ls.ws[i] = Wbuf[static_cast<size_t>(j)].get();
        }
        ProjArgs pa{Ls, ip.items.get(), X, ldx, n, s, tiles_n, zero};
        with_tile(tbm, [&](auto TM) {
            with_tile(tbn, [&](auto TN) {
                constexpr int M = decltype(TM)::value, N = decltype(TN)::value;
                if constexpr (tile::shape_ok(M, N)) {
                    constexpr int bytes = tile::smem_bytes_t(tile::STAGES, M, N);
                    attr_once<k_ml_proj<M, N>>(bytes);
                    k_ml_proj<M, N>
                        <<<dim3(unsigned(ip.count), unsigned(max_tiles_m * tiles_n)), THREADS, bytes, c.stream>>>(pa);
                } else {
                    throw std::logic_error("hodlr_apply: unsupported tile shape");
                }
            });
        });
        HG_LAUNCH();
        ++c.launches;
        if (ip.nred) {
            int maxblk = 0;
            for (int i = 0; i < Ls.nl; ++i) maxblk = std::max(maxblk, Ls.R[i] * s);
            ReduceArgs ra{Ls, ip.rl.get(), ip.ri.get(), ip.rf.get(), ip.rc.get(), s};
            k_ml_reduce<<<dim3(unsigned(cdiv(maxblk, 256)), unsigned(ip.nred)), 256, 0, c.stream>>>(ra);
            HG_LAUNCH();
            ++c.launches;
        }
        a = e;
    }
    const TileList& tl = t.leaves().tiles(BM);
    UpdArgs ua{L, tl.items.get(), t.tau(), n, Y, ldy, s, alpha, beta,
               zero.bounds && zero.out_depth <= t.tau() ? zero.out_depth : -1, zero.parity};
    // the update's N tile may differ from the projection's (its M is always 64)
    const int tbn_u = tile::tile_for_n(s, BM), tiles_nu = (s + tbn_u - 1) / tbn_u;
    const bool packed = L.coff[L.nl] <= PACK_MAX && (L.coff[L.nl] + BK - 1) / BK < L.ktoff[L.nl];
    with_tile(tbn_u, [&](auto TN) {
        constexpr int N = decltype(TN)::value;
        constexpr int bytes = tile::smem_bytes_t(2, BM, N);
        if (packed) {
            constexpr int pbytes = tile::smem_bytes_t(UPD_NS, BM, N);
            static DeviceOnce once;  // static table + dynamic stages exceed the default 48 KB
            if (once.first())
                HG_CUDA(cudaFuncSetAttribute(k_ml_update_packed<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, pbytes));
            k_ml_update_packed<N><<<dim3(unsigned(tl.count), unsigned(tiles_nu)), THREADS, pbytes, c.stream>>>(ua);
        } else {
            attr_once<k_ml_update<N>>(bytes);
            k_ml_update<N><<<dim3(unsigned(tl.count), unsigned(tiles_nu)), THREADS, bytes, c.stream>>>(ua);
        }
    });
    HG_LAUNCH();
    ++c.launches;
}

std::vector<DVecP> hodlr_project(const DHodlr& h, const double* X, i64 ldx, int s, bool transpose,
                                 const std::vector<int>& ncol) {
    const i64 n = h.n();
    const DTree& t = *h.tree;
    const int tau = h.tau();
    std::vector<DVecP> out(static_cast<size_t>(tau));
    if (s <= 0 || tau < 1) return out;
    if (tau > MAXL) throw std::length_error("hodlr_project: too many levels");
    auto& c = current();
    {  // thin bases: one pass over X for all levels (k_proj_cat)
        std::vector<int> nc(static_cast<size_t>(tau));
        std::vector<double*> tout(static_cast<size_t>(tau), nullptr);
        int ncat = 0;
        for (int i = 0; i < tau; ++i) {
            nc[static_cast<size_t>(i)] = std::min(s, ncol[static_cast<size_t>(i)]);
            if (nc[static_cast<size_t>(i)] > 0) ncat += h.Rl(i + 1);
        }
        if (proj_cat_ok(h, 1, tau, nc.data(), ncat)) {
            for (int i = 0; i < tau; ++i)
                if (nc[static_cast<size_t>(i)] > 0 && h.Rl(i + 1) > 0) {
                    out[static_cast<size_t>(i)] =
                        make_dvec(static_cast<size_t>(t.part(i + 1).nseg()) * h.Rl(i + 1) * s, false);
                    tout[static_cast<size_t>(i)] = out[static_cast<size_t>(i)]->get();
                }
            proj_cat(h, X, ldx, s, transpose, 1, tau, nc.data(), tout.data());
            return out;
        }
    }
    int rmax0 = 1, cmax0 = 1;
    for (int l = 1; l <= tau; ++l) {
        rmax0 = std::max(rmax0, h.Rl(l));
        cmax0 = std::max(cmax0, std::min(s, ncol[static_cast<size_t>(l - 1)]));
    }
    const int tbm0 = tile::tile_for(rmax0), tbn0 = tile::tile_for_n(cmax0, tbm0);
    const ItemPlan& ip = item_plan(t, 1, tau, proj_chunk(t, tau, cdiv(rmax0, tbm0) * cdiv(cmax0, tbn0)));
    MlLevels L{};
    L.nl = tau;
    std::vector<DVec> Wbuf(static_cast<size_t>(tau));
    double flops = 0;
    int rmax = 1, cmax = 0;
    for (int i = 0; i < tau; ++i) {
        const int l = 1 + i, R = h.Rl(l);
        const int nc = std::min(s, ncol[static_cast<size_t>(i)]);
        const Partition& pt = t.part(l);
        L.depth[i] = l;
        L.R[i] = nc > 0 ? R : 0;
        L.P[i] = transpose ? h.Ul(l) : h.Vl(l);
        L.Q[i] = nullptr;
        L.ncol[i] = nc;
        if (L.R[i] > 0) {
            out[static_cast<size_t>(i)] = make_dvec(static_cast<size_t>(pt.nseg()) * R * s, false);
            if (ip.nchunks[static_cast<size_t>(i)])
                Wbuf[static_cast<size_t>(i)].alloc(static_cast<size_t>(ip.nchunks[static_cast<size_t>(i)]) * R * s);
            rmax = std::max(rmax, R);
            cmax = std::max(cmax, nc);
        }
        L.T[i] = out[static_cast<size_t>(i)] ? out[static_cast<size_t>(i)]->get() : nullptr;
        L.ws[i] = Wbuf[static_cast<size_t>(i)].get();
        flops += 2.0 * double(n) * L.R[i] * nc;
    }
    if (cmax == 0) return out;
    ProfScope prof(PROF_SEG_TN, flops, 8.0 * double(n) * cmax);
    if (prof_enabled()) prof.key(prof_tag("mlproject s=%d Rmax=%d tr=%d", s, rmax, int(transpose)));
    const int tbm = tile::tile_for(rmax), tbn = tile::tile_for_n(cmax, tbm);
    const int max_tiles_m = (rmax + tbm - 1) / tbm, tiles_n = (cmax + tbn - 1) / tbn;
    ProjArgs pa{L, ip.items.get(), X, ldx, n, s, tiles_n, ZeroRows{}};
    with_tile(tbm, [&](auto TM) {
        with_tile(tbn, [&](auto TN) {
            constexpr int M = decltype(TM)::value, N = decltype(TN)::value;
            if constexpr (tile::shape_ok(M, N)) {
                constexpr int bytes = tile::smem_bytes_t(tile::STAGES, M, N);
                attr_once<k_ml_proj<M, N>>(bytes);
                k_ml_proj<M, N>
                    <<<dim3(unsigned(ip.count), unsigned(max_tiles_m * tiles_n)), THREADS, bytes, c.stream>>>(pa);
            } else {
                throw std::logic_error("hodlr_project: unsupported tile shape");
            }
        });
    });
    HG_LAUNCH();
    ++c.launches;
    if (ip.nred) {
        int maxblk = 0;
        for (int i = 0; i < L.nl; ++i) maxblk = std::max(maxblk, L.R[i] * s);
        ReduceArgs ra{L, ip.rl.get(), ip.ri.get(), ip.rf.get(), ip.rc.get(), s};
        k_ml_reduce<<<dim3(unsigned(cdiv(maxblk, 256)), unsigned(ip.nred)), 256, 0, c.stream>>>(ra);
        HG_LAUNCH();
        ++c.launches;
    }
    return out;
}

}  // namespace hg
