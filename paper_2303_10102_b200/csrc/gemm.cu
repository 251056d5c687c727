// Segmented FP64 GEMM engine and deterministic reductions (see kernels.cuh).
//
// Tile engine (tile.cuh): a TBM x TBN output tile per 128-thread CTA on the
// FP64 tensor cores (DMMA m8n8k4), the tile shape picked per call from the
// problem's M and N, K staged 16 at a time through a cp.async pipeline.
// Split-K partials are reduced in a fixed order so every result is bitwise
// reproducible run to run.
#include <cstdlib>
#include "kernels.cuh"
#include "prof.cuh"
#include "tile.cuh"

namespace hg {

namespace {

using tile::Acc;
using tile::BK;
using tile::BM;
using tile::BN;
using tile::THREADS;
__device__ __forceinline__ int cdiv_d(int a, int b) { return (a + b - 1) / b; }
// Short-K GEMMs (seg_nn: k = rank; leaf_mm: k = leaf size) are latency-bound:
// two stages (40 KB) keep five CTAs resident per SM instead of three.
constexpr int NS_SHORT = 2;
constexpr int SEG_CHUNK = 512;  // rows per split-K work item
constexpr int RED_BLOCKS = 296; // 2 x 148 SMs; fixed => deterministic reductions

// ------------------------------------------------------------------ seg_tn
struct SegTnArgs {
    const double* A;
    i64 lda;
    int ca;
    const double* B;
    i64 ldb;
    int cb;
    const WorkItem* items;
    int tiles_m;
    double* out;
    i64 ostride;
    int ldo;
    int direct;
    double alpha, beta;
};

/// T_s tile = A[rows]^T B[rows]: both operands k-contiguous (rows = k).
template <int TBM, int TBN>
__global__ void __launch_bounds__(THREADS) k_seg_tn(SegTnArgs g) {
    extern __shared__ double smem[];
    const WorkItem it = g.items[blockIdx.x];
    const int m0 = (blockIdx.y % g.tiles_m) * TBM, n0 = (blockIdx.y / g.tiles_m) * TBN;
    tile::LoadKCT<TBM> la{g.A + it.row0 + i64(m0) * g.lda, g.lda, it.rows, g.ca - m0};
    tile::LoadKCT<TBN> lb{g.B + it.row0 + i64(n0) * g.ldb, g.ldb, it.rows, g.cb - n0};
    typename tile::Shape<TBM, TBN>::Acc acc;
    acc.zero();
    tile::run_t<tile::STAGES, TBM, TBN>(la, lb, cdiv_d(it.rows, BK), smem, acc);
    double* o = g.out + (g.direct ? i64(it.seg) : i64(blockIdx.x)) * g.ostride;
    tile::for_each_t<TBM, TBN>(acc, [&](int mi, int ni, double v) {
        const int m = m0 + mi, n = n0 + ni;
        if (m >= g.ca || n >= g.cb) return;
        double* p = o + m + i64(n) * g.ldo;
        if (g.direct)
            *p = g.alpha * v + (g.beta != 0.0 ? g.beta * *p : 0.0);
        else
            *p = v;
    });
}

__global__ void k_seg_reduce(const double* ws, i64 wstride, int ca, int cb, const int* seg_first, double* T,
                             i64 tstride, int ldt, double alpha, double beta) {
    const int s = blockIdx.y;
    const i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= i64(ca) * cb) return;
    double sum = 0.0;
    for (int c = seg_first[s]; c < seg_first[s + 1]; ++c) sum += ws[i64(c) * wstride + e];
    const int m = int(e % ca), n = int(e / ca);
    double* t = T + i64(s) * tstride + m + i64(n) * ldt;
    *t = alpha * sum + (beta != 0.0 ? beta * *t : 0.0);
}

// ------------------------------------------------------------------ seg_nn
struct SegNnArgs {
    const double* X;
    i64 ldx;
    int k;
    const double* T;
    i64 tstride;
    int ldt;
    TMap map;
    double* Y;
    i64 ldy;
    int w;
    const WorkItem* items;
    double alpha, beta;
};

/// Y[rows] = X[rows] T_sel: X m-contiguous (rows = m), T k-contiguous.
template <int TBM, int TBN>
__global__ void __launch_bounds__(THREADS) k_seg_nn(SegNnArgs g) {
    extern __shared__ double smem[];
    const WorkItem it = g.items[blockIdx.x];
    const int n0 = blockIdx.y * TBN;
    const double* Tb = g.T + i64((it.seg >> g.map.shift) ^ g.map.xr) * g.map.mult * g.tstride +
                       i64(g.map.add) * g.tstride + ((it.seg & 1) ? g.map.row_odd : g.map.row_even);
    tile::LoadMCT<TBM> la{g.X + it.row0, g.ldx, it.rows, g.k};
    tile::LoadKCT<TBN> lb{Tb + i64(n0) * g.ldt, g.ldt, g.k, g.w - n0};
    typename tile::Shape<TBM, TBN>::Acc acc;
    acc.zero();
    // The accumulate-into-Y operand is fetched before the (short-K) main loop
    // so its latency overlaps the GEMM instead of trailing it.
    typename tile::Shape<TBM, TBN>::Acc yv;
    yv.zero();
    if (g.beta != 0.0)
        tile::for_each_slot<TBM, TBN>(yv, [&](double& s, int m, int ni) {
            const int n = n0 + ni;
            if (n < g.w && m < it.rows) s = g.Y[i64(it.row0 + m) + i64(n) * g.ldy];
        });
    tile::run_t<NS_SHORT, TBM, TBN>(la, lb, cdiv_d(g.k, BK), smem, acc);
    tile::for_each_slot2<TBM, TBN>(acc, yv, [&](double v, double y, int m, int ni) {
        const int n = n0 + ni;
        if (n >= g.w || m >= it.rows) return;
        g.Y[i64(it.row0 + m) + i64(n) * g.ldy] = g.alpha * v + g.beta * y;
    });
}

/// Streaming variant for short K (k <= 48) and wide w: the CTA keeps its
/// 64-row X tile in shared memory and walks a run of column tiles. The op is
/// HBM-bound (AI = k/8 flop/B): T tiles are staged one ahead with cp.async,
/// and the accumulated Y tile goes straight to registers in the accumulator
/// layout one tile ahead (no shared staging, so three CTAs fit per SM and
/// more of Y is in flight).
constexpr int SNN_KT = 5;  // k <= 80 (k slices of X / T held in shared memory)

template <int TBN, int KT>
struct SnnLayout {
    static constexpr int XE = KT * tile::stage_elems(BM);   // X, all k slices
    static constexpr int TE = KT * tile::stage_elems(TBN);  // T tile, all k slices
    static constexpr int BYTES = int(sizeof(double)) * (XE + 2 * TE);
};

template <int TBN, int KT>
__global__ void __launch_bounds__(THREADS) k_seg_nn_stream(SegNnArgs g, int groups) {
    using Lay = SnnLayout<TBN, KT>;
    using Acc = typename tile::Shape<BM, TBN>::Acc;
    extern __shared__ double smem[];
    double* Xs = smem;
    double* Ts = smem + Lay::XE;  // 2 buffers of TE
    const WorkItem it = g.items[blockIdx.x / groups];
    const int grp = blockIdx.x % groups;
    const int ntiles = cdiv_d(g.w, TBN), per = cdiv_d(ntiles, groups);
    const int j0 = grp * per, j1 = min(ntiles, j0 + per);
    if (j0 >= j1) return;
    const double* Tb = g.T + i64((it.seg >> g.map.shift) ^ g.map.xr) * g.map.mult * g.tstride +
                       i64(g.map.add) * g.tstride + ((it.seg & 1) ? g.map.row_odd : g.map.row_even);
    const int kt_n = cdiv_d(g.k, BK);
    tile::LoadMCT<BM> lx{g.X + it.row0, g.ldx, it.rows, g.k};
    for (int kt = 0; kt < kt_n; ++kt) lx.issue(Xs + kt * tile::stage_elems(BM), kt);
    const bool ld_y = g.beta != 0.0;
    auto issue_t = [&](int j, int buf) {
        const int n0 = j * TBN;
        tile::LoadKCT<TBN> lt{Tb + i64(n0) * g.ldt, g.ldt, g.k, g.w - n0};
        double* T = Ts + buf * Lay::TE;
        for (int kt = 0; kt < kt_n; ++kt) lt.issue(T + kt * tile::stage_elems(TBN), kt);
    };
    auto load_y = [&](int j, Acc& y) {
        const int n0 = j * TBN;
        tile::for_each_slot<BM, TBN>(y, [&](double& v, int m, int ni) {
            const int n = n0 + ni;
            v = (n < g.w && m < it.rows) ? g.Y[i64(it.row0 + m) + i64(n) * g.ldy] : 0.0;
        });
    };
    // Y two tiles ahead in registers (more of the HBM stream in flight per SM)
    Acc ycur, ynext, ynext2;
    if (ld_y) {
        load_y(j0, ycur);
        if (j0 + 1 < j1) load_y(j0 + 1, ynext);
    }
    issue_t(j0, 0);
    tile::cp_commit();
    for (int j = j0; j < j1; ++j) {
        const int buf = (j - j0) & 1;
        tile::cp_wait<0>();
        __syncthreads();  // tile j (and X) landed; every warp is done with the other buffer
        if (j + 1 < j1) issue_t(j + 1, buf ^ 1);
        if (ld_y && j + 2 < j1) load_y(j + 2, ynext2);
        tile::cp_commit();
        Acc acc;
        acc.zero();
        const double* T = Ts + buf * Lay::TE;
        for (int kt = 0; kt < kt_n; ++kt)
            tile::mma_stage<false, true, BM, TBN>(Xs + kt * tile::stage_elems(BM), T + kt * tile::stage_elems(TBN),
                                                  acc);
        const int n0 = j * TBN;
        tile::for_each_slot2<BM, TBN>(acc, ycur, [&](double v, double y, int m, int ni) {
            const int n = n0 + ni;
            if (n >= g.w || m >= it.rows) return;
            g.Y[i64(it.row0 + m) + i64(n) * g.ldy] = g.alpha * v + (ld_y ? g.beta * y : 0.0);
        });
        if (ld_y) {
            ycur = ynext;
            ynext = ynext2;
        }
    }
    tile::cp_wait<0>();
}

// ----------------------------------------------------------------- leaf_mm
struct LeafMmArgs {
    const int* bounds;
    int rt;
    const double* L;
    i64 lstride;
    int ldl;
    const double* X;
    i64 ldx;
    double* Y;
    i64 ldy;
    int w;
    double alpha, beta;
};

/// Y[leaf rows] = op(L_b) X[leaf rows]; op(L) is m-contiguous (no transpose)
/// or k-contiguous (transpose), X is k-contiguous.
template <bool TRANS, int TBN>
__global__ void __launch_bounds__(THREADS) k_leaf_mm(LeafMmArgs g) {
    extern __shared__ double smem[];
    const int b = blockIdx.x / g.rt, mt = blockIdx.x % g.rt;
    const int lo = g.bounds[b], m = g.bounds[b + 1] - lo, r0 = mt * BM;
    if (r0 >= m) return;
    const int n0 = blockIdx.y * TBN;
    const double* Lb = g.L + i64(b) * g.lstride;
    tile::LoadKCT<TBN, false> lb{g.X + lo + i64(n0) * g.ldx, g.ldx, m, g.w - n0};
    typename tile::Shape<BM, TBN>::Acc acc;
    acc.zero();
    typename tile::Shape<BM, TBN>::Acc yv;
    yv.zero();
    if (g.beta != 0.0)  // fetch the accumulated Y before the main loop (latency overlap)
        tile::for_each_slot<BM, TBN>(yv, [&](double& y, int mi0, int ni) {
            const int mi = r0 + mi0, n = n0 + ni;
            if (n < g.w && mi < m) y = g.Y[i64(lo + mi) + i64(n) * g.ldy];
        });
    if (!TRANS) {
        tile::LoadMCT<BM, false> la{Lb + r0, g.ldl, m - r0, m};
        tile::run_t<NS_SHORT, BM, TBN>(la, lb, cdiv_d(m, BK), smem, acc);
    } else {
        tile::LoadKCT<BM, false> la{Lb + i64(r0) * g.ldl, g.ldl, m, m - r0};
        tile::run_t<NS_SHORT, BM, TBN>(la, lb, cdiv_d(m, BK), smem, acc);
    }
    tile::for_each_slot2<BM, TBN>(acc, yv, [&](double v, double y, int mi0, int ni) {
        const int mi = r0 + mi0, n = n0 + ni;
        if (n >= g.w || mi >= m) return;
        g.Y[i64(lo + mi) + i64(n) * g.ldy] = g.alpha * v + g.beta * y;
    });
}

__device__ double block_sum(double v);

/// Partial sums of sum((L_b X) .* Z) over the leaves: the leaf products are
/// never stored (the cross-term leaf part of trace_pair, product_rep.cpp:212-224).
/// Each CTA runs `tiles_per` column tiles of one 64-row leaf tile and writes
/// one partial (fixed order => deterministic).
struct DotZ {
    const double* Z[LEAF_DOT_MAXZ];
    double alpha[LEAF_DOT_MAXZ];
    int nz;
};

template <int TBN>
__global__ void __launch_bounds__(THREADS) k_leaf_mm_dot(LeafMmArgs g, DotZ zs, i64 ldz, int tiles_per,
                                                         double* partial) {
    extern __shared__ double smem[];
    const int b = blockIdx.x / g.rt, mt = blockIdx.x % g.rt;
    const int lo = g.bounds[b], m = g.bounds[b + 1] - lo, r0 = mt * BM;
    double part[LEAF_DOT_MAXZ] = {};
    if (r0 < m) {
        const double* Lb = g.L + i64(b) * g.lstride;
        const int ntiles = cdiv_d(g.w, TBN);
        const int t1 = min(ntiles, int(blockIdx.y + 1) * tiles_per);
        for (int tn = int(blockIdx.y) * tiles_per; tn < t1; ++tn) {
            const int n0 = tn * TBN;
            tile::LoadKCT<TBN, false> lb{g.X + lo + i64(n0) * g.ldx, g.ldx, m, g.w - n0};
            tile::LoadMCT<BM, false> la{Lb + r0, g.ldl, m - r0, m};
            typename tile::Shape<BM, TBN>::Acc acc;
            acc.zero();
            tile::run_t<NS_SHORT, BM, TBN>(la, lb, cdiv_d(m, BK), smem, acc);
            __syncthreads();  // every warp is done with the stages before the next tile refills them
            // one product, dotted with every Z (the product is never stored)
            tile::for_each_slot<BM, TBN>(acc, [&](double& v, int mi0, int ni) {
                const int mi = r0 + mi0, n = n0 + ni;
                if (n < g.w && mi < m)
#pragma unroll
                    for (int z = 0; z < LEAF_DOT_MAXZ; ++z)
                        if (z < zs.nz) part[z] = fma(v, zs.Z[z][i64(lo + mi) + i64(n) * ldz], part[z]);
            });
        }
    }
#pragma unroll
    for (int z = 0; z < LEAF_DOT_MAXZ; ++z) {
        if (z >= zs.nz) break;
        const double sz = block_sum(part[z]);
        if (threadIdx.x == 0)
            partial[i64(z) * gridDim.x * gridDim.y + blockIdx.x + i64(blockIdx.y) * gridDim.x] = zs.alpha[z] * sz;
    }
}

/// Per-leaf Grams M_z,b = A_z[b] B[b]^T (A_z, B: n x K, rows of leaf b, K
/// contracted) dotted with every leaf array L_a: sum_b <L_a,b, M_z,b> =
/// tr(A_z^T L_a B). One CTA per (leaf, 64-row tile, 64-column tile); the
/// partial of (z, a) at partial[(z * nl + a) * nblocks + block].
struct LeafGramArgs {
    const int* bounds;
    int rt;
    const double* A[LEAF_DOT_MAXZ];
    int na;
    const double* B;
    i64 ld;
    int K;
    const double* L[LEAF_DOT_MAXZ];
    int nl;
    i64 lstride;
    int ldl;
};

__global__ void __launch_bounds__(THREADS) k_leaf_gram_dot(const __grid_constant__ LeafGramArgs g, double* partial) {
    extern __shared__ double smem[];
    const int blk = blockIdx.x, rt2 = g.rt * g.rt;
    const int b = blk / rt2, rc = blk % rt2, r0 = (rc / g.rt) * BM, c0 = (rc % g.rt) * BM;
    const int lo = g.bounds[b], m = g.bounds[b + 1] - lo;
    double part[LEAF_DOT_MAXZ][LEAF_DOT_MAXZ] = {};
    if (r0 < m && c0 < m) {
        for (int z = 0; z < g.na; ++z) {
            tile::LoadMCT<BM> la{g.A[z] + lo + r0, g.ld, m - r0, g.K};
            tile::LoadMCT<BM> lb{g.B + lo + c0, g.ld, m - c0, g.K};
            typename tile::Shape<BM, BM>::Acc acc;
            acc.zero();
            tile::run_t<NS_SHORT, BM, BM>(la, lb, cdiv_d(g.K, BK), smem, acc);
            __syncthreads();  // stages free before the next z refills them
            tile::for_each_slot<BM, BM>(acc, [&](double& v, int mi0, int ni) {
                const int r = r0 + mi0, c = c0 + ni;
                if (r < m && c < m)
#pragma unroll
                    for (int a = 0; a < LEAF_DOT_MAXZ; ++a)
                        if (a < g.nl) part[z][a] = fma(v, g.L[a][i64(b) * g.lstride + r + i64(c) * g.ldl], part[z][a]);
            });
        }
    }
    const i64 nb = gridDim.x;
#pragma unroll
    for (int z = 0; z < LEAF_DOT_MAXZ; ++z)
#pragma unroll
        for (int a = 0; a < LEAF_DOT_MAXZ; ++a) {
            if (z >= g.na || a >= g.nl) continue;
            const double sv = block_sum(part[z][a]);
            if (threadIdx.x == 0) partial[i64(z * g.nl + a) * nb + blk] = sv;
        }
}

// ------------------------------------------------------------ elementwise
/// Y = alpha X + beta Y; grid (row blocks, column groups), no 64-bit div/mod.
__global__ void k_axpby(i64 n, int w, double alpha, const double* X, i64 ldx, double beta, double* Y, i64 ldy) {
    for (int j = blockIdx.y; j < w; j += gridDim.y)
        for (i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += i64(gridDim.x) * blockDim.x) {
            double* y = Y + i + j * ldy;
            const double x = X ? alpha * X[i + j * ldx] : 0.0;
            *y = x + (beta != 0.0 ? beta * *y : 0.0);
        }
}

/// Y rows of even segments = ae Xe, of odd segments = ao Xo (a null source
/// writes zeros): each row reads the one source it keeps.
__global__ void k_parity_select(const WorkItem* items, int w, const double* Xe, i64 ldxe, double ae,
                                const double* Xo, i64 ldxo, double ao, double* Y, i64 ldy) {
    const WorkItem it = items[blockIdx.x];
    if (int(threadIdx.x) >= it.rows) return;  // one thread per row (items have <= blockDim rows)
    const bool odd = it.seg & 1;
    const double a = odd ? ao : ae;
    const double* X = odd ? Xo : Xe;
    const i64 ldx = odd ? ldxo : ldxe;
    const i64 row = i64(it.row0) + threadIdx.x;
    double* y = Y + row;
    if (X) {
        const double* x = X + row;
#pragma unroll 4
        for (int j = 0; j < w; ++j) y[i64(j) * ldy] = a * x[i64(j) * ldx];
    } else {
#pragma unroll 4
        for (int j = 0; j < w; ++j) y[i64(j) * ldy] = 0.0;
    }
}

// -------------------------------------------------------------- reductions
__device__ double block_sum(double v) {
    __shared__ double sh[32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    v = (threadIdx.x < (blockDim.x >> 5)) ? sh[lane] : 0.0;
    if (wid == 0)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;  // valid in thread 0
}

struct PairDot {
    int ra, rb, xr, ldg, ldh;
    i64 gs, hs;
    const double *G, *H;
    __device__ double operator()(i64 e) const {
        const i64 per = i64(ra) * rb;
        const int s = int(e / per);
        const int rem = int(e % per), a = rem % ra, b = rem / ra;
        return G[i64(s) * gs + a + i64(b) * ldg] * H[i64(s ^ xr) * hs + b + i64(a) * ldh];
    }
};

struct XorDot {
    int ra, rc, xr, ld;
    i64 gs;
    const double *G, *H;
    __device__ double operator()(i64 e) const {
        const i64 per = i64(ra) * rc;
        const int s = int(e / per);
        const int rem = int(e % per), a = rem % ra, c = rem / ra;
        const i64 o = a + i64(c) * ld;
        return G[i64(s) * gs + o] * H[i64(s ^ xr) * gs + o];
    }
};

struct LeafTrace {
    const int* bounds;
    int bmax, ldl;
    i64 lstride;
    const double* L;
    __device__ double operator()(i64 e) const {
        const int b = int(e / bmax), i = int(e % bmax);
        if (i >= bounds[b + 1] - bounds[b]) return 0.0;
        return L[i64(b) * lstride + i + i64(i) * ldl];
    }
};

struct LeafPair {
    const int* bounds;
    int bmax, ldl;
    i64 lstride;
    const double *A, *B;
    __device__ double operator()(i64 e) const {
        const i64 per = i64(bmax) * bmax;
        const int b = int(e / per);
        const int rem = int(e % per), r = rem % bmax, c = rem / bmax;
        const int m = bounds[b + 1] - bounds[b];
        if (r >= m || c >= m) return 0.0;
        const i64 base = i64(b) * lstride;
        return A[base + c + i64(r) * ldl] * B[base + r + i64(c) * ldl];
    }
};

constexpr int DOT_BLOCKS = 4 * 148;  // fixed => deterministic
constexpr int DOT_CH = 4096;          // elements per chunk (16 per thread)

/// Chunks of DOT_CH elements of every segment, block b taking chunks b, b +
/// DOT_BLOCKS, ... (16 independent loads of each operand per thread in
/// flight, four accumulators); one partial per block.
__global__ void __launch_bounds__(256) k_seg_dot(int nseg, int xr, const double* A, i64 gsa, const double* B,
                                                 i64 gsb, i64 len, double* partial) {
    const i64 cps = (len + DOT_CH - 1) / DOT_CH, nchunk = cps * nseg;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (i64 c = blockIdx.x; c < nchunk; c += gridDim.x) {
        const int s = int(c / cps);
        const i64 e0 = (c - i64(s) * cps) * DOT_CH;
        const double* a = A + i64(s) * gsa + e0;
        const double* b = B + i64(s ^ xr) * gsb + e0;
        const int m = int(min(i64(DOT_CH), len - e0));
        double av[16], bv[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const int e = int(threadIdx.x) + k * 256;
            av[k] = e < m ? __ldcs(a + e) : 0.0;
            bv[k] = e < m ? __ldcs(b + e) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k & 3] = fma(av[k], bv[k], acc[k & 3]);
    }
    double v = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    v = block_sum(v);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

template <class F>
__global__ void k_reduce_partial(F f, i64 total, double* partial) {
    double v = 0.0;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += i64(gridDim.x) * blockDim.x) v += f(e);
    v = block_sum(v);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

__global__ void k_reduce_final(const double* partial, int np, double* out, int accumulate) {
    double v = 0.0;
    for (int i = threadIdx.x; i < np; i += blockDim.x) v += partial[i];
    v = block_sum(v);
    if (threadIdx.x == 0) *out = accumulate ? *out + v : v;
}

template <class F>
void reduce(F f, i64 total, double* out, bool accumulate) {
    auto& c = current();
    DVec partial(RED_BLOCKS);
    k_reduce_partial<<<RED_BLOCKS, 256, 0, c.stream>>>(f, total, partial.get());
    HG_LAUNCH();
    k_reduce_final<<<1, 256, 0, c.stream>>>(partial.get(), RED_BLOCKS, out, accumulate ? 1 : 0);
    HG_LAUNCH();
    c.launches += 2;
}

}  // namespace

void seg_tn(const Partition& p, const double* A, i64 lda, int ca, const double* B, i64 ldb, int cb, double* T,
            i64 tstride, int ldt, double alpha, double beta) {
    if (ca <= 0 || cb <= 0) return;
    auto& c = current();
    const double rows = double(p.hbounds().back() - p.hbounds().front());
    ProfScope prof(PROF_SEG_TN, 2.0 * rows * ca * cb, 8.0 * (rows * (ca + cb) + double(p.nseg()) * ca * cb));
    if (prof_enabled()) prof.key(prof_tag("tn nseg=%d ca=%d cb=%d", p.nseg(), ca, cb));
    int tbm = tile::tile_for(ca), tbn = tile::tile_for(cb);
    if (ca > 32 && ca <= 40 && tbn % 32 == 0)  // 1 x 4 warp grid
        tbm = 40;
    else if (cb > 32 && cb <= 40 && tbm % 32 == 0)  // 4 x 1 warp grid
        tbn = 40;
    const int tiles_m = cdiv(ca, tbm), tiles_n = cdiv(cb, tbn);
    // Split-K chunk: the shortest (from SEG_CHUNK rows, doubling) that still
    // gives >= 8 CTAs per SM; longer chunks write fewer ca x cb partials.
    int chunk = SEG_CHUNK;
    while (chunk < p.max_seg() && (i64(rows) / (2 * chunk)) * tiles_m * tiles_n >= 8 * c.num_sms) chunk *= 2;
    const TileList& tl = p.tiles(chunk);
    SegTnArgs g{A, lda, ca, B, ldb, cb, tl.items.get(), tiles_m, T, tstride, ldt, 1, alpha, beta};
    DVec ws;
    if (!tl.one_per_seg) {
        const i64 wstride = i64(ca) * cb;
        ws.alloc(static_cast<size_t>(wstride) * static_cast<size_t>(tl.count));
        g.out = ws.get();
        g.ostride = wstride;
        g.ldo = ca;
        g.direct = 0;
    }
    const dim3 grid(unsigned(tl.count), unsigned(tiles_m * tiles_n));
    with_tile(tbm, [&](auto TM) {
        with_tile(tbn, [&](auto TN) {
            constexpr int M = decltype(TM)::value, N = decltype(TN)::value;
            if constexpr (tile::shape_ok(M, N)) {
                constexpr int bytes = tile::smem_bytes_t(tile::STAGES, M, N);
                attr_once<k_seg_tn<M, N>>(bytes);
                k_seg_tn<M, N><<<grid, THREADS, bytes, c.stream>>>(g);
            } else {
                throw std::logic_error("seg_tn: unsupported tile shape");
            }
        });
    });
    HG_LAUNCH();
    ++c.launches;
    if (tl.one_per_seg) return;
    const i64 wstride = i64(ca) * cb;
    dim3 rgrid(unsigned(cdiv(wstride, 256)), unsigned(p.nseg()));
    k_seg_reduce<<<rgrid, 256, 0, c.stream>>>(ws.get(), wstride, ca, cb, tl.seg_first.get(), T, tstride, ldt, alpha,
                                              beta);
    HG_LAUNCH();
    ++c.launches;
}

void seg_nn(const Partition& p, const double* X, i64 ldx, int k, const double* T, i64 tstride, int ldt, TMap map,
            double* Y, i64 ldy, int w, double alpha, double beta) {
    if (w <= 0) return;
    auto& c = current();
    if (k <= 0) {
        if (beta != 1.0) panel_axpby(p.hbounds().back(), w, 0.0, nullptr, 0, beta, Y, ldy);
        return;
    }
    const double rows = double(p.hbounds().back() - p.hbounds().front());
    ProfScope prof(PROF_SEG_NN, 2.0 * rows * k * w, 8.0 * rows * (k + (beta != 0.0 ? 2.0 : 1.0) * w));
    if (prof_enabled()) prof.key(prof_tag("nn nseg=%d k=%d w=%d", p.nseg(), k, w));
    // Short K over many columns: the streaming kernel (X tile resident).
    if (k <= BK * SNN_KT && w >= 128 && p.max_seg() > 96 && !std::getenv("HG_NO_NN_STREAM")) {
        constexpr int TN = 32;
        const TileList& tl = p.tiles(BM);
        SegNnArgs g{X, ldx, k, T, tstride, ldt, map, Y, ldy, w, tl.items.get(), alpha, beta};
        const int want = 4 * c.num_sms, ntiles = cdiv(w, TN);
        const int groups = std::max(1, std::min(ntiles / 4, cdiv(want, tl.count)));
        if (k <= 3 * BK) {
            attr_once<k_seg_nn_stream<TN, 3>>(SnnLayout<TN, 3>::BYTES);
            k_seg_nn_stream<TN, 3>
                <<<unsigned(tl.count * groups), THREADS, SnnLayout<TN, 3>::BYTES, c.stream>>>(g, groups);
        } else {
            attr_once<k_seg_nn_stream<TN, 5>>(SnnLayout<TN, 5>::BYTES);
            k_seg_nn_stream<TN, 5>
                <<<unsigned(tl.count * groups), THREADS, SnnLayout<TN, 5>::BYTES, c.stream>>>(g, groups);
        }
        HG_LAUNCH();
        ++c.launches;
        return;
    }
    // Row tile: 64, or one tile per segment when every segment is short
    // (e.g. the 2R-row node blocks of the capacitance solves).
    const int tbm = p.max_seg() <= 96 ? std::max(48, tile::tile_for(p.max_seg())) : BM;
    const TileList& tl = p.tiles(tbm);
    SegNnArgs g{X, ldx, k, T, tstride, ldt, map, Y, ldy, w, tl.items.get(), alpha, beta};
    const int tbn = tile::tile_for_n(w, tbm);
    with_tile(tbm, [&](auto TM) {
        with_tile(tbn, [&](auto TN) {
            constexpr int M = decltype(TM)::value, N = decltype(TN)::value;
            if constexpr ((M == 64 || M == 80 || M == 96 || M == 48) && tile::shape_ok(M, N)) {
                constexpr int bytes = tile::smem_bytes_t(NS_SHORT, M, N);
                attr_once<k_seg_nn<M, N>>(bytes);
                k_seg_nn<M, N><<<dim3(unsigned(tl.count), unsigned(cdiv(w, N))), THREADS, bytes, c.stream>>>(g);
            } else {
                throw std::logic_error("seg_nn: unsupported row tile");
            }
        });
    });
    HG_LAUNCH();
    ++c.launches;
}

void leaf_mm(const Partition& leaves, const double* L, i64 lstride, int ldl, bool trans, const double* X, i64 ldx,
             double* Y, i64 ldy, int w, double alpha, double beta) {
    if (w <= 0) return;
    auto& c = current();
    const int rt = cdiv(leaves.max_seg(), BM);
    const double rows = double(leaves.hbounds().back()), bm = double(leaves.max_seg());
    ProfScope prof(PROF_LEAF_MM, 2.0 * rows * bm * w, 8.0 * (rows * bm + rows * w * (beta != 0.0 ? 3.0 : 2.0)));
    if (prof_enabled()) prof.key(prof_tag("leafmm w=%d tr=%d", w, int(trans)));
    LeafMmArgs g{leaves.dbounds(), rt, L, lstride, ldl, X, ldx, Y, ldy, w, alpha, beta};
    const int tbn = tile::tile_for_n(w, BM);
    with_tile(tbn, [&](auto TN) {
        constexpr int N = decltype(TN)::value;
        constexpr int bytes = tile::smem_bytes_t(NS_SHORT, BM, N);
        const dim3 grid(unsigned(leaves.nseg() * rt), unsigned(cdiv(w, N)));
        if (trans) {
            attr_once<k_leaf_mm<true, N>>(bytes);
            k_leaf_mm<true, N><<<grid, THREADS, bytes, c.stream>>>(g);
        } else {
            attr_once<k_leaf_mm<false, N>>(bytes);
            k_leaf_mm<false, N><<<grid, THREADS, bytes, c.stream>>>(g);
        }
    });
    HG_LAUNCH();
    ++c.launches;
}

void leaf_mm_dot(const Partition& leaves, const double* L, i64 lstride, int ldl, const double* X, i64 ldx,
                 const double* Z, i64 ldz, int w, double alpha, double* out, bool accumulate) {
    leaf_mm_dot_multi(leaves, L, lstride, ldl, X, ldx, {Z}, ldz, w, {alpha}, {out}, accumulate);
}

void leaf_mm_dot_multi(const Partition& leaves, const double* L, i64 lstride, int ldl, const double* X, i64 ldx,
                       const std::vector<const double*>& Zs, i64 ldz, int w, const std::vector<double>& alphas,
                       const std::vector<double*>& outs, bool accumulate) {
    const size_t nzt = Zs.size();
    if (w <= 0) {
        if (!accumulate)
            for (double* o : outs) HG_CUDA(cudaMemsetAsync(o, 0, sizeof(double), current().stream));
        return;
    }
    auto& c = current();
    const int rt = cdiv(leaves.max_seg(), BM);
    const double rows = double(leaves.hbounds().back()), bm = double(leaves.max_seg());
    ProfScope prof(PROF_LEAF_MM, 2.0 * rows * bm * w, 8.0 * (rows * bm + (1.0 + double(nzt)) * rows * w));
    if (prof_enabled()) prof.key(prof_tag("leafmmdot w=%d z=%d", w, int(nzt)));
    LeafMmArgs g{leaves.dbounds(), rt, L, lstride, ldl, X, ldx, nullptr, 0, w, 1.0, 0.0};
    const int tbn = tile::tile_for_n(w, BM);
    for (size_t z0 = 0; z0 < nzt; z0 += LEAF_DOT_MAXZ) {
        DotZ zs{};
        zs.nz = int(std::min<size_t>(LEAF_DOT_MAXZ, nzt - z0));
        for (int z = 0; z < zs.nz; ++z) {
            zs.Z[z] = Zs[z0 + size_t(z)];
            zs.alpha[z] = alphas[z0 + size_t(z)];
        }
        with_tile(tbn, [&](auto TN) {
            constexpr int N = decltype(TN)::value;
            constexpr int bytes = tile::smem_bytes_t(NS_SHORT, BM, N);
            const int ntiles = cdiv(w, N), tiles_per = std::min(ntiles, 4);
            const dim3 grid(unsigned(leaves.nseg() * rt), unsigned(cdiv(ntiles, tiles_per)));
            const i64 np = i64(grid.x) * grid.y;
            DVec partial(static_cast<size_t>(np) * static_cast<size_t>(zs.nz));
            attr_once<k_leaf_mm_dot<N>>(bytes);
            k_leaf_mm_dot<N><<<grid, THREADS, bytes, c.stream>>>(g, zs, ldz, tiles_per, partial.get());
            HG_LAUNCH();
            ++c.launches;
            for (int z = 0; z < zs.nz; ++z) {
                k_reduce_final<<<1, 256, 0, c.stream>>>(partial.get() + i64(z) * np, int(np), outs[z0 + size_t(z)],
                                                        accumulate ? 1 : 0);
                HG_LAUNCH();
                ++c.launches;
            }
        });
    }
}

void leaf_gram_dot(const Partition& leaves, const std::vector<const double*>& As, const double* B, i64 ld, int K,
                   const std::vector<const double*>& Ls, i64 lstride, int ldl, const std::vector<double*>& outs,
                   bool accumulate) {
    const int na = int(As.size()), nl = int(Ls.size());
    if (na > LEAF_DOT_MAXZ || nl > LEAF_DOT_MAXZ) throw std::length_error("leaf_gram_dot: too many operands");
    if (na == 0 || nl == 0) return;
    if (K <= 0) {
        if (!accumulate)
            for (double* o : outs) HG_CUDA(cudaMemsetAsync(o, 0, sizeof(double), current().stream));
        return;
    }
    auto& c = current();
    const int rt = cdiv(leaves.max_seg(), BM);
    const double rows = double(leaves.hbounds().back()), bm = double(leaves.max_seg());
    ProfScope prof(PROF_LEAF_MM, 2.0 * na * rows * bm * K, 8.0 * ((na + 1.0) * rows * K + nl * na * rows * bm));
    if (prof_enabled()) prof.key(prof_tag("leafgram K=%d z=%d l=%d", K, na, nl));
    LeafGramArgs g{};
    g.bounds = leaves.dbounds();
    g.rt = rt;
    for (int z = 0; z < na; ++z) g.A[z] = As[static_cast<size_t>(z)];
    g.na = na;
    g.B = B;
    g.ld = ld;
    g.K = K;
    for (int a = 0; a < nl; ++a) g.L[a] = Ls[static_cast<size_t>(a)];
    g.nl = nl;
    g.lstride = lstride;
    g.ldl = ldl;
    constexpr int bytes = tile::smem_bytes_t(NS_SHORT, BM, BM);
    const unsigned grid = unsigned(leaves.nseg() * rt * rt);
    DVec partial(static_cast<size_t>(grid) * static_cast<size_t>(na * nl));
    attr_once<k_leaf_gram_dot>(bytes);
    k_leaf_gram_dot<<<grid, THREADS, bytes, c.stream>>>(g, partial.get());
    HG_LAUNCH();
    ++c.launches;
    for (int e = 0; e < na * nl; ++e) {
        k_reduce_final<<<1, 256, 0, c.stream>>>(partial.get() + i64(e) * grid, int(grid), outs[static_cast<size_t>(e)],
                                                accumulate ? 1 : 0);
        HG_LAUNCH();
        ++c.launches;
    }
}

void panel_axpby(i64 n, int w, double alpha, const double* X, i64 ldx, double beta, double* Y, i64 ldy) {
    if (n <= 0 || w <= 0) return;
    auto& c = current();
    const int bx = int(std::min<i64>((n + 255) / 256, 148 * 8));
    const int by = std::min(w, std::max(1, (148 * 16) / bx));
    k_axpby<<<dim3(unsigned(bx), unsigned(by)), 256, 0, c.stream>>>(n, w, alpha, X, ldx, beta, Y, ldy);
    HG_LAUNCH();
    ++c.launches;
}

void panel_parity_select(const Partition& p, int w, const double* Xe, i64 ldxe, double a_even, const double* Xo,
                         i64 ldxo, double a_odd, double* Y, i64 ldy) {
    if (w <= 0) return;
    auto& c = current();
    const TileList& tl = p.tiles(256);
    k_parity_select<<<tl.count, 256, 0, c.stream>>>(tl.items.get(), w, Xe, ldxe, a_even, Xo, ldxo, a_odd, Y, ldy);
    HG_LAUNCH();
    ++c.launches;
}

void seg_dot(int nseg, int xr, const double* A, i64 gsa, const double* B, i64 gsb, i64 len, double* out,
             bool accumulate) {
    auto& c = current();
    if (nseg <= 0 || len <= 0) {
        if (!accumulate) HG_CUDA(cudaMemsetAsync(out, 0, sizeof(double), c.stream));
        return;
    }
    ProfScope prof(PROF_REDUCE, 2.0 * double(nseg) * len, 16.0 * double(nseg) * len);
    DVec partial(DOT_BLOCKS);
    k_seg_dot<<<DOT_BLOCKS, 256, 0, c.stream>>>(nseg, xr, A, gsa, B, gsb, len, partial.get());
    HG_LAUNCH();
    k_reduce_final<<<1, 256, 0, c.stream>>>(partial.get(), DOT_BLOCKS, out, accumulate ? 1 : 0);
    HG_LAUNCH();
    c.launches += 2;
}

void dot_panels(i64 n, int w, const double* A, i64 lda, const double* B, i64 ldb, double* out, bool accumulate) {
    if (lda == n && ldb == n)
        seg_dot(1, 0, A, 0, B, 0, n * w, out, accumulate);
    else
        seg_dot(w, 0, A, lda, B, ldb, n, out, accumulate);
}

void seg_pair_dot(int nseg, int xr, const double* G, i64 gs, int ldg, int ra, int rb, const double* H, i64 hs,
                  int ldh, double* out, bool accumulate) {
    reduce(PairDot{ra, rb, xr, ldg, ldh, gs, hs, G, H}, i64(nseg) * ra * rb, out, accumulate);
}

void seg_xor_dot(int nseg, int xr, const double* G, const double* H, i64 gs, int ld, int ra, int rc, double* out,
                 bool accumulate) {
    if (ld == ra) {  // contiguous ra x rc blocks
        seg_dot(nseg, xr, G, gs, H, gs, i64(ra) * rc, out, accumulate);
        return;
    }
    reduce(XorDot{ra, rc, xr, ld, gs, G, H}, i64(nseg) * ra * rc, out, accumulate);
}

void leaf_trace(const Partition& leaves, const double* L, i64 lstride, int ldl, double* out, bool accumulate) {
    reduce(LeafTrace{leaves.dbounds(), leaves.max_seg(), ldl, lstride, L}, i64(leaves.nseg()) * leaves.max_seg(), out,
           accumulate);
}

void leaf_pair_dot(const Partition& leaves, const double* A, const double* B, i64 lstride, int ldl, double* out,
                   bool accumulate) {
    const int bm = leaves.max_seg();
    reduce(LeafPair{leaves.dbounds(), bm, ldl, lstride, A, B}, i64(leaves.nseg()) * bm * bm, out, accumulate);
}

double read_scalar(const double* d) {
    double h = 0;
    HG_CUDA(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, current().stream));
    HG_CUDA(cudaStreamSynchronize(current().stream));
    return h;
}

}  // namespace hg
