// Device covariance oracles: dense matrices, 1D Matérn (dense on-the-fly and
// O(n) scan), user callbacks. Reference interface: oracle.hpp:15-143.
#include <cmath>

#include "oracle.cuh"
#include "prof.cuh"
#include "tile.cuh"

namespace hg {

void gemm_nn(i64 m, int n, int k, const double* A, i64 lda, const double* B, i64 ldb, double* C, i64 ldc,
             double alpha, double beta) {
    const Partition& p = get_tree(m, 0)->part(0);
    seg_nn(p, A, lda, k, B, 0, int(ldb), TMap::same(), C, ldc, n, alpha, beta);
}

namespace {

// ------------------------------------------------------------------ dense
class DenseOracle : public DOracle {
public:
    DenseOracle(i64 n, const double* K, int p, const double* dK) : DOracle(n, p) {
        k_.upload(K, static_cast<size_t>(n) * static_cast<size_t>(n));
        if (p) dk_.upload(dK, static_cast<size_t>(p) * static_cast<size_t>(n) * static_cast<size_t>(n));
    }

protected:
    void do_apply(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy) const override {
        if (j >= p_) throw std::invalid_argument("apply_derivative: parameter index");
        if (j >= 0 && p_ == 0) {
            panel_axpby(n_, s, 0.0, nullptr, 0, 0.0, Y, ldy);
            return;
        }
        const double* M = j < 0 ? k_.get() : dk_.get() + i64(j) * n_ * n_;
        gemm_nn(n_, s, int(n_), M, n_, V, ldv, Y, ldy, 1.0, 0.0);
    }

private:
    DVec k_, dk_;
};

// ----------------------------------------------------------------- Matérn
/// exp(-lambda d) * sum_m c[m] d^m (same table as oracle/hodlr.cpp).
struct Poly {
    double lambda;
    double c[4];
    int nt;
};

Poly matern_poly(int nu2, int which, double sigma2, double ell) {
    Poly P{};
    const double cnu = nu2 == 1 ? 1.0 : (nu2 == 3 ? std::sqrt(3.0) : std::sqrt(5.0));
    P.lambda = cnu / ell;
    const double L = P.lambda, s = which == 0 ? 1.0 : sigma2;
    if (which <= 0) {
        P.c[0] = s;
        if (nu2 >= 3) P.c[1] = s * L;
        if (nu2 == 5) P.c[2] = s * L * L / 3.0;
        P.nt = nu2 == 1 ? 1 : (nu2 == 3 ? 2 : 3);
    } else if (nu2 == 1) {
        P.c[1] = s * L / ell;
        P.nt = 2;
    } else if (nu2 == 3) {
        P.c[2] = s * L * L / ell;
        P.nt = 3;
    } else {
        P.c[2] = s * L * L / (3.0 * ell);
        P.c[3] = s * L * L * L / (3.0 * ell);
        P.nt = 4;
    }
    return P;
}

__device__ __forceinline__ double poly_eval(const Poly& P, double d) {
    double p = 0.0, dm = 1.0;
    for (int m = 0; m < P.nt; ++m) {
        p += P.c[m] * dm;
        dm *= d;
    }
    return p * exp(-P.lambda * d);
}

using tile::BK;
using tile::BM;
using tile::BN;

/// Kernel tile K(r0 + m, kt*BK + k) computed straight into the m-contiguous
/// shared layout (a computing loader for tile::run).
struct LoadMatern {
    static constexpr bool KC = false;
    static constexpr int ROWS = 64;
    const double* x;
    int r0, n;
    Poly P;
    __device__ __forceinline__ void issue(double* S, int kt) const {
        const int m = threadIdx.x & 63;
        const double xr = r0 + m < n ? x[r0 + m] : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int k = (threadIdx.x >> 6) + 2 * q, kk = kt * BK + k;
            S[k * tile::LD_MC + m] = (r0 + m < n && kk < n) ? poly_eval(P, fabs(xr - x[kk])) : 0.0;
        }
    }
};

/// Y = K V with K(i,j) = k(|x_i - x_j|) formed tile by tile in shared memory.
__global__ void __launch_bounds__(tile::THREADS) k_matern_dense(const double* x, int n, Poly P, const double* V,
                                                                i64 ldv, int s, double* Y, i64 ldy) {
    extern __shared__ double smem[];
    const int r0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    LoadMatern la{x, r0, n, P};
    tile::LoadKC lb{V + i64(n0) * ldv, ldv, n, s - n0};
    tile::Acc acc;
    acc.zero();
    tile::run(la, lb, (n + BK - 1) / BK, smem, acc);
    tile::for_each(acc, [&](int mi, int ni, double v) {
        const int r = r0 + mi, c = n0 + ni;
        if (r < n && c < s) Y[i64(r) + i64(c) * ldy] = v;
    });
}

__device__ __forceinline__ void propagate(double* st, int nt, double d, double rho) {
    // st_m <- rho * sum_{q<=m} C(m,q) d^{m-q} st_q
    // All four moments are carried (branch-free); coefficients past the
    // kernel's degree are zero, so the extra moments never reach the output.
    (void)nt;
    const double d2 = d * d;
    const double n3 = st[3] + 3.0 * d * st[2] + 3.0 * d2 * st[1] + d2 * d * st[0];
    const double n2 = st[2] + 2.0 * d * st[1] + d2 * st[0];
    const double n1 = st[1] + d * st[0];
    st[0] *= rho;
    st[1] = rho * n1;
    st[2] = rho * n2;
    st[3] = rho * n3;
}

__global__ void k_steps(const double* x, int n, double lambda, double* dx, double* rho) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double d = i > 0 ? x[i] - x[i - 1] : 0.0;
        dx[i] = d;
        rho[i] = exp(-lambda * d);
    }
}

struct ScanArgs {
    const double* dx;   // dx[i] = x_i - x_{i-1}
    const double* rho;  // exp(-lambda dx[i])
    const double* x;
    int n, ch, nch, s, nt;
    const double* V;
    i64 ldv;
    double* Y;
    i64 ldy;
    double* locF;  // [col][chunk][4]
    double* locB;
    double c[4];
    double diag;  // added to the diagonal: nugget (value) - c0 (double-counted self term)
    double lambda;
};

// Block-cooperative scan: a CTA owns one chunk of SC_CH rows x 32 columns,
// staged in shared memory (coalesced); warp w scans rows [32w, 32w+32) of
// every column (lane = column), sub-chunk summaries are combined by one warp.
constexpr int SC_SUB = 32, SC_WARPS = 16, SC_CH = SC_SUB * SC_WARPS, SC_LD = 33;

struct ScanSmem {
    double* Vs;   // SC_CH x SC_LD
    double* dxs;  // SC_CH + 1
    double* rhs;  // SC_CH + 1
    double* sub;  // 2 x SC_WARPS x 32 x 4 (forward / backward summaries)
    double* cin;  // 2 x SC_WARPS x 32 x 4 (carry-ins)
};

__device__ ScanSmem scan_smem(double* sm) {
    ScanSmem s;
    s.Vs = sm;
    s.dxs = s.Vs + SC_CH * SC_LD;
    s.rhs = s.dxs + SC_CH + 1;
    s.sub = s.rhs + SC_CH + 1;
    s.cin = s.sub + 2 * SC_WARPS * 32 * 4;
    return s;
}

/// Stage V[lo:hi, c0:c0+32] and the step tables; local sub-chunk scans.
__device__ void scan_stage(const ScanArgs& g, const ScanSmem& S, int lo, int rows, int c0) {
    for (int e = threadIdx.x; e < rows * 32; e += blockDim.x) {
        const int r = e % rows, cc = e / rows, col = c0 + cc;
        S.Vs[r * SC_LD + cc] = col < g.s ? g.V[i64(lo + r) + i64(col) * g.ldv] : 0.0;
    }
    for (int r = threadIdx.x; r <= rows; r += blockDim.x) {
        const bool in = lo + r < g.n;
        S.dxs[r] = in ? g.dx[lo + r] : 0.0;
        S.rhs[r] = in ? g.rho[lo + r] : 1.0;
    }
    __syncthreads();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = w * SC_SUB, r1 = min(rows, r0 + SC_SUB);
    double st[4] = {0, 0, 0, 0};
    for (int r = r0; r < r1; ++r) {
        if (r > r0) propagate(st, g.nt, S.dxs[r], S.rhs[r]);
        st[0] += S.Vs[r * SC_LD + lane];
    }
    double* f = S.sub + ((0 * SC_WARPS + w) * 32 + lane) * 4;
    for (int m = 0; m < 4; ++m) f[m] = st[m];
    for (int m = 0; m < 4; ++m) st[m] = 0.0;
    for (int r = r1 - 1; r >= r0; --r) {
        if (r < r1 - 1) propagate(st, g.nt, S.dxs[r + 1], S.rhs[r + 1]);
        st[0] += S.Vs[r * SC_LD + lane];
    }
    double* b = S.sub + ((1 * SC_WARPS + w) * 32 + lane) * 4;
    for (int m = 0; m < 4; ++m) b[m] = st[m];
    __syncthreads();
}

__global__ void __launch_bounds__(SC_CH) k_scan_local(ScanArgs g) {
    extern __shared__ double sm[];
    const ScanSmem S = scan_smem(sm);
    const int chunk = blockIdx.x, c0 = blockIdx.y * 32;
    const int lo = chunk * g.ch, rows = min(g.n, lo + g.ch) - lo;
    scan_stage(g, S, lo, rows, c0);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, col = c0 + lane;
    const int nsub = (rows + SC_SUB - 1) / SC_SUB;
    if (w == 0 && col < g.s) {  // chunk forward summary at its last point
        double st[4];
        for (int m = 0; m < 4; ++m) st[m] = S.sub[(0 * 32 + lane) * 4 + m];
        for (int v = 1; v < nsub; ++v) {
            const double d = g.x[lo + min(rows, (v + 1) * SC_SUB) - 1] - g.x[lo + v * SC_SUB - 1];
            propagate(st, g.nt, d, exp(-g.lambda * d));
            for (int m = 0; m < 4; ++m) st[m] += S.sub[((0 * SC_WARPS + v) * 32 + lane) * 4 + m];
        }
        double* o = g.locF + (i64(col) * g.nch + chunk) * 4;
        for (int m = 0; m < 4; ++m) o[m] = st[m];
    } else if (w == 1 && col < g.s) {  // chunk backward summary at its first point
        double st[4];
        for (int m = 0; m < 4; ++m) st[m] = S.sub[((1 * SC_WARPS + nsub - 1) * 32 + lane) * 4 + m];
        for (int v = nsub - 2; v >= 0; --v) {
            const double d = g.x[lo + (v + 1) * SC_SUB] - g.x[lo + v * SC_SUB];
            propagate(st, g.nt, d, exp(-g.lambda * d));
            for (int m = 0; m < 4; ++m) st[m] += S.sub[((1 * SC_WARPS + v) * 32 + lane) * 4 + m];
        }
        double* o = g.locB + (i64(col) * g.nch + chunk) * 4;
        for (int m = 0; m < 4; ++m) o[m] = st[m];
    }
}

/// Carries: locF[c] becomes the full forward state at the chunk's last point,
/// locB[c] the full backward state at its first point (sequential per column;
/// the chunk-to-chunk transfer exp(-lambda dx) is recomputed from x).
__global__ void k_scan_carry(ScanArgs g, double lambda) {
    // One CTA per column: chunk summaries staged in shared memory, the
    // forward carry run by warp 0's lane 0 and the backward one by warp 1's.
    extern __shared__ double sh[];
    const int col = blockIdx.x, nch = g.nch;
    double* F = g.locF + i64(col) * nch * 4;
    double* B = g.locB + i64(col) * nch * 4;
    double* sF = sh;
    double* sB = sh + 4 * nch;
    double* xe = sh + 8 * nch;  // x at each chunk's last point
    double* xs = sh + 9 * nch;  // x at each chunk's first point
    for (int e = threadIdx.x; e < 4 * nch; e += blockDim.x) {
        sF[e] = F[e];
        sB[e] = B[e];
    }
    for (int c = threadIdx.x; c < nch; c += blockDim.x) {
        xe[c] = g.x[min(g.n, (c + 1) * g.ch) - 1];
        xs[c] = g.x[c * g.ch];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double st[4] = {sF[0], sF[1], sF[2], sF[3]};
        for (int c = 1; c < nch; ++c) {
            const double d = xe[c] - xe[c - 1];
            propagate(st, g.nt, d, exp(-lambda * d));
            for (int m = 0; m < 4; ++m) {
                st[m] += sF[c * 4 + m];
                sF[c * 4 + m] = st[m];
            }
        }
    } else if (threadIdx.x == 32) {
        double st[4];
        for (int m = 0; m < 4; ++m) st[m] = sB[(nch - 1) * 4 + m];
        for (int c = nch - 2; c >= 0; --c) {
            const double d = xs[c + 1] - xs[c];
            propagate(st, g.nt, d, exp(-lambda * d));
            for (int m = 0; m < 4; ++m) {
                st[m] += sB[c * 4 + m];
                sB[c * 4 + m] = st[m];
            }
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 4 * nch; e += blockDim.x) {
        F[e] = sF[e];
        B[e] = sB[e];
    }
}

__global__ void __launch_bounds__(SC_CH) k_scan_final(ScanArgs g) {
    extern __shared__ double sm[];
    const ScanSmem S = scan_smem(sm);
    const int chunk = blockIdx.x, c0 = blockIdx.y * 32;
    const int lo = chunk * g.ch, rows = min(g.n, lo + g.ch) - lo;
    scan_stage(g, S, lo, rows, c0);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, col = c0 + lane;
    const int nsub = (rows + SC_SUB - 1) / SC_SUB;
    // Carry-ins of every sub-chunk: forward state at the row before it,
    // backward state at the row after it (chunk carries from k_scan_carry).
    if (w == 0) {
        double st[4] = {0, 0, 0, 0};
        if (chunk > 0 && col < g.s)
            for (int m = 0; m < 4; ++m) st[m] = g.locF[(i64(col) * g.nch + chunk - 1) * 4 + m];
        double xprev = lo > 0 ? g.x[lo - 1] : g.x[0];
        for (int v = 0; v < nsub; ++v) {
            for (int m = 0; m < 4; ++m) S.cin[((0 * SC_WARPS + v) * 32 + lane) * 4 + m] = st[m];
            const double xend = g.x[lo + min(rows, (v + 1) * SC_SUB) - 1];
            const double d = xend - xprev;
            propagate(st, g.nt, d, exp(-g.lambda * d));
            for (int m = 0; m < 4; ++m) st[m] += S.sub[((0 * SC_WARPS + v) * 32 + lane) * 4 + m];
            xprev = xend;
        }
    } else if (w == 1) {
        double st[4] = {0, 0, 0, 0};
        if (chunk < g.nch - 1 && col < g.s)
            for (int m = 0; m < 4; ++m) st[m] = g.locB[(i64(col) * g.nch + chunk + 1) * 4 + m];
        double xnext = lo + rows < g.n ? g.x[lo + rows] : g.x[g.n - 1];
        for (int v = nsub - 1; v >= 0; --v) {
            for (int m = 0; m < 4; ++m) S.cin[((1 * SC_WARPS + v) * 32 + lane) * 4 + m] = st[m];
            const double xs = g.x[lo + v * SC_SUB];
            const double d = xnext - xs;
            propagate(st, g.nt, d, exp(-g.lambda * d));
            for (int m = 0; m < 4; ++m) st[m] += S.sub[((1 * SC_WARPS + v) * 32 + lane) * 4 + m];
            xnext = xs;
        }
    }
    __syncthreads();
    const int r0 = w * SC_SUB, r1 = min(rows, r0 + SC_SUB);
    double aF[SC_SUB];
    double st[4];
    for (int m = 0; m < 4; ++m) st[m] = S.cin[((0 * SC_WARPS + w) * 32 + lane) * 4 + m];
#pragma unroll
    for (int q = 0; q < SC_SUB; ++q) {
        const int r = r0 + q;
        if (r < r1) {
            if (lo + r > 0) propagate(st, g.nt, S.dxs[r], S.rhs[r]);
            st[0] += S.Vs[r * SC_LD + lane];
            double a = 0.0;
            a = g.c[0] * st[0] + g.c[1] * st[1] + g.c[2] * st[2] + g.c[3] * st[3];
            aF[q] = a;
        }
    }
    for (int m = 0; m < 4; ++m) st[m] = S.cin[((1 * SC_WARPS + w) * 32 + lane) * 4 + m];
#pragma unroll
    for (int q = SC_SUB - 1; q >= 0; --q) {
        const int r = r0 + q;
        if (r < r1) {
            if (lo + r < g.n - 1) propagate(st, g.nt, S.dxs[r + 1], S.rhs[r + 1]);
            const double v = S.Vs[r * SC_LD + lane];
            st[0] += v;
            double a = 0.0;
            a = g.c[0] * st[0] + g.c[1] * st[1] + g.c[2] * st[2] + g.c[3] * st[3];
            S.Vs[r * SC_LD + lane] = aF[q] + a + g.diag * v;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < rows * 32; e += blockDim.x) {
        const int r = e % rows, cc = e / rows, cl = c0 + cc;
        if (cl < g.s) g.Y[i64(lo + r) + i64(cl) * g.ldy] = S.Vs[r * SC_LD + cc];
    }
}

class MaternOracle : public DOracle {
public:
    MaternOracle(i64 n, const double* x, int nu2, double sigma2, double ell, double nugget, bool scan)
        : DOracle(n, 2), nu2_(nu2), sigma2_(sigma2), ell_(ell), nugget_(nugget), scan_(scan) {
        if (nu2 != 1 && nu2 != 3 && nu2 != 5) throw std::invalid_argument("Matern: nu in {1/2, 3/2, 5/2}");
        for (i64 i = 1; i < n; ++i)
            if (x[i] < x[i - 1]) throw std::invalid_argument("Matern: points must be sorted");
        x_.upload(x, static_cast<size_t>(n));
        dx_.alloc(static_cast<size_t>(n));
        rho_.alloc(static_cast<size_t>(n));
    }
    void set_parameters(const double* th, int p) override {
        if (p != 2) throw std::invalid_argument("Matern: theta = (sigma2, ell)");
        sigma2_ = th[0];
        ell_ = th[1];
        cached_lambda_ = -1.0;
    }

protected:
    void do_apply(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy) const override {
        if (j >= 2) throw std::invalid_argument("apply_derivative: parameter index");
        const Poly P = matern_poly(nu2_, j, sigma2_, ell_);
        auto& c = current();
        ProfScope prof(PROF_ORACLE, scan_ ? 4.0 * double(n_) * s * P.nt * P.nt : 2.0 * double(n_) * n_ * s,
                       16.0 * double(n_) * s);
        if (!scan_) {
            static bool attr = false;
            if (!attr) {
                HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_matern_dense),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, tile::SMEM_BYTES));
                attr = true;
            }
            dim3 grid(unsigned(cdiv(n_, BM)), unsigned(cdiv(s, BN)));
            k_matern_dense<<<grid, tile::THREADS, tile::SMEM_BYTES, c.stream>>>(x_.get(), int(n_), P, V, ldv, s, Y,
                                                                                ldy);
            HG_LAUNCH();
            ++c.launches;
            if (j < 0 && nugget_ != 0.0) panel_axpby(n_, s, nugget_, V, ldv, 1.0, Y, ldy);
            return;
        }
        if (cached_lambda_ != P.lambda) {
            k_steps<<<cdiv(n_, 256), 256, 0, c.stream>>>(x_.get(), int(n_), P.lambda, dx_.get(), rho_.get());
            HG_LAUNCH();
            ++c.launches;
            cached_lambda_ = P.lambda;
        }
        const int ch = SC_CH;
        const int nch = cdiv(n_, ch);
        const size_t csm = static_cast<size_t>(nch) * 10 * sizeof(double);
        if (csm > 220 * 1024) throw std::length_error("Matern scan: n above 2^21 not supported");
        DVec locF(static_cast<size_t>(nch) * static_cast<size_t>(s) * 4),
            locB(static_cast<size_t>(nch) * static_cast<size_t>(s) * 4);
        ScanArgs g{dx_.get(), rho_.get(), x_.get(), int(n_), ch, nch, s, P.nt, V, ldv, Y, ldy, locF.get(),
                   locB.get(), {P.c[0], P.c[1], P.c[2], P.c[3]}, (j < 0 ? nugget_ : 0.0) - P.c[0], P.lambda};
        const size_t ssm = (static_cast<size_t>(SC_CH) * SC_LD + 2 * (SC_CH + 1) + 4 * SC_WARPS * 32 * 4) *
                           sizeof(double);
        static bool attr = false;
        if (!attr) {
            HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_scan_local),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(ssm)));
            HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_scan_final),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(ssm)));
            HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_scan_carry),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            attr = true;
        }
        dim3 grid(unsigned(nch), unsigned(cdiv(s, 32)));
        k_scan_local<<<grid, SC_CH, ssm, c.stream>>>(g);
        HG_LAUNCH();
        k_scan_carry<<<s, 256, csm, c.stream>>>(g, P.lambda);
        HG_LAUNCH();
        k_scan_final<<<grid, SC_CH, ssm, c.stream>>>(g);
        HG_LAUNCH();
        c.launches += 3;
    }

private:
    int nu2_;
    double sigma2_, ell_, nugget_;
    bool scan_;
    DVec x_;
    mutable DVec dx_, rho_;
    mutable double cached_lambda_ = -1.0;
};

class CallbackOracle : public DOracle {
public:
    CallbackOracle(i64 n, int p, ApplyFn fn, void* user) : DOracle(n, p), fn_(fn), user_(user) {}

protected:
    void do_apply(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy) const override {
        if (fn_(user_, j, V, ldv, s, Y, ldy, current().stream) != 0)
            throw std::runtime_error("oracle callback failed");
    }

private:
    ApplyFn fn_;
    void* user_;
};

}  // namespace

std::unique_ptr<DOracle> make_dense_oracle(i64 n, const double* K, int p, const double* dK) {
    return std::make_unique<DenseOracle>(n, K, p, dK);
}

std::unique_ptr<DOracle> make_matern_oracle(i64 n, const double* x, int nu2, double sigma2, double ell,
                                            double nugget, bool scan) {
    return std::make_unique<MaternOracle>(n, x, nu2, sigma2, ell, nugget, scan);
}

std::unique_ptr<DOracle> make_callback_oracle(i64 n, int p, ApplyFn fn, void* user) {
    return std::make_unique<CallbackOracle>(n, p, fn, user);
}

}  // namespace hg
