// Device covariance oracles: dense matrices, 1D Matérn (dense on-the-fly and
// O(n s) chunked moments, matern_chunk.cuh), user callbacks. Reference interface: oracle.hpp:15-143.
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

#include "matern_chunk.cuh"

class MaternOracle : public DOracle {
public:
    MaternOracle(i64 n, const double* x, int nu2, double sigma2, double ell, double nugget, bool scan)
        : DOracle(n, 2), nu2_(nu2), sigma2_(sigma2), ell_(ell), nugget_(nugget), scan_(scan) {
        if (nu2 != 1 && nu2 != 3 && nu2 != 5) throw std::invalid_argument("Matern: nu in {1/2, 3/2, 5/2}");
        // the scan recurrence needs sorted points; the dense kernel takes any order
        for (i64 i = 1; scan && i < n; ++i)
            if (x[i] < x[i - 1]) throw std::invalid_argument("Matern: points must be sorted");
        x_.upload(x, static_cast<size_t>(n));
    }
    void set_parameters(const double* th, int p) override {
        if (p != 2) throw std::invalid_argument("Matern: theta = (sigma2, ell)");
        sigma2_ = th[0];
        ell_ = th[1];
    }
    /// K = sigma2 k_nu(d / ell) + nugget I, so dK/dsigma2 = (K - nugget I) / sigma2.
    bool affine_derivative(int j, double* a, double* b) const override {
        if (j != 0 || sigma2_ == 0.0) return false;
        *a = 1.0 / sigma2_;
        *b = -nugget_ / sigma2_;
        return true;
    }

protected:
    void do_apply(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy) const override {
        run(j, V, ldv, s, Y, ldy, ZeroRows{});
    }
    void do_apply_masked(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy, const ZeroRows& z) const override {
        run(j, V, ldv, s, Y, ldy, z);
    }

private:
    void run(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy, const ZeroRows& z) const {
        if (j >= 2) throw std::invalid_argument("apply_derivative: parameter index");
        const Poly P = matern_poly(nu2_, j, sigma2_, ell_);
        auto& c = current();
        ProfScope prof(PROF_ORACLE, scan_ ? 2.0 * double(n_) * s * (MC_ROWS + 4 * P.nt) : 2.0 * double(n_) * n_ * s,
                       24.0 * double(n_) * s);
        if (!scan_) {
            static DeviceOnce attr;
            if (attr.first())
                HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_matern_dense),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, tile::SMEM_BYTES));
            dim3 grid(unsigned(cdiv(n_, BM)), unsigned(cdiv(s, BN)));
            k_matern_dense<<<grid, tile::THREADS, tile::SMEM_BYTES, c.stream>>>(x_.get(), int(n_), P, V, ldv, s, Y,
                                                                                ldy);
            HG_LAUNCH();
            ++c.launches;
            if (j < 0 && nugget_ != 0.0) panel_axpby(n_, s, nugget_, V, ldv, 1.0, Y, ldy);
            return;
        }
        const int nsup = cdiv(n_, MC_TILE);
        const size_t msz = static_cast<size_t>(nsup) * static_cast<size_t>(s) * 4;
        DVec Lf(msz), Lb(msz), Ff(msz), Fb(msz);
        MatChunkArgs g{x_.get(), int(n_), nsup, s, P.nt, P.lambda, {P.c[0], P.c[1], P.c[2], P.c[3]},
                       j < 0 ? nugget_ : 0.0, V, ldv, Y, ldy, Lf.get(), Lb.get(), Ff.get(), Fb.get(),
                       z.bounds, z.nseg, z.parity, z.out_depth >= 0 ? 1 : 0};
        static DeviceOnce attr;
        if (attr.first()) {
            HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_mat_moments),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(MC_SMEM)));
            HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_mat_apply),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(MC_SMEM)));
        }
        const dim3 grid(static_cast<unsigned>(nsup), 1u);
        k_mat_moments<<<grid, MC_TILE, MC_SMEM, c.stream>>>(g);
        HG_LAUNCH();
        k_mat_carry<<<dim3(unsigned(s), 2), MC_CARRY_THREADS, 0, c.stream>>>(g);
        HG_LAUNCH();
        k_mat_apply<<<grid, MC_TILE, MC_SMEM, c.stream>>>(g);
        HG_LAUNCH();
        c.launches += 3;
    }

    int nu2_;
    double sigma2_, ell_, nugget_;
    bool scan_;
    DVec x_;
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

/// Row gather/scatter of a column-major panel: dst[perm? ...] (see PermutedOracle).
__global__ void k_permute_rows(i64 n, int s, const i64* p, const double* src, i64 lds, double* dst, i64 ldd,
                               int scatter) {
    const i64 i = i64(blockIdx.x) * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (i >= n || c >= s) return;
    if (scatter)
        dst[p[i] + c * ldd] = src[i + c * lds];  // reordered layout -> base layout
    else
        dst[i + c * ldd] = src[p[i] + c * lds];  // base layout -> reordered layout
}

/// PermutedOracle (oracle.hpp:58-111): K'(i, j) = K(p_i, p_j) with p mapping
/// reordered positions to base indices; V is scattered into the base layout,
/// the base oracle applied (its counters advance too, like base_.apply), and
/// the result gathered back. The base must outlive this view.
class PermutedOracle : public DOracle {
public:
    PermutedOracle(DOracle* base, const std::int64_t* to_base) : DOracle(base->dim(), base->num_params()), base_(base) {
        std::vector<i64> p(to_base, to_base + n_);  // int64_t -> i64
        std::vector<char> seen(static_cast<size_t>(n_), 0);
        for (i64 v : p) {
            if (v < 0 || v >= n_ || seen[static_cast<size_t>(v)])
                throw std::invalid_argument("PermutedOracle: permutation size mismatch");
            seen[static_cast<size_t>(v)] = 1;
        }
        p_.upload(p);
    }
    void set_parameters(const double* theta, int p) override { base_->set_parameters(theta, p); }

protected:
    void do_apply(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy) const override {
        DVec W(static_cast<size_t>(n_) * s), Z(static_cast<size_t>(n_) * s);
        dim3 grid(unsigned(cdiv(n_, 256)), unsigned(s));
        k_permute_rows<<<grid, 256, 0, current().stream>>>(n_, s, p_.get(), V, ldv, W.get(), n_, 1);
        HG_LAUNCH();
        count_launch();
        base_->apply(j, W.get(), n_, s, Z.get(), n_);
        k_permute_rows<<<grid, 256, 0, current().stream>>>(n_, s, p_.get(), Z.get(), n_, Y, ldy, 0);
        HG_LAUNCH();
        count_launch();
    }

private:
    DOracle* base_;
    DBuf<i64> p_;
};

}  // namespace

std::unique_ptr<DOracle> make_permuted_oracle(DOracle* base, const std::int64_t* to_base) {
    return std::make_unique<PermutedOracle>(base, to_base);
}

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
