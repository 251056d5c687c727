// Forward-model covariance oracles of BASELINE.json configs 2, 3 and 5
// (SURVEY §8f #1), matrix-free on the device; the CPU restatements with the
// same formulas live in oracle/ (models.cpp) and the tests build the same
// matrices densely.
//
// C2 co-kriging (1D): f ~ GP, Matérn nu = 1/2, on the m interior points
// x_i = i h of [0,1] (h = 1/(m+1)); u solves A u = f with the second-order FD
// operator A = tridiag(-1, 2, -1)/h^2 + kappa^2 I (homogeneous Dirichlet).
// Joint vector [u; f] interleaved per point (rows 2i = u_i, 2i+1 = f_i):
//   K = [[A^-1 Kf A^-1, A^-1 Kf], [Kf A^-1, Kf]] + nugget I,
// (BASELINE.json states no nugget, but without one K is numerically singular
// in FP64: K_uu's spectrum decays like the FD symbol^-2 on top of Kf's, cond
// beyond 1e15 at m = 256; the nugget is an explicit parameter, default 1e-6),
//   K V:       w = A^-1 V_u + V_f, z = Kf w,  Y_f = z, Y_u = A^-1 z;
//   dK/dsigma2, dK/dell: the same with Kf -> dKf;
//   dK/dkappa: a = A^-1 V_u, b = A^-1 a, z1 = Kf (a + V_f), z2 = Kf b,
//              Y_u = -2 kappa A^-1 (A^-1 z1 + z2), Y_f = -2 kappa z2
//   (dA/dkappa = 2 kappa I). A^-1 by the Thomas algorithm with factors
//   precomputed once per kappa; both sweeps are first-order linear
//   recurrences evaluated as parallel affine scans on the column resident in
//   shared memory (one CTA per column), with a serial fallback for columns
//   longer than shared memory.
//
// C3/C5 SPDE (2D): u solves (-Lap_h + kappa^2) u = f on the N x N periodic
// grid of the unit square (5-point stencil, h = 1/N), f a stationary
// Matérn nu = 3/2 field. Both operators are diagonal in the 2D DFT:
//   mu(k)  = (4/h^2)(sin^2(pi kx/N) + sin^2(pi ky/N)) + kappa^2,
//   lam_f(k) = sigma2 N^2 s(k) / sum_k' s(k'),  s(k) = (3/ell^2 + 4 pi^2 |k~|^2)^(-5/2)
// (the 2D Matérn 3/2 spectral density at the centred integer frequencies
// k~, normalised so that Var f = sigma2 exactly), and
//   K V = IDFT( (lam_f / mu^2 + nugget) . DFT(V) ) / N^2
// (a fixed observation-noise nugget: u alone has cond(K) ~ 1e17 at N = 256,
// singular in FP64, and its weak HODLR at the configs' ranks is positive
// definite only above ~10 Var(u); hodlrgp.py defaults to that)
// with dK/dsigma2 -> lam/sigma2, dK/dell -> d(lam_f)/dell / mu^2 and
// dK/dkappa -> -4 kappa lam_f / mu^3. The rows of V follow the caller's
// point order (e.g. the KD ordering of the grid): order[i] = grid index
// iy*N + ix of row i. cuFFT D2Z/Z2D, batched over the columns.
#include <cufft.h>

#include <cmath>
#include <map>
#include <mutex>

#include "oracle.cuh"
#include "prof.cuh"

namespace hg {

#define HG_CUFFT(x)                                                                                \
    do {                                                                                           \
        cufftResult r_ = (x);                                                                      \
        if (r_ != CUFFT_SUCCESS)                                                                   \
            throw ::hg::CudaError(std::string(#x) + " failed: cufft status " + std::to_string(int(r_))); \
    } while (0)

namespace {

// ------------------------------------------------------------- Thomas solve
constexpr int TH_R = 64;

/// X = A^-1 D, A = tridiag(a, b, a): d'_0 = d_0 im_0, d'_i = (d_i - a d'_{i-1}) im_i,
/// x_{n-1} = d'_{n-1}, x_i = d'_i - cp_i x_{i+1} (im_i = 1/m_i, cp_i = a im_i).
/// One thread per column; 64-row tiles of the panel and of the factors are
/// staged through shared memory (coalesced global traffic, and the serial
/// recurrence only touches shared memory). D and X may alias.
__global__ void __launch_bounds__(32) k_thomas(int n, int s, double a, const double* cp, const double* im,
                                               const double* D, i64 ldd, double* X, i64 ldx) {
    __shared__ double tile[TH_R][33];
    __shared__ double fac[TH_R];
    const int c0 = blockIdx.x * 32, lane = threadIdx.x;
    double prev = 0.0;
    for (int r0 = 0; r0 < n; r0 += TH_R) {
        const int rows = min(TH_R, n - r0);
        for (int cc = 0; cc < 32; ++cc) {
            const int cl = c0 + cc;
            for (int r = lane; r < rows; r += 32) tile[r][cc] = cl < s ? D[i64(r0 + r) + i64(cl) * ldd] : 0.0;
        }
        for (int r = lane; r < rows; r += 32) fac[r] = im[r0 + r];
        __syncwarp();
        for (int r = 0; r < rows; ++r) {
            const double d = tile[r][lane];
            prev = (r0 + r == 0 ? d : d - a * prev) * fac[r];
            tile[r][lane] = prev;
        }
        __syncwarp();
        for (int cc = 0; cc < 32; ++cc) {
            const int cl = c0 + cc;
            if (cl < s)
                for (int r = lane; r < rows; r += 32) X[i64(r0 + r) + i64(cl) * ldx] = tile[r][cc];
        }
        __syncwarp();
    }
    double next = 0.0;
    for (int r0 = ((n - 1) / TH_R) * TH_R; r0 >= 0; r0 -= TH_R) {
        const int rows = min(TH_R, n - r0);
        for (int cc = 0; cc < 32; ++cc) {
            const int cl = c0 + cc;
            for (int r = lane; r < rows; r += 32) tile[r][cc] = cl < s ? X[i64(r0 + r) + i64(cl) * ldx] : 0.0;
        }
        for (int r = lane; r < rows; r += 32) fac[r] = cp[r0 + r];
        __syncwarp();
        for (int r = rows - 1; r >= 0; --r) {
            const double x = r0 + r == n - 1 ? tile[r][lane] : tile[r][lane] - fac[r] * next;
            tile[r][lane] = x;
            next = x;
        }
        __syncwarp();
        for (int cc = 0; cc < 32; ++cc) {
            const int cl = c0 + cc;
            if (cl < s)
                for (int r = lane; r < rows; r += 32) X[i64(r0 + r) + i64(cl) * ldx] = tile[r][cc];
        }
        __syncwarp();
    }
}

/// Thomas solve with the column resident in shared memory and both sweeps as
/// parallel scans: the forward sweep y_i = alpha_i y_{i-1} + im_i d_i
/// (alpha_i = -a im_i) and the backward sweep x_i = d'_i - cp_i x_{i+1} are
/// first-order linear recurrences, so each of 256 threads reduces its run of
/// rows to an affine map (A, B), the maps are combined by a Kogge-Stone scan,
/// and every run is replayed from its carry-in. One CTA per column.
constexpr int TS_THR = 256;

__device__ __forceinline__ void affine_scan(double& A, double& B, double* sA, double* sB, bool reverse) {
    const int t = threadIdx.x;
    const int me = reverse ? TS_THR - 1 - t : t;  // position in scan order
    sA[me] = A;
    sB[me] = B;
    __syncthreads();
    for (int off = 1; off < TS_THR; off <<= 1) {
        double a1 = 1.0, b1 = 0.0;
        const bool take = me >= off;
        if (take) {
            a1 = sA[me - off];
            b1 = sB[me - off];
        }
        __syncthreads();
        if (take) {  // (A, B) o (a1, b1): x -> A (a1 x + b1) + B
            sB[me] = A * b1 + B;
            sA[me] = A * a1;
            A = sA[me];
            B = sB[me];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(TS_THR) k_thomas_col(int n, double a, const double* cp, const double* im,
                                                       const double* D, i64 ldd, double* X, i64 ldx) {
    extern __shared__ double col[];  // n
    __shared__ double sA[TS_THR], sB[TS_THR];
    const int c = blockIdx.x, t = threadIdx.x;
    const double* d = D + i64(c) * ldd;
    double* x = X + i64(c) * ldx;
    for (int i = t; i < n; i += TS_THR) col[i] = d[i];
    __syncthreads();
    const int per = (n + TS_THR - 1) / TS_THR;
    const int r0 = min(n, t * per), r1 = min(n, r0 + per);
    // forward: y_i = (d_i - a y_{i-1}) im_i
    double A = 1.0, B = 0.0;
    for (int i = r0; i < r1; ++i) {
        const double al = i == 0 ? 0.0 : -a * im[i];
        A *= al;
        B = al * B + im[i] * col[i];
    }
    affine_scan(A, B, sA, sB, false);
    double y = t == 0 ? 0.0 : sB[t - 1];  // carry-in: state after the previous run
    __syncthreads();
    for (int i = r0; i < r1; ++i) {
        y = (i == 0 ? col[i] : col[i] - a * y) * im[i];
        col[i] = y;
    }
    __syncthreads();
    // backward: x_i = d'_i - cp_i x_{i+1}, runs in reverse order
    A = 1.0;
    B = 0.0;
    for (int i = r1 - 1; i >= r0; --i) {
        const double al = i == n - 1 ? 0.0 : -cp[i];
        A *= al;
        B = al * B + col[i];
    }
    affine_scan(A, B, sA, sB, true);
    const int me = TS_THR - 1 - t;
    double xn = me == 0 ? 0.0 : sB[me - 1];
    __syncthreads();
    for (int i = r1 - 1; i >= r0; --i) {
        xn = i == n - 1 ? col[i] : col[i] - cp[i] * xn;
        col[i] = xn;
    }
    __syncthreads();
    for (int i = t; i < n; i += TS_THR) x[i] = col[i];
}

/// Rows 2i (u) and 2i+1 (f) of an interleaved panel <-> two m-row panels.
__global__ void k_deinterleave(int m, int s, const double* V, i64 ldv, double* U, double* F) {
    const i64 tot = i64(m) * s;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += i64(gridDim.x) * blockDim.x) {
        const int i = int(e % m), c = int(e / m);
        U[e] = V[2 * i64(i) + i64(c) * ldv];
        F[e] = V[2 * i64(i) + 1 + i64(c) * ldv];
    }
}
__global__ void k_interleave(int m, int s, const double* U, const double* F, double au, double af, double* Y,
                             i64 ldy) {
    const i64 tot = i64(m) * s;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += i64(gridDim.x) * blockDim.x) {
        const int i = int(e % m), c = int(e / m);
        Y[2 * i64(i) + i64(c) * ldy] = au * U[e];
        Y[2 * i64(i) + 1 + i64(c) * ldy] = af * F[e];
    }
}

int grid_blocks(i64 tot) { return int(std::min<i64>((tot + 255) / 256, 148 * 16)); }

class CoKrigingOracle : public DOracle {
public:
    CoKrigingOracle(i64 m, double sigma2, double ell, double kappa, double nugget)
        : DOracle(2 * m, 3), m_(m), sigma2_(sigma2), ell_(ell), kappa_(-1.0), nugget_(nugget) {
        if (m < 2) throw std::invalid_argument("co-kriging: need at least 2 interior points");
        const double h = 1.0 / double(m + 1);
        std::vector<double> x(static_cast<size_t>(m));
        for (i64 i = 0; i < m; ++i) x[static_cast<size_t>(i)] = double(i + 1) * h;
        kf_ = make_matern_oracle(m, x.data(), 1, sigma2, ell, 0.0, true);
        set_kappa(kappa);
    }
    void set_parameters(const double* th, int p) override {
        if (p != 3) throw std::invalid_argument("co-kriging: theta = (sigma2, ell, kappa)");
        sigma2_ = th[0];
        ell_ = th[1];
        kf_->set_parameters(th, 2);
        set_kappa(th[2]);
    }

protected:
    void do_apply(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy) const override {
        if (j >= 3) throw std::invalid_argument("apply_derivative: parameter index");
        auto& c = current();
        ProfScope prof(PROF_ORACLE, 0.0, 0.0);
        const size_t ms = static_cast<size_t>(m_) * static_cast<size_t>(s);
        DVec vu(ms), vf(ms), a(ms), z(ms);
        k_deinterleave<<<grid_blocks(i64(ms)), 256, 0, c.stream>>>(int(m_), s, V, ldv, vu.get(), vf.get());
        HG_LAUNCH();
        solve(vu.get(), a.get(), s);  // a = A^-1 V_u
        if (j < 2) {
            panel_axpby(m_, s, 1.0, vf.get(), m_, 1.0, a.get(), m_);  // w = a + V_f
            kf_->apply(j < 0 ? -1 : j, a.get(), m_, s, z.get(), m_);  // z = Kf^(j) w
            solve(z.get(), vu.get(), s);                                // Y_u = A^-1 z
            k_interleave<<<grid_blocks(i64(ms)), 256, 0, c.stream>>>(int(m_), s, vu.get(), z.get(), 1.0, 1.0, Y, ldy);
            if (j < 0 && nugget_ != 0.0) {
                HG_LAUNCH();
                panel_axpby(n_, s, nugget_, V, ldv, 1.0, Y, ldy);
            }
        } else {
            DVec b(ms), z2(ms);
            solve(a.get(), b.get(), s);                                 // b = A^-2 V_u
            panel_axpby(m_, s, 1.0, vf.get(), m_, 1.0, a.get(), m_);  // a + V_f
            kf_->apply(-1, a.get(), m_, s, z.get(), m_);                // z1
            kf_->apply(-1, b.get(), m_, s, z2.get(), m_);               // z2
            solve(z.get(), vu.get(), s);                                // A^-1 z1
            panel_axpby(m_, s, 1.0, z2.get(), m_, 1.0, vu.get(), m_);  // + z2
            solve(vu.get(), vf.get(), s);                               // A^-1 (...)
            k_interleave<<<grid_blocks(i64(ms)), 256, 0, c.stream>>>(int(m_), s, vf.get(), z2.get(), -2.0 * kappa_,
                                                                     -2.0 * kappa_, Y, ldy);
        }
        HG_LAUNCH();
        c.launches += 2;
    }

private:
    void set_kappa(double kappa) {
        if (kappa == kappa_) return;
        kappa_ = kappa;
        const int m = int(m_);
        const double h = 1.0 / double(m + 1);
        a_ = -1.0 / (h * h);
        const double b = 2.0 / (h * h) + kappa * kappa;
        std::vector<double> cp(static_cast<size_t>(m)), im(static_cast<size_t>(m));
        double mm = b;
        im[0] = 1.0 / mm;
        cp[0] = a_ * im[0];
        for (int i = 1; i < m; ++i) {
            mm = b - a_ * cp[static_cast<size_t>(i - 1)];
            im[static_cast<size_t>(i)] = 1.0 / mm;
            cp[static_cast<size_t>(i)] = a_ * im[static_cast<size_t>(i)];
        }
        cp_.upload(cp);
        im_.upload(im);
    }
    void solve(const double* D, double* X, int s) const {
        auto& c = current();
        const size_t smem = static_cast<size_t>(m_) * sizeof(double);
        if (smem <= 200 * 1024) {  // column resident: parallel-scan sweeps, one CTA per column
            static DeviceOnce attr;
            if (attr.first())
                HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_thomas_col),
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            k_thomas_col<<<unsigned(s), TS_THR, smem, c.stream>>>(int(m_), a_, cp_.get(), im_.get(), D, m_, X, m_);
        } else {
            k_thomas<<<unsigned(cdiv(s, 32)), 32, 0, c.stream>>>(int(m_), s, a_, cp_.get(), im_.get(), D, m_, X, m_);
        }
        HG_LAUNCH();
        ++c.launches;
    }
    i64 m_;
    double sigma2_, ell_, kappa_, nugget_, a_ = 0.0;
    std::unique_ptr<DOracle> kf_;
    DVec cp_, im_;
};

// --------------------------------------------------------------- 2D SPDE
__global__ void k_gather(i64 nn, int s, const i64* order, const double* V, i64 ldv, double* G) {
    const i64 tot = nn * s;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += i64(gridDim.x) * blockDim.x) {
        const i64 i = e % nn, c = e / nn;
        G[(order ? order[i] : i) + c * nn] = V[i + c * ldv];
    }
}
__global__ void k_scatter(i64 nn, int s, const i64* order, const double* G, double* Y, i64 ldy) {
    const i64 tot = nn * s;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += i64(gridDim.x) * blockDim.x) {
        const i64 i = e % nn, c = e / nn;
        Y[i + c * ldy] = G[(order ? order[i] : i) + c * nn];
    }
}
__global__ void k_spectral_scale(i64 nh, int s, const double* lam, cufftDoubleComplex* F) {
    const i64 tot = nh * s;
    for (i64 e = i64(blockIdx.x) * blockDim.x + threadIdx.x; e < tot; e += i64(gridDim.x) * blockDim.x) {
        const double l = lam[e % nh];
        F[e].x *= l;
        F[e].y *= l;
    }
}

class Spde2dOracle : public DOracle {
public:
    Spde2dOracle(int N, double sigma2, double ell, double kappa, double nugget, const std::int64_t* order)
        : DOracle(i64(N) * N, 3), N_(N), nugget_(nugget) {
        if (N < 4 || (N & 1)) throw std::invalid_argument("spde2d: grid side must be even and >= 4");
        if (order) {
            std::vector<char> seen(static_cast<size_t>(n_), 0);
            for (i64 i = 0; i < n_; ++i) {
                if (order[i] < 0 || order[i] >= n_ || seen[static_cast<size_t>(order[i])])
                    throw std::invalid_argument("spde2d: order must be a permutation of the grid");
                seen[static_cast<size_t>(order[i])] = 1;
            }
            order_.upload(reinterpret_cast<const long long*>(order), static_cast<size_t>(n_));
        }
        const double th[3] = {sigma2, ell, kappa};
        set_parameters(th, 3);
    }
    ~Spde2dOracle() override {
        for (auto& kv : plans_) {
            cufftDestroy(kv.second.first);
            cufftDestroy(kv.second.second);
        }
    }
    void set_parameters(const double* th, int p) override {
        if (p != 3) throw std::invalid_argument("spde2d: theta = (sigma2, ell, kappa)");
        const double sigma2 = th[0], ell = th[1], kappa = th[2];
        const int N = N_, NH = N / 2 + 1;
        const double h = 1.0 / N, pi = 3.14159265358979323846, a = 3.0 / (ell * ell);
        auto centred = [&](int k) { return double(k <= N / 2 ? k : k - N); };
        // normalisations over the full spectrum
        double S = 0.0, Sd = 0.0;
        for (int ky = 0; ky < N; ++ky)
            for (int kx = 0; kx < N; ++kx) {
                const double b = 4.0 * pi * pi * (centred(kx) * centred(kx) + centred(ky) * centred(ky));
                S += std::pow(a + b, -2.5);
                Sd += 15.0 / (ell * ell * ell) * std::pow(a + b, -3.5);
            }
        std::vector<double> l0(static_cast<size_t>(N) * NH), l1(l0.size()), l2(l0.size()), l3(l0.size());
        const double nn = double(N) * N;
        for (int ky = 0; ky < N; ++ky)
            for (int kx = 0; kx < NH; ++kx) {
                const size_t e = static_cast<size_t>(ky) * NH + kx;
                const double b = 4.0 * pi * pi * (centred(kx) * centred(kx) + centred(ky) * centred(ky));
                const double sk = std::pow(a + b, -2.5), dsk = 15.0 / (ell * ell * ell) * std::pow(a + b, -3.5);
                const double sx = std::sin(pi * kx / N), sy = std::sin(pi * ky / N);
                const double mu = 4.0 / (h * h) * (sx * sx + sy * sy) + kappa * kappa;
                const double lf = sigma2 * nn * sk / S;
                const double dlf = sigma2 * nn * (dsk * S - sk * Sd) / (S * S);
                // cuFFT Z2D is unnormalised: fold 1/N^2 into the multipliers
                l0[e] = (lf / (mu * mu) + nugget_) / nn;
                l1[e] = lf / sigma2 / (mu * mu) / nn;
                l2[e] = dlf / (mu * mu) / nn;
                l3[e] = -4.0 * kappa * lf / (mu * mu * mu) / nn;
            }
        lam_[0].upload(l0);
        lam_[1].upload(l1);
        lam_[2].upload(l2);
        lam_[3].upload(l3);
    }

protected:
    void do_apply(int j, const double* V, i64 ldv, int s, double* Y, i64 ldy) const override {
        if (j >= 3) throw std::invalid_argument("apply_derivative: parameter index");
        auto& c = current();
        ProfScope prof(PROF_ORACLE, 0.0, 0.0);
        const i64 nn = n_, nh = i64(N_) * (N_ / 2 + 1);
        DVec G(static_cast<size_t>(nn) * static_cast<size_t>(s));
        DBuf<cufftDoubleComplex> F(static_cast<size_t>(nh) * static_cast<size_t>(s));
        const i64* ord = order_.empty() ? nullptr : reinterpret_cast<const i64*>(order_.get());
        k_gather<<<grid_blocks(nn * s), 256, 0, c.stream>>>(nn, s, ord, V, ldv, G.get());
        HG_LAUNCH();
        const auto& pl = plans(s);
        HG_CUFFT(cufftExecD2Z(pl.first, G.get(), F.get()));
        k_spectral_scale<<<grid_blocks(nh * s), 256, 0, c.stream>>>(nh, s, lam_[j + 1].get(), F.get());
        HG_LAUNCH();
        HG_CUFFT(cufftExecZ2D(pl.second, F.get(), G.get()));
        k_scatter<<<grid_blocks(nn * s), 256, 0, c.stream>>>(nn, s, ord, G.get(), Y, ldy);
        HG_LAUNCH();
        c.launches += 5;
    }

private:
    const std::pair<cufftHandle, cufftHandle>& plans(int s) const {
        std::lock_guard<std::mutex> lk(mu_);
        auto it = plans_.find(s);
        if (it == plans_.end()) {
            int dims[2] = {N_, N_};
            cufftHandle f, b;
            HG_CUFFT(cufftPlanMany(&f, 2, dims, nullptr, 1, N_ * N_, nullptr, 1, N_ * (N_ / 2 + 1), CUFFT_D2Z, s));
            HG_CUFFT(cufftPlanMany(&b, 2, dims, nullptr, 1, N_ * (N_ / 2 + 1), nullptr, 1, N_ * N_, CUFFT_Z2D, s));
            it = plans_.emplace(s, std::make_pair(f, b)).first;
        }
        HG_CUFFT(cufftSetStream(it->second.first, current().stream));
        HG_CUFFT(cufftSetStream(it->second.second, current().stream));
        return it->second;
    }
    int N_;
    double nugget_;
    DBuf<long long> order_;
    DVec lam_[4];
    mutable std::mutex mu_;
    mutable std::map<int, std::pair<cufftHandle, cufftHandle>> plans_;
};

}  // namespace

std::unique_ptr<DOracle> make_cokriging_oracle(i64 m, double sigma2, double ell, double kappa, double nugget) {
    return std::make_unique<CoKrigingOracle>(m, sigma2, ell, kappa, nugget);
}

std::unique_ptr<DOracle> make_spde2d_oracle(int N, double sigma2, double ell, double kappa, double nugget,
                                            const std::int64_t* order) {
    return std::make_unique<Spde2dOracle>(N, sigma2, ell, kappa, nugget, order);
}

}  // namespace hg
