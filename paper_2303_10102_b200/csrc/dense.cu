// Exact dense evaluation on the device: dense_exact (mle.cpp:345-380), the
// dense branch of fit_mle's Evaluator (mle.cpp:128-175) and accuracy_metrics
// (mle.cpp:382-403). Not the hot path: it is the n <= 2^13 accuracy
// reference the paper's tables compare the HODLR evaluation against, so the
// Cholesky factor and its solves are cuSOLVER's (a plain library
// factorization, like cuBLAS for plain GEMMs); the traces and Fisher sums
// reuse the deterministic reductions of gemm.cu.
#include <cusolverDn.h>

#include <cmath>
#include <map>
#include <mutex>

#include "dense.cuh"
#include "kernels.cuh"
#include "tree.cuh"

#define HG_SOLVER(x)                                                                                       \
    do {                                                                                                   \
        cusolverStatus_t s_ = (x);                                                                         \
        if (s_ != CUSOLVER_STATUS_SUCCESS)                                                                 \
            throw ::hg::CudaError(std::string(#x) + " failed: cusolver status " + std::to_string(int(s_))); \
    } while (0)

namespace hg {

namespace {

constexpr double kLog2Pi = 1.8378770664093454836;
constexpr i64 kDenseGuard = i64(1) << 13;  // mle.cpp:348

cusolverDnHandle_t solver() {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, cusolverDnHandle_t> handles;
    std::lock_guard<std::mutex> lk(mu);
    auto& c = current();
    auto key = std::make_pair(c.device, c.stream);
    auto it = handles.find(key);
    if (it != handles.end()) return it->second;
    cusolverDnHandle_t h;
    HG_SOLVER(cusolverDnCreate(&h));
    HG_SOLVER(cusolverDnSetStream(h, c.stream));
    handles[key] = h;
    return h;
}

int blocks_for(i64 tot) { return int(std::min<i64>((tot + 255) / 256, 148 * 16)); }

__global__ void k_eye(i64 n, double* A) {
    const i64 tot = n * n;
    for (i64 e = blockIdx.x * i64(blockDim.x) + threadIdx.x; e < tot; e += i64(gridDim.x) * blockDim.x)
        A[e] = (e % (n + 1) == 0) ? 1.0 : 0.0;
}

__global__ void k_diag(i64 n, const double* A, double* d) {
    const i64 i = blockIdx.x * i64(blockDim.x) + threadIdx.x;
    if (i < n) d[i] = A[i + i * n];
}

/// part[c][i] = sum_{j in chunk c} A(i, j) x(j): rows across threads
/// (coalesced column reads), column chunks across blockIdx.y.
__global__ void k_gemv_part(int n, const double* __restrict__ A, const double* __restrict__ x, int jchunk,
                            double* __restrict__ part) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int j0 = blockIdx.y * jchunk, j1 = min(n, j0 + jchunk);
    double acc = 0.0;
    for (int j = j0; j < j1; ++j) acc = fma(A[i + i64(j) * n], x[j], acc);
    part[i64(blockIdx.y) * n + i] = acc;
}

__global__ void k_sum_parts(int n, int nc, const double* __restrict__ part, double* __restrict__ y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double acc = 0.0;
    for (int c = 0; c < nc; ++c) acc += part[i64(c) * n + i];
    y[i] = acc;
}

void eye(i64 n, double* A) {
    k_eye<<<blocks_for(n * n), 256, 0, current().stream>>>(n, A);
    HG_LAUNCH();
    count_launch();
}

/// y = A x (A n x n column-major), deterministic.
void gemv(int n, const double* A, const double* x, double* y) {
    constexpr int NC = 32;
    const int jchunk = (n + NC - 1) / NC;
    DVec part(static_cast<size_t>(n) * NC);
    auto& c = current();
    k_gemv_part<<<dim3(static_cast<unsigned>((n + 127) / 128), static_cast<unsigned>(NC)), 128, 0, c.stream>>>(
        n, A, x, jchunk, part.get());
    HG_LAUNCH();
    k_sum_parts<<<(n + 255) / 256, 256, 0, c.stream>>>(n, NC, part.get(), y);
    HG_LAUNCH();
    c.launches += 2;
}

/// Lower Cholesky of K = oracle.apply(I) (Eigen::LLT, mle.cpp:352-353).
struct DenseChol {
    i64 n;
    DVec I, L;
    explicit DenseChol(const DOracle& o) : n(o.dim()) {
        const size_t nn = static_cast<size_t>(n) * static_cast<size_t>(n);
        I.alloc(nn);
        L.alloc(nn);
        eye(n, I.get());
        o.apply(-1, I.get(), n, int(n), L.get(), n);
        auto h = solver();
        int lwork = 0;
        HG_SOLVER(cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, int(n), L.get(), int(n), &lwork));
        DVec work(static_cast<size_t>(std::max(lwork, 1)));
        DBuf<int> info(1);
        HG_SOLVER(cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, int(n), L.get(), int(n), work.get(), lwork, info.get()));
        int hinfo = 0;
        HG_CUDA(cudaMemcpyAsync(&hinfo, info.get(), sizeof(int), cudaMemcpyDeviceToHost, current().stream));
        sync();
        if (hinfo != 0) throw NotPositiveDefinite("dense covariance not SPD");
    }
    void solve(double* B, int s) const {
        DBuf<int> info(1);
        HG_SOLVER(cusolverDnDpotrs(solver(), CUBLAS_FILL_MODE_LOWER, int(n), s, L.get(), int(n), B, int(n), info.get()));
    }
    double logdet() const {  // sum_i 2 log L_ii in index order (mle.cpp:358)
        DVec d(static_cast<size_t>(n));
        k_diag<<<int((n + 255) / 256), 256, 0, current().stream>>>(n, L.get(), d.get());
        HG_LAUNCH();
        count_launch();
        std::vector<double> h = d.download();
        double ld = 0.0;
        for (double v : h) ld += 2.0 * std::log(v);
        return ld;
    }
};

/// Residual copy, w = K^-1 r, and the log-likelihood.
double loglik_and_w(const DenseChol& c, const double* r, DVec& w, double* rw_dev) {
    const i64 n = c.n;
    w.alloc(static_cast<size_t>(n));
    HG_CUDA(cudaMemcpyAsync(w.get(), r, sizeof(double) * static_cast<size_t>(n), cudaMemcpyDeviceToDevice,
                            current().stream));
    c.solve(w.get(), 1);
    dot_panels(n, 1, r, n, w.get(), n, rw_dev, false);
    const double ld = c.logdet();  // synchronizes
    return -0.5 * double(n) * kLog2Pi - 0.5 * ld - 0.5 * read_scalar(rw_dev);
}

/// Host LLT of a small SPD matrix (Eigen::LLT semantics: fails on a
/// non-positive pivot). Returns false on failure.
bool small_llt(const std::vector<double>& A, int p, std::vector<double>& L) {
    L.assign(static_cast<size_t>(p) * p, 0.0);
    for (int j = 0; j < p; ++j) {
        double d = A[j + j * p];
        for (int k = 0; k < j; ++k) d -= L[j + k * p] * L[j + k * p];
        if (!(d > 0.0)) return false;
        L[j + j * p] = std::sqrt(d);
        for (int i = j + 1; i < p; ++i) {
            double v = A[i + j * p];
            for (int k = 0; k < j; ++k) v -= L[i + k * p] * L[j + k * p];
            L[i + j * p] = v / L[j + j * p];
        }
    }
    return true;
}

std::vector<double> llt_solve(const std::vector<double>& L, int p, std::vector<double> b, int s) {
    for (int c = 0; c < s; ++c) {
        double* x = b.data() + static_cast<size_t>(c) * p;
        for (int i = 0; i < p; ++i) {
            for (int k = 0; k < i; ++k) x[i] -= L[i + k * p] * x[k];
            x[i] /= L[i + i * p];
        }
        for (int i = p - 1; i >= 0; --i) {
            for (int k = i + 1; k < p; ++k) x[i] -= L[k + i * p] * x[k];
            x[i] /= L[i + i * p];
        }
    }
    return b;
}

/// Eigen::PartialPivLU(A).solve(I) for small p (no throw on singular input).
std::vector<double> lu_inverse(std::vector<double> A, int p) {
    std::vector<int> piv(static_cast<size_t>(p));
    for (int k = 0; k < p; ++k) {
        int m = k;
        for (int i = k + 1; i < p; ++i)
            if (std::abs(A[i + k * p]) > std::abs(A[m + k * p])) m = i;
        piv[k] = m;
        if (m != k)
            for (int j = 0; j < p; ++j) std::swap(A[k + j * p], A[m + j * p]);
        const double d = A[k + k * p];
        if (d != 0.0)
            for (int i = k + 1; i < p; ++i) A[i + k * p] /= d;
        for (int j = k + 1; j < p; ++j)
            for (int i = k + 1; i < p; ++i) A[i + j * p] -= A[i + k * p] * A[k + j * p];
    }
    std::vector<double> X(static_cast<size_t>(p) * p, 0.0);
    for (int i = 0; i < p; ++i) X[i + i * p] = 1.0;
    for (int c = 0; c < p; ++c) {
        double* x = X.data() + static_cast<size_t>(c) * p;
        for (int k = 0; k < p; ++k) std::swap(x[k], x[piv[k]]);
        for (int i = 0; i < p; ++i)
            for (int k = 0; k < i; ++k) x[i] -= A[i + k * p] * x[k];
        for (int i = p - 1; i >= 0; --i) {
            for (int k = i + 1; k < p; ++k) x[i] -= A[i + k * p] * x[k];
            x[i] /= A[i + i * p];
        }
    }
    return X;
}

}  // namespace

// mle.cpp:345-380
DenseExact dense_exact(const DOracle& o, const double* r) {
    const i64 n = o.dim();
    if (n > kDenseGuard) throw std::length_error("dense_exact: n exceeds dense guard");
    const int p = o.num_params();
    const size_t nn = static_cast<size_t>(n) * static_cast<size_t>(n);
    DenseChol c(o);
    // scalars: [r.w | w.Kj w (p) | tr M_j (p) | sum M_i .* M_j^T (p x p)]
    DVec sc(static_cast<size_t>(1 + 2 * p + p * p));
    sc.zero();
    DVec w;
    DenseExact out;
    out.loglik = loglik_and_w(c, r, w, sc.get());
    std::vector<DVec> M(static_cast<size_t>(p));
    DVec y(static_cast<size_t>(n));
    const Partition& whole = uniform_partition(1, int(n));
    for (int j = 0; j < p; ++j) {
        DVec& m = M[static_cast<size_t>(j)];
        m.alloc(nn);
        o.apply(j, c.I.get(), n, int(n), m.get(), n);  // K_j
        gemv(int(n), m.get(), w.get(), y.get());
        dot_panels(n, 1, w.get(), n, y.get(), n, sc.get() + 1 + j, false);
        c.solve(m.get(), int(n));  // K^-1 K_j
        leaf_trace(whole, m.get(), 0, int(n), sc.get() + 1 + p + j, false);
    }
    for (int i = 0; i < p; ++i)
        for (int j = i; j < p; ++j)
            seg_pair_dot(1, 0, M[static_cast<size_t>(i)].get(), 0, int(n), int(n), int(n), M[static_cast<size_t>(j)].get(),
                         0, int(n), sc.get() + 1 + 2 * p + i + j * p, false);
    const std::vector<double> h = sc.download();
    out.score.resize(static_cast<size_t>(p));
    out.fisher.assign(static_cast<size_t>(p) * p, 0.0);
    for (int j = 0; j < p; ++j) out.score[j] = -0.5 * h[1 + p + j] + 0.5 * h[1 + j];
    for (int i = 0; i < p; ++i)
        for (int j = i; j < p; ++j) {
            const double t = 0.5 * h[1 + 2 * p + i + j * p];
            out.fisher[i + j * p] = t;
            out.fisher[j + i * p] = t;
        }
    return out;
}

double dense_objective(const DOracle& o, const double* r) {
    DenseChol c(o);
    DVec w, sc(1);
    return -loglik_and_w(c, r, w, sc.get());
}

double dense_objective_grad(const DOracle& o, const double* r, std::vector<double>& grad) {
    const i64 n = o.dim();
    const int p = o.num_params();
    const size_t nn = static_cast<size_t>(n) * static_cast<size_t>(n);
    DenseChol c(o);
    DVec sc(static_cast<size_t>(1 + 2 * p));
    sc.zero();
    DVec w;
    const double ll = loglik_and_w(c, r, w, sc.get());
    DVec kinv(nn), kj(nn), y(static_cast<size_t>(n));
    HG_CUDA(cudaMemcpyAsync(kinv.get(), c.I.get(), sizeof(double) * nn, cudaMemcpyDeviceToDevice, current().stream));
    c.solve(kinv.get(), int(n));
    for (int j = 0; j < p; ++j) {
        o.apply(j, c.I.get(), n, int(n), kj.get(), n);
        dot_panels(n, int(n), kinv.get(), n, kj.get(), n, sc.get() + 1 + j, false);
        gemv(int(n), kj.get(), w.get(), y.get());
        dot_panels(n, 1, w.get(), n, y.get(), n, sc.get() + 1 + p + j, false);
    }
    const std::vector<double> h = sc.download();
    grad.resize(static_cast<size_t>(p));
    for (int j = 0; j < p; ++j) grad[j] = -(-0.5 * h[1 + j] + 0.5 * h[1 + p + j]);
    return -ll;
}

// mle.cpp:382-403
AccuracyMetrics accuracy_metrics(double loglik, const std::vector<double>& se, const std::vector<double>& fe,
                                 double loglik_approx, const std::vector<double>& sa, const std::vector<double>& fa) {
    const int p = int(se.size());
    if (int(sa.size()) != p || int(fe.size()) != p * p || int(fa.size()) != p * p)
        throw std::invalid_argument("accuracy_metrics: dimension mismatch");
    auto nrm = [](const std::vector<double>& v) {
        double s = 0.0;
        for (double x : v) s += x * x;
        return std::sqrt(s);
    };
    AccuracyMetrics out;
    std::vector<double> ds(static_cast<size_t>(p)), di(static_cast<size_t>(p) * p);
    for (int i = 0; i < p; ++i) ds[i] = se[i] - sa[i];
    for (int e = 0; e < p * p; ++e) di[e] = fe[e] - fa[e];
    out.eps_L = std::abs(loglik - loglik_approx) / std::abs(loglik);
    out.eps_S = nrm(ds) / nrm(se);
    out.eps_I = nrm(di) / nrm(fe);
    std::vector<double> L;
    if (!small_llt(fe, p, L)) throw std::invalid_argument("accuracy_metrics: exact Fisher not SPD");
    const std::vector<double> x = llt_solve(L, p, ds, 1);
    double g = 0.0;
    for (int i = 0; i < p; ++i) g += ds[i] * x[i];
    out.eta_g = std::sqrt(g);
    std::vector<double> I(static_cast<size_t>(p) * p, 0.0);
    for (int i = 0; i < p; ++i) I[i + i * p] = 1.0;
    const std::vector<double> inv_e = llt_solve(L, p, I, p), inv_a = lu_inverse(fa, p);
    double tr = 0.0;  // trace(di (inv_e - inv_a))
    for (int i = 0; i < p; ++i)
        for (int k = 0; k < p; ++k) tr += di[i + k * p] * (inv_e[k + i * p] - inv_a[k + i * p]);
    out.eta_I = std::sqrt(std::max(0.0, tr));
    return out;
}

}  // namespace hg
