// C ABI of the strong-admissibility H-matrix (hstrong.cuh).
#include <cuda_runtime.h>

#include <functional>

#include "../../include/hodlrgp_b200.h"
#include "hstrong.cuh"

using namespace hg;

// Handle layouts shared with capi.cu.
struct hg_ctx_s {
    Ctx c;
};
struct hg_oracle_s {
    std::unique_ptr<DOracle> o;
};
struct hg_hstrong_s {
    DHStrong h;
};

namespace hg {
hg_status capi_guard(hg_ctx_t ctx, const std::function<void()>& f);
}

extern "C" {

hg_status hg_hstrong_plan(const int64_t* order, int nside, int tau, double eta, int64_t k, int64_t* n_lowrank,
                          int64_t* n_dense, int64_t* lowrank_entries, int64_t* dense_entries, int64_t* stored_doubles) {
    return capi_guard(nullptr, [&] {
        require(order != nullptr, "hstrong: order is required");
        const HsPlan P = hs_plan(reinterpret_cast<const std::int64_t*>(order), nside, tau, eta, int(k));
        i64 le = 0, de = 0, st = 0;
        for (const auto& b : P.lr) {
            const i64 mt = P.tree.level(b.d)[static_cast<size_t>(b.t)].size();
            const i64 ms = P.tree.level(b.d)[static_cast<size_t>(b.s)].size();
            le += mt * ms;
            st += (mt + ms) * k;
        }
        for (const auto& b : P.dn) {
            const i64 e = P.tree.leaves()[static_cast<size_t>(b.t)].size() * P.tree.leaves()[static_cast<size_t>(b.s)].size();
            de += e;
            st += b.t == b.s ? e : 2 * e;  // off-diagonal dense blocks keep their transpose
        }
        *n_lowrank = i64(P.lr.size());
        *n_dense = i64(P.dn.size());
        *lowrank_entries = le;
        *dense_entries = de;
        *stored_doubles = st;
    });
}

hg_status hg_hstrong_build(hg_ctx_t ctx, hg_oracle_t o, int param, const int64_t* order, int nside, int tau,
                           double eta, int64_t k, int power_iters, uint64_t seed, hg_hstrong_t* out) {
    return capi_guard(ctx, [&] {
        require(order != nullptr, "hstrong: order is required");
        auto* h = new hg_hstrong_s{hs_build(*o->o, param, reinterpret_cast<const std::int64_t*>(order), nside, tau,
                                            eta, int(k), power_iters, seed)};
        *out = h;
    });
}

hg_status hg_hstrong_free(hg_hstrong_t h) {
    return capi_guard(nullptr, [&] { delete h; });
}

hg_status hg_hstrong_matvec(hg_ctx_t ctx, hg_hstrong_t h, const double* X, int64_t ldx, int64_t s, double* Y,
                            int64_t ldy, int loc) {
    return capi_guard(ctx, [&] {
        const i64 n = h->h.n();
        require(ldx >= n && ldy >= n && s >= 0, "hstrong matvec: dimension mismatch");
        auto& c = current();
        const size_t bytes = sizeof(double) * size_t(n) * size_t(s);
        if (loc == HG_DEVICE) {
            hs_apply(h->h, X, ldx, int(s), Y, ldy);
            return;
        }
        DVec xd(size_t(n) * size_t(s)), yd(size_t(n) * size_t(s));
        if (bytes) {
            HG_CUDA(cudaMemcpy2DAsync(xd.get(), sizeof(double) * size_t(n), X, sizeof(double) * size_t(ldx),
                                      sizeof(double) * size_t(n), size_t(s), cudaMemcpyHostToDevice, c.stream));
            hs_apply(h->h, xd.get(), n, int(s), yd.get(), n);
            HG_CUDA(cudaMemcpy2DAsync(Y, sizeof(double) * size_t(ldy), yd.get(), sizeof(double) * size_t(n),
                                      sizeof(double) * size_t(n), size_t(s), cudaMemcpyDeviceToHost, c.stream));
        }
        sync();
    });
}

hg_status hg_hstrong_trace_product(hg_ctx_t ctx, hg_hstrong_t a, hg_hstrong_t b, double* out) {
    return capi_guard(ctx, [&] {
        DVec d(1);
        hs_trace_product(a->h, b->h, d.get());
        *out = read_scalar(d.get());
    });
}

hg_status hg_hstrong_blocks(hg_hstrong_t h, int64_t* n_lowrank, int64_t* n_dense, int64_t* bytes) {
    return capi_guard(nullptr, [&] {
        *n_lowrank = i64(h->h.plan.lr.size());
        *n_dense = i64(h->h.plan.dn.size());
        *bytes = i64(h->h.bytes());
    });
}

}  // extern "C"
