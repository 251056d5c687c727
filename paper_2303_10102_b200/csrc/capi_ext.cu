// C ABI: full MLE evaluation on host or device buffers, per-kernel profiling.
#include <cuda_runtime.h>

#include <functional>

#include "../../include/hodlrgp_b200.h"
#include "api.cuh"
#include "prof.cuh"

using namespace hg;

// Handle layouts shared with capi.cu.
struct hg_ctx_s {
    Ctx c;
};
struct hg_oracle_s {
    std::unique_ptr<DOracle> o;
};

namespace hg {
hg_status capi_guard(hg_ctx_t ctx, const std::function<void()>& f);
}

extern "C" {

hg_status hg_mle_evaluate(hg_ctx_t ctx, hg_oracle_t o, int tau, int64_t k, uint64_t seed, const double* y,
                          const double* B, int64_t nrhs, double* X, int loc, double* loglik, double* score_out,
                          double* fisher, double* times) {
    return capi_guard(ctx, [&] {
        auto& c = current();
        const i64 n = o->o->dim();
        DTreeP tree = get_tree(n, tau);
        DSketchPlanP plan = get_plan(tree, k, seed);
        cudaEvent_t ev[7];
        for (auto& e : ev) HG_CUDA(cudaEventCreate(&e));
        HG_CUDA(cudaEventRecord(ev[0], c.stream));
        // inputs (host -> device when loc == HG_HOST)
        DVec ybuf, Bbuf;
        const double* yd = y;
        const double* Bd = B;
        if (loc == HG_HOST) {
            ybuf.upload(y, size_t(n));
            yd = ybuf.get();
            if (nrhs > 0) {
                Bbuf.upload(B, size_t(n) * size_t(nrhs));
                Bd = Bbuf.get();
            }
        }
        DBuildResult br = build(*o->o, tree, k, *plan, true);
        HG_CUDA(cudaEventRecord(ev[1], c.stream));
        DFactor f = factorize(br.h, HG_LEFT);
        HG_CUDA(cudaEventRecord(ev[2], c.stream));
        *loglik = log_likelihood(f, yd);
        if (nrhs > 0) {  // the seeded right-hand sides (BASELINE.json C4)
            DVec Xd(size_t(n) * size_t(nrhs));
            panel_axpby(n, int(nrhs), 1.0, Bd, n, 0.0, Xd.get(), n);
            factor_solve(f, Xd.get(), n, int(nrhs));
            HG_CUDA(cudaMemcpyAsync(X, Xd.get(), sizeof(double) * size_t(n) * size_t(nrhs),
                                    loc == HG_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c.stream));
        }
        HG_CUDA(cudaEventRecord(ev[3], c.stream));
        std::vector<const DHodlr*> d;
        for (auto& x : br.deriv) d.push_back(&x);
        std::vector<DProductRep> reps;
        auto s = score(f, d, yd, &reps);
        for (size_t j = 0; j < s.size(); ++j) score_out[j] = s[j];
        HG_CUDA(cudaEventRecord(ev[4], c.stream));
        auto fi = fisher_from_reps(reps);
        for (size_t i = 0; i < fi.size(); ++i) fisher[i] = fi[i];
        HG_CUDA(cudaEventRecord(ev[5], c.stream));
        HG_CUDA(cudaEventSynchronize(ev[5]));
        if (times)
            for (int i = 0; i < 5; ++i) {
                float ms = 0;
                HG_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
                times[i] = ms * 1e-3;
            }
        for (auto& e : ev) cudaEventDestroy(e);
    });
}

void hg_prof_enable(int on) { prof_enable(on != 0); }

int hg_prof_read(int reset, double* ms, double* flops, double* bytes, int64_t* launches) {
    auto t = prof_read(reset != 0);
    for (size_t i = 0; i < t.size(); ++i) {
        ms[i] = t[i].ms;
        flops[i] = t[i].flops;
        bytes[i] = t[i].bytes;
        launches[i] = t[i].launches;
    }
    return int(t.size());
}

}  // extern "C"
