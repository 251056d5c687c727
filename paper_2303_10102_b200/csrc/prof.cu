#include <mutex>

#include "common.cuh"
#include "prof.cuh"

namespace hg {

namespace {
struct Pending {
    int cat;
    double flops, bytes;
    cudaEvent_t a, b;
};
bool g_on = false;
std::mutex g_mu;
std::vector<Pending> g_pending;
std::vector<ProfTotals> g_tot(PROF_NCAT);
}  // namespace

bool prof_enabled() { return g_on; }
void prof_enable(bool on) { g_on = on; }

ProfScope::ProfScope(int cat, double flops, double bytes) : cat_(cat), flops_(flops), bytes_(bytes) {
    if (!g_on) return;
    cudaEventCreate(&a_);
    cudaEventRecord(a_, current().stream);
}

ProfScope::~ProfScope() {
    if (!a_) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, current().stream);
    std::lock_guard<std::mutex> lk(g_mu);
    g_pending.push_back(Pending{cat_, flops_, bytes_, a_, b});
}

std::vector<ProfTotals> prof_read(bool reset) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& p : g_pending) {
        cudaEventSynchronize(p.b);
        float ms = 0;
        cudaEventElapsedTime(&ms, p.a, p.b);
        auto& t = g_tot[size_t(p.cat)];
        t.ms += ms;
        t.flops += p.flops;
        t.bytes += p.bytes;
        t.launches += 1;
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    g_pending.clear();
    auto out = g_tot;
    if (reset) g_tot.assign(PROF_NCAT, ProfTotals{});
    return out;
}

}  // namespace hg
