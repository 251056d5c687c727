#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>

#include <algorithm>

#include "common.cuh"
#include "prof.cuh"

namespace hg {

namespace {
struct Pending {
    int cat;
    double flops, bytes;
    cudaEvent_t a, b;
    std::string key;
};
bool detail() {
    static const bool on = [] {
        const char* e = std::getenv("HG_PROF_DETAIL");
        return e && std::atoi(e) != 0;
    }();
    return on;
}
bool g_on = false;
std::mutex g_mu;
std::vector<Pending> g_pending;
std::vector<ProfTotals> g_tot(PROF_NCAT);
}  // namespace

bool prof_enabled() { return g_on; }

std::string prof_tag(const char* fmt, ...) {
    char buf[160];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    return buf;
}
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
    g_pending.push_back(Pending{cat_, flops_, bytes_, a_, b, key_});
}

std::vector<ProfTotals> prof_read(bool reset) {
    std::lock_guard<std::mutex> lk(g_mu);
    std::map<std::string, ProfTotals> by_key;
    for (auto& p : g_pending) {
        cudaEventSynchronize(p.b);
        float ms = 0;
        cudaEventElapsedTime(&ms, p.a, p.b);
        auto& t = g_tot[size_t(p.cat)];
        t.ms += ms;
        t.flops += p.flops;
        t.bytes += p.bytes;
        t.launches += 1;
        if (detail() && !p.key.empty()) {
            auto& d = by_key[p.key];
            d.ms += ms;
            d.flops += p.flops;
            d.bytes += p.bytes;
            d.launches += 1;
        }
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    g_pending.clear();
    if (!by_key.empty()) {
        std::vector<std::pair<std::string, ProfTotals>> v(by_key.begin(), by_key.end());
        std::sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.second.ms > b.second.ms; });
        for (const auto& [k, t] : v)
            std::fprintf(stderr, "[hg prof] %-48s %9.3f ms %5lld calls %7.2f TF/s %8.1f GB/s\n", k.c_str(), t.ms,
                         t.launches, t.flops / (t.ms * 1e9), t.bytes / (t.ms * 1e6));
    }
    auto out = g_tot;
    if (reset) g_tot.assign(PROF_NCAT, ProfTotals{});
    return out;
}

}  // namespace hg
