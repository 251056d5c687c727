// Stream-ordered caching device allocator (see common.cuh).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <set>
#include <unordered_map>

#include "common.cuh"

namespace hg {

namespace {

struct Block {
    size_t bytes;
    cudaStream_t stream;
};

struct Cache {
    std::mutex mu;
    // free blocks per stream, by size
    std::map<cudaStream_t, std::multimap<size_t, void*>> free;
    std::unordered_map<void*, Block> live;  // handed out
    std::set<cudaStream_t> retired;         // streams of destroyed contexts
    size_t cached = 0, in_use = 0;
};

/// Cached bytes are capped at 60% of device memory.
size_t cache_limit() {
    static const size_t lim = [] {
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) tot = size_t(80) << 30;
        return tot / 10 * 6;
    }();
    return lim;
}

Cache& cache() {
    static Cache* c = new Cache;  // never destroyed: frees may run at exit
    return *c;
}

bool trace() {
    static const bool on = [] {
        const char* e = std::getenv("HG_TRACE_ALLOC");
        return e && std::atoi(e) != 0;
    }();
    return on;
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

size_t round_up(size_t b) {
    const size_t g = b >= (size_t(1) << 20) ? (size_t(2) << 20) : 512;
    return (b + g - 1) / g * g;
}

void flush_locked(Cache& c) {
    for (auto& [s, m] : c.free)
        for (auto& [sz, p] : m) {
            cudaFreeAsync(p, s);
            c.cached -= sz;
        }
    c.free.clear();
}

}  // namespace

void* dev_alloc(size_t bytes) {
    Cache& c = cache();
    const cudaStream_t s = current().stream;
    const size_t want = round_up(bytes);
    const double t0 = trace() ? now_ms() : 0.0;
    std::lock_guard<std::mutex> lk(c.mu);
    auto fs = c.free.find(s);
    if (fs != c.free.end()) {
        auto it = fs->second.lower_bound(want);
        if (it != fs->second.end() && it->first <= want + want / 8) {
            void* p = it->second;
            const size_t sz = it->first;
            fs->second.erase(it);
            c.cached -= sz;
            c.in_use += sz;
            c.live[p] = Block{sz, s};
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, want, s);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        flush_locked(c);
        cudaStreamSynchronize(s);
        e = cudaMallocAsync(&p, want, s);
    }
    HG_CUDA(e);
    c.in_use += want;
    c.live[p] = Block{want, s};
    if (trace()) {
        const double ms = now_ms() - t0;
        if (ms > 1.0)
            std::fprintf(stderr, "[hg alloc] miss %.1f MB took %.2f ms (in use %.1f GB, cached %.1f GB)\n",
                         double(want) / 1e6, ms, double(c.in_use) / 1e9, double(c.cached) / 1e9);
    }
    return p;
}

void dev_free(void* p) {
    if (!p) return;
    Cache& c = cache();
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.live.find(p);
    if (it == c.live.end()) return;  // not ours (never happens)
    const Block b = it->second;
    c.live.erase(it);
    c.in_use -= b.bytes;
    if (c.retired.count(b.stream)) {  // its stream is gone: plain free
        cudaFree(p);
        return;
    }
    if (c.cached + b.bytes > cache_limit()) {
        cudaFreeAsync(p, b.stream);
        return;
    }
    c.cached += b.bytes;
    c.free[b.stream].emplace(b.bytes, p);
}

void dev_stream_retire(cudaStream_t s) {
    Cache& c = cache();
    std::lock_guard<std::mutex> lk(c.mu);
    auto fs = c.free.find(s);
    if (fs != c.free.end()) {
        for (auto& [sz, p] : fs->second) {
            cudaFreeAsync(p, s);
            c.cached -= sz;
        }
        c.free.erase(fs);
    }
    c.retired.insert(s);
}

void dev_stream_adopt(cudaStream_t s) {
    Cache& c = cache();
    std::lock_guard<std::mutex> lk(c.mu);
    c.retired.erase(s);
}

void dev_cache_flush() {
    Cache& c = cache();
    std::lock_guard<std::mutex> lk(c.mu);
    flush_locked(c);
}

void dev_cache_stats(size_t* cached, size_t* in_use) {
    Cache& c = cache();
    std::lock_guard<std::mutex> lk(c.mu);
    if (cached) *cached = c.cached;
    if (in_use) *in_use = c.in_use;
}

}  // namespace hg
