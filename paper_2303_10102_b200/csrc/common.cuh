// Common device-side infrastructure for the B200 HODLR hot path.
//
// One context = one device + one CUDA stream. All device memory comes from the
// stream-ordered pool (cudaMallocAsync) so per-call temporaries are cheap;
// every kernel of a context runs on its stream.
#pragma once

#include <cuda_runtime.h>

#include "../../include/hodlrgp_b200.h"  // HG_OPT_* / HG_ASSOC_* / HG_COMPRESS_* values

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace hg {

using i64 = long long;

// ---------------------------------------------------------------- errors
/// factorization.hpp:14-16 — non-positive capacitance / leaf determinant.
struct NotPositiveDefinite : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define HG_CUDA(x)                                                                              \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) (void)cudaGetLastError(); /* do not leave it for a later check */ \
        if (e_ != cudaSuccess)                                                                  \
            throw ::hg::CudaError(std::string(#x) + " failed: " + cudaGetErrorString(e_) +     \
                                  " at " __FILE__ ":" + std::to_string(__LINE__));              \
    } while (0)
#define HG_LAUNCH() HG_CUDA(cudaGetLastError())

inline void require(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}

// --------------------------------------------------------------- context
struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    std::uint64_t launches = 0;  // kernels launched through this context
    int product_assoc = 0;       // HG_OPT_PRODUCT_ASSOCIATION (HG_ASSOC_*)
    int compression = 0;         // HG_OPT_COMPRESSION (HG_COMPRESS_*)
    int q2_basis = 0;            // HG_OPT_Q2_BASIS (HG_Q2_*)
    int compress_at = 0;         // HG_OPT_COMPRESS_AT (HG_COMPRESS_AT_*)
    int sketch_rng = 0;          // HG_OPT_SKETCH_RNG (HG_SKETCH_RNG_*)
};


Ctx& current();           // thread's active context (set by the C ABI)
void set_current(Ctx* c);

inline void count_launch() { ++current().launches; }

/// Per-device one-time flag: function attributes (dynamic shared memory
/// opt-in) are per device, and hg_ctx_create allows contexts on several
/// devices in one process. `static DeviceOnce o; if (o.first()) ...`.
struct DeviceOnce {
    bool seen[64] = {};
    bool first() {
        const int d = current().device & 63;
        if (seen[d]) return false;
        seen[d] = true;
        return true;
    }
};

// ------------------------------------------------------- device allocator
/// Stream-ordered caching allocator. A step of the MLE pipeline allocates
/// the same multiset of multi-GB panels every iteration; the driver pool
/// (cudaMallocAsync) re-maps physical pages to satisfy them from fragmented
/// free space, which costs up to ~1 s of host time per call at n = 2^20.
/// Freed blocks are therefore kept per stream and handed back, best fit
/// within 1/8 of the request, to later allocations on the SAME stream (stream
/// order makes the reuse safe without events). Misses fall through to
/// cudaMallocAsync; on out-of-memory every cached block is returned to the
/// pool and the allocation retried once. HG_TRACE_ALLOC=1 reports calls
/// slower than 1 ms.
void* dev_alloc(size_t bytes);
void dev_free(void* p);
/// Return every cached block to the driver pool (all streams).
void dev_cache_flush();
/// Bytes currently cached (free, held for reuse) and handed out.
void dev_cache_stats(size_t* cached, size_t* in_use);
/// A context's stream is about to be destroyed / has been created.
void dev_stream_retire(cudaStream_t s);
void dev_stream_adopt(cudaStream_t s);

// ---------------------------------------------------------- device buffer
/// Stream-ordered device allocation (RAII, deep-copyable).
template <class T>
class DBuf {
public:
    DBuf() = default;
    explicit DBuf(size_t n) { alloc(n); }
    ~DBuf() { release(); }
    DBuf(const DBuf& o) { copy_from(o); }
    DBuf& operator=(const DBuf& o) {
        if (this != &o) {
            release();
            copy_from(o);
        }
        return *this;
    }
    DBuf(DBuf&& o) noexcept : p_(o.p_), n_(o.n_), own_(o.own_) {
        o.p_ = nullptr;
        o.n_ = 0;
    }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = o.p_;
            n_ = o.n_;
            own_ = o.own_;
            o.p_ = nullptr;
            o.n_ = 0;
        }
        return *this;
    }
    /// Non-owning view of n elements at p (see make_view).
    static DBuf view(T* p, size_t n) {
        DBuf b;
        b.p_ = p;
        b.n_ = n;
        b.own_ = false;
        return b;
    }
    void alloc(size_t n) {
        release();
        n_ = n;
        own_ = true;
        if (n) p_ = static_cast<T*>(dev_alloc(n * sizeof(T)));
    }
    void zero() {
        if (n_) HG_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), current().stream));
    }
    void upload(const T* h, size_t n) {
        if (n != n_) alloc(n);
        if (n) HG_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, current().stream));
    }
    void upload(const std::vector<T>& v) { upload(v.data(), v.size()); }
    std::vector<T> download() const {
        std::vector<T> v(n_);
        if (n_) {
            HG_CUDA(cudaMemcpyAsync(v.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost, current().stream));
            HG_CUDA(cudaStreamSynchronize(current().stream));
        }
        return v;
    }
    T* get() const { return p_; }
    size_t size() const { return n_; }
    bool empty() const { return n_ == 0; }
    void release() {
        if (p_ && own_) dev_free(p_);
        p_ = nullptr;
        n_ = 0;
        own_ = true;
    }

private:
    void copy_from(const DBuf& o) {
        p_ = nullptr;
        n_ = 0;
        own_ = true;
        if (o.n_) {
            alloc(o.n_);
            HG_CUDA(cudaMemcpyAsync(p_, o.p_, n_ * sizeof(T), cudaMemcpyDeviceToDevice, current().stream));
        }
    }
    T* p_ = nullptr;
    size_t n_ = 0;
    bool own_ = true;
};

using DVec = DBuf<double>;
using DVecP = std::shared_ptr<DVec>;

/// Shared non-owning view of n doubles at p inside `owner` (kept alive by the view).
inline DVecP make_view(const DVecP& owner, double* p, size_t n) {
    return DVecP(new DVec(DVec::view(p, n)), [owner](DVec* d) { delete d; });
}

inline DVecP make_dvec(size_t n, bool zero = true) {
    auto p = std::make_shared<DVec>(n);
    if (zero) p->zero();
    return p;
}

inline void sync() { HG_CUDA(cudaStreamSynchronize(current().stream)); }

inline int cdiv(i64 a, i64 b) { return int((a + b - 1) / b); }

}  // namespace hg
