// Optional per-kernel device timing (CUDA events around each launch) and an
// algorithmic flop/byte ledger per kernel class — the live roofline numbers
// bench.py reports. Disabled by default (no events are recorded).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

namespace hg {

enum ProfCat {
    PROF_SEG_TN = 0,
    PROF_SEG_NN,
    PROF_LEAF_MM,
    PROF_LEAF_SOLVE,
    PROF_LEAF_FACTOR,
    PROF_CAP_LU,
    PROF_CAP_SOLVE,
    PROF_QR,
    PROF_FORM_Q,
    PROF_ORACLE,
    PROF_REDUCE,
    PROF_OTHER,
    PROF_MATVEC,
    PROF_NCAT
};

struct ProfTotals {
    double ms = 0, flops = 0, bytes = 0;
    long long launches = 0;
};

bool prof_enabled();
void prof_enable(bool on);
/// Synchronizes, folds pending event pairs into totals, returns them.
std::vector<ProfTotals> prof_read(bool reset);

/// printf-style shape tag.
std::string prof_tag(const char* fmt, ...);

/// Records an event pair around the kernel(s) launched in its scope.
class ProfScope {
public:
    ProfScope(int cat, double flops, double bytes);
    ~ProfScope();
    /// Shape tag for HG_PROF_DETAIL=1 (per-shape breakdown printed by prof_read).
    void key(const std::string& k) {
        if (a_) key_ = k;
    }

private:
    int cat_;
    std::string key_;
    double flops_, bytes_;
    cudaEvent_t a_ = nullptr;
};

}  // namespace hg
