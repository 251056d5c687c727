// Aggregate header of the device hot path (used by the C ABI).
#pragma once

#include "prodrep.cuh"

namespace hg {

DHodlr hodlr_deep_copy(const DHodlr& h);

// Filled in by oracle.cu / build.cu.
struct DOracle {
    virtual ~DOracle() = default;
};
struct DBuildResult {};

}  // namespace hg
