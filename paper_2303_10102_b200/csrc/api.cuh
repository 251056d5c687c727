// Aggregate header of the device hot path (used by the C ABI).
#pragma once

#include "hodlr.cuh"

namespace hg {

DHodlr hodlr_deep_copy(const DHodlr& h);

// Filled in by factor.cu / prodrep.cu / oracle.cu / build.cu.
struct DFactor {};
struct DProductRep {};
struct DOracle {
    virtual ~DOracle() = default;
};
struct DBuildResult {};

}  // namespace hg
