// Matrix-free peeling construction of the HODLR approximation and of its
// parameter-derivative matrices (randomized range sketching).
//
// Reference: sketch.hpp:17-85, sketch.cpp:10-356. The SketchPlan Gaussian
// samplers are drawn on the host with std::mt19937_64 +
// std::normal_distribution<double> in the reference's fill order and uploaded
// once, so CPU and GPU consume identical sketch matrices.
#pragma once

#include "oracle.cuh"
#include "qr.cuh"
#include "hodlr.cuh"

namespace hg {

struct DSketchPlan {
    DTreeP tree;
    i64 k = 0;
    std::uint64_t seed = 0;
    std::vector<DVecP> level;  // [l-1]: n x k (Gaussian on right-child rows, zero elsewhere)
    DVecP leaf;                // n x bmax: stacked identities
};
using DSketchPlanP = std::shared_ptr<const DSketchPlan>;

/// sketch.cpp:10-31 (cached per tree, k, seed).
DSketchPlanP get_plan(DTreeP tree, i64 k, std::uint64_t seed);

/// randomized_range (sketch.cpp:37-76) of one rows x k block on the device:
/// pivoted QR, Q = first k Householder columns, diag(R) >= 0 by sign flip,
/// numeric rank = #|r_ii| > 64 eps |r_00|, deficient columns completed with
/// e_0, e_1, ... orthogonalised twice. R, perm, nr are device pointers.
void randomized_range(const double* Y, i64 ldy, int rows, int k, double* Q, i64 ldq, double* R, int* perm, int* nr);

/// diff_qr (sketch.cpp:78-111) of b = q r under perturbation dB (device).
void diff_qr(const double* dB, i64 lddb, const double* Q, i64 ldq, const double* R, int rows, int k, double* dQ,
             i64 lddq, double* dQspan, i64 ldds, double* dR, int* ill);

struct DBuildResult {
    DHodlr h;
    std::vector<DHodlr> deriv;
    int warnings = 0;
    int p = 0;
    std::vector<std::int64_t> decisions;  // per (level, node): numeric_rank, w2, rw[0..p)
};

/// sketch.cpp:128-343
DBuildResult build(const DOracle& o, DTreeP tree, i64 k, const DSketchPlan& plan, bool with_deriv);

}  // namespace hg
