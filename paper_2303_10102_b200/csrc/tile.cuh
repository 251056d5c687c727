// Shared FP64 register-tile micro-kernel (64x64 CTA tile, 4x4 per thread,
// K staged 16 at a time through padded shared memory).
#pragma once

namespace hg {
namespace tile {

constexpr int TM = 64, TN = 64, KS = 16, NT = 256;

__device__ __forceinline__ void mma16(const double (&As)[KS][TM + 1], const double (&Bs)[KS][TN + 1],
                                      double (&acc)[4][4], int tm, int tn) {
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk][tm + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tn + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
}

}  // namespace tile
}  // namespace hg
