// Shared FP64 tensor-core micro-kernel: 64x64 CTA tile, 8 warps (2 x 4),
// each warp a 32x16 sub-tile of 4x2 DMMA m8n8k4 tiles (mma.sync .f64 — the
// FP64 tensor path on sm_100a; tcgen05 has no f64 kind). K is staged 16 deep
// through shared memory laid out k-major (As[k][m], Bs[k][n]) with a row
// stride of 68 doubles so a half-warp's fragment loads hit 16 distinct banks.
#pragma once

namespace hg {
namespace tile {

constexpr int TM = 64, TN = 64, KS = 16, NT = 256;
constexpr int LDS = TM + 4;  // shared row stride (doubles)

struct Acc {
    double v[4][2][2];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) v[i][j][0] = v[i][j][1] = 0.0;
    }
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

/// acc += As[0:KS][warp rows]^T-view * Bs[0:KS][warp cols] (k-major tiles).
__device__ __forceinline__ void mma_tile(const double (&As)[KS][LDS], const double (&Bs)[KS][LDS], Acc& acc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int k4 = 0; k4 < KS; k4 += 4) {
        double a[4], b[2];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[k4 + t][wm + i * 8 + g];
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j] = Bs[k4 + t][wn + j * 8 + g];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) dmma(acc.v[i][j], a[i], b[j]);
    }
}

/// Visit every accumulator element owned by this thread: f(m, n, value).
template <class F>
__device__ __forceinline__ void for_each(const Acc& acc, F&& f) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) f(wm + i * 8 + g, wn + j * 8 + 2 * t + e, acc.v[i][j][e]);
}

}  // namespace tile
}  // namespace hg
