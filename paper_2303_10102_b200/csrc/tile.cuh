// FP64 tensor-core tile engine shared by every GEMM-shaped kernel.
//
// CTA tile 64x64, 4 warps in a 2x2 grid, each warp 32x32 = 4x4 DMMA m8n8k4
// tiles (mma.sync .f64 — the FP64 tensor path on sm_100a; tcgen05 has no f64
// kind). K advances 16 at a time through a 3-stage cp.async pipeline.
//
// Shared layouts follow each operand's global contiguity so that both the
// cp.async copies and the fragment loads are bank-conflict free:
//   KC ("k-contiguous", e.g. a column-major panel whose rows are the
//       reduction index): smem [m][k], row stride 20 doubles;
//   MC ("m-contiguous", e.g. a column-major panel whose rows are the output
//       rows): smem [k][m], row stride 68 doubles.
// Both strides are 4 mod 16 doubles: a half-warp's fragment (g = 0..3,
// t = 0..3) maps to 16 distinct 8-byte bank pairs.
#pragma once

#include <cstdint>

namespace hg {
namespace tile {

constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3, THREADS = 128;
constexpr int LD_KC = BK + 4;  // 20
constexpr int LD_MC = BM + 4;  // 68
constexpr int TILE_ELEMS = (BM * LD_KC > BK * LD_MC) ? BM * LD_KC : BK * LD_MC;  // one operand stage

struct Acc {
    double v[4][4][2];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) v[i][j][0] = v[i][j][1] = 0.0;
    }
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int bytes = valid ? 8 : 0;  // 0 => zero-fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

/// Fragment element (m, k) of an operand stage in its layout.
template <bool KC>
__device__ __forceinline__ double frag(const double* S, int m, int k) {
    return KC ? S[m * LD_KC + k] : S[k * LD_MC + m];
}

/// One BK slice: acc += A(:, k) B(:, k)^T over the warp's 32x32 sub-tile.
template <bool AKC, bool BKC>
__device__ __forceinline__ void mma_stage(const double* As, const double* Bs, Acc& acc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = frag<AKC>(As, wm + i * 8 + g, k4 + t);
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = frag<BKC>(Bs, wn + j * 8 + g, k4 + t);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma(acc.v[i][j], a[i], b[j]);
    }
}

/// Pipelined main loop. Loader objects provide
///   static constexpr bool KC;
///   __device__ void issue(double* stage, int kt);   // cp.async one BK slice
template <int NS = STAGES, class LA, class LB>
__device__ __forceinline__ void run(LA& la, LB& lb, int ktiles, double* smem, Acc& acc) {
    double* As = smem;
    double* Bs = smem + NS * TILE_ELEMS;
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) {
        if (s < ktiles) {
            la.issue(As + s * TILE_ELEMS, s);
            lb.issue(Bs + s * TILE_ELEMS, s);
        }
        cp_commit();
    }
    for (int kt = 0; kt < ktiles; ++kt) {
        cp_wait<NS - 2>();
        __syncthreads();  // tile kt landed; every warp is done with tile kt-1's buffer
        const int nk = kt + NS - 1;
        if (nk < ktiles) {
            la.issue(As + (nk % NS) * TILE_ELEMS, nk);
            lb.issue(Bs + (nk % NS) * TILE_ELEMS, nk);
        }
        cp_commit();
        const int st = kt % NS;
        mma_stage<LA::KC, LB::KC>(As + st * TILE_ELEMS, Bs + st * TILE_ELEMS, acc);
    }
    cp_wait<0>();
}

constexpr int smem_bytes(int ns) { return 2 * ns * TILE_ELEMS * int(sizeof(double)); }
constexpr int SMEM_BYTES = smem_bytes(STAGES);

/// Column-major operand whose rows are the reduction index k (k-contiguous):
/// element (k, m) at base[k + m * ld], valid for k < kmax, m < mmax.
struct LoadKC {
    static constexpr bool KC = true;
    const double* base;
    long long ld;
    int kmax, mmax;
    __device__ __forceinline__ void issue(double* S, int kt) const {
        const int k = threadIdx.x & 15;
        const int kk = kt * BK + k;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int m = (threadIdx.x >> 4) + 8 * q;
            const bool v = kk < kmax && m < mmax;
            cp_async8(S + m * LD_KC + k, v ? base + kk + m * ld : base, v);
        }
    }
};

/// Column-major operand whose rows are the output index m (m-contiguous):
/// element (m, k) at base[m + k * ld], valid for m < mmax, k < kmax.
struct LoadMC {
    static constexpr bool KC = false;
    const double* base;
    long long ld;
    int mmax, kmax;
    __device__ __forceinline__ void issue(double* S, int kt) const {
        const int m = threadIdx.x & 63;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int k = (threadIdx.x >> 6) + 2 * q;
            const int kk = kt * BK + k;
            const bool v = m < mmax && kk < kmax;
            cp_async8(S + k * LD_MC + m, v ? base + m + kk * ld : base, v);
        }
    }
};

/// Visit every accumulator element owned by this thread: f(m, n, value).
template <class F>
__device__ __forceinline__ void for_each(const Acc& acc, F&& f) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) f(wm + i * 8 + g, wn + j * 8 + 2 * t + e, acc.v[i][j][e]);
}

}  // namespace tile
}  // namespace hg
