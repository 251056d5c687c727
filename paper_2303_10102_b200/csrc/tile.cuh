// FP64 tensor-core tile engine shared by every GEMM-shaped kernel.
//
// CTA tile TBM x TBN (multiples of 16, 16..96), 4 warps in a 2x2 grid, each
// warp (TBM/2) x (TBN/2) = (TBM/16) x (TBN/16) DMMA m8n8k4 tiles (mma.sync
// .f64 — the FP64 tensor path on sm_100a; tcgen05 has no f64 kind). K
// advances 16 at a time through a multi-stage cp.async pipeline. The tile
// shape is picked per call from the problem's M and N (tile_for): HODLR
// ranks and panel widths are 40, 80, 3.. so a fixed 64x64 tile wastes up to
// 60% of the tensor-core work in padding.
//
// Shared layouts follow each operand's global contiguity so that both the
// cp.async copies and the fragment loads are bank-conflict free:
//   KC ("k-contiguous", e.g. a column-major panel whose rows are the
//       reduction index): smem [m][k], row stride 20 doubles;
//   MC ("m-contiguous", e.g. a column-major panel whose rows are the output
//       rows): smem [k][m], row stride ROWS + 4 doubles.
// Both strides are 4 mod 16 doubles: a half-warp's fragment (g = 0..3,
// t = 0..3) maps to 16 distinct 8-byte bank pairs.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <type_traits>

#include "common.cuh"

namespace hg {
namespace tile {

constexpr int BM = 64, BN = 64, BK = 16, STAGES = 3, THREADS = 128;
constexpr int LD_KC = BK + 4;  // 20
constexpr int LD_MC = BM + 4;  // 68 (64-row tiles)

/// Shared elements of one operand stage with ROWS tile rows (either layout).
constexpr int stage_elems(int rows) { return (rows * LD_KC > BK * (rows + 4)) ? rows * LD_KC : BK * (rows + 4); }
constexpr int TILE_ELEMS = stage_elems(64);

/// Accumulators of one warp: (TBM/16) x (TBN/16) DMMA tiles.
template <int WM, int WN>
struct AccT {
    double v[WM][WN][2];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < WM; ++i)
#pragma unroll
            for (int j = 0; j < WN; ++j) v[i][j][0] = v[i][j][1] = 0.0;
    }
};
using Acc = AccT<4, 4>;

/// Warp grid of a TBM x TBN tile (4 warps): WGM x WGN with WGM * WGN = 4,
/// each warp (TBM / WGM) x (TBN / WGN) = WM x WN DMMA tiles. 2 x 2 when both
/// extents are multiples of 16; 4 x 1 for N = 40 (M a multiple of 32); 1 x 4
/// for M = 40 (N a multiple of 32).
constexpr bool shape_ok(int m, int n) {
    const int wgn = (m % 16 == 0 && n % 16 == 0) ? 2 : (m % 32 == 0 ? 1 : 4);
    const int wgm = 4 / wgn;
    return m % (8 * wgm) == 0 && n % (8 * wgn) == 0;
}

template <int TBM, int TBN>
struct Shape {
    static constexpr int WGN = (TBM % 16 == 0 && TBN % 16 == 0) ? 2 : (TBM % 32 == 0 ? 1 : 4);
    static constexpr int WGM = 4 / WGN;
    static constexpr int WM = TBM / (8 * WGM), WN = TBN / (8 * WGN);
    static_assert(WM * 8 * WGM == TBM && WN * 8 * WGN == TBN, "tile extents do not fit the warp grid");
    using Acc = AccT<WM, WN>;
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
/// 16-byte copy that bypasses L1 (streamed operands); `bytes` in {0, 8, 16}
/// valid source bytes, the rest of the 16 zero-filled. Both addresses must be
/// 16-byte aligned.
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
/// An operand whose column starts are all 16-byte aligned (pairs of
/// consecutive elements of a column can move as one 16-byte copy).
__device__ __forceinline__ bool pairs_aligned(const double* base, long long ld) {
    return (reinterpret_cast<uintptr_t>(base) & 15) == 0 && (ld & 1) == 0;
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

/// Fragment element (m, k) of an operand stage with ROWS rows in its layout.
template <bool KC, int ROWS>
__device__ __forceinline__ double frag(const double* S, int m, int k) {
    return KC ? S[m * LD_KC + k] : S[k * (ROWS + 4) + m];
}

/// One BK slice: acc += A(:, k) B(:, k)^T over the warp's sub-tile.
template <bool AKC, bool BKC, int TBM, int TBN>
__device__ __forceinline__ void mma_stage(const double* As, const double* Bs, typename Shape<TBM, TBN>::Acc& acc) {
    using S = Shape<TBM, TBN>;
    constexpr int WM = S::WM, WN = S::WN;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp / S::WGN) * (TBM / S::WGM), wn = (warp % S::WGN) * (TBN / S::WGN);
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
        double a[WM], b[WN];
#pragma unroll
        for (int i = 0; i < WM; ++i) a[i] = frag<AKC, TBM>(As, wm + i * 8 + g, k4 + t);
#pragma unroll
        for (int j = 0; j < WN; ++j) b[j] = frag<BKC, TBN>(Bs, wn + j * 8 + g, k4 + t);
#pragma unroll
        for (int i = 0; i < WM; ++i)
#pragma unroll
            for (int j = 0; j < WN; ++j) dmma(acc.v[i][j], a[i], b[j]);
    }
}

/// Pipelined main loop over a TBM x TBN tile. Loader objects provide
///   static constexpr bool KC;  static constexpr int ROWS;
///   __device__ void issue(double* stage, int kt);   // cp.async one BK slice
template <int NS, int TBM, int TBN, class LA, class LB>
__device__ __forceinline__ void run_t(LA& la, LB& lb, int ktiles, double* smem, typename Shape<TBM, TBN>::Acc& acc) {
    static_assert(LA::ROWS == TBM && LB::ROWS == TBN, "loader extents must match the tile");
    constexpr int AE = stage_elems(TBM), BE = stage_elems(TBN);
    double* As = smem;
    double* Bs = smem + NS * AE;
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) {
        if (s < ktiles) {
            la.issue(As + s * AE, s);
            lb.issue(Bs + s * BE, s);
        }
        cp_commit();
    }
    for (int kt = 0; kt < ktiles; ++kt) {
        cp_wait<NS - 2>();
        __syncthreads();  // tile kt landed; every warp is done with tile kt-1's buffer
        const int nk = kt + NS - 1;
        if (nk < ktiles) {
            la.issue(As + (nk % NS) * AE, nk);
            lb.issue(Bs + (nk % NS) * BE, nk);
        }
        cp_commit();
        const int st = kt % NS;
        mma_stage<LA::KC, LB::KC, TBM, TBN>(As + st * AE, Bs + st * BE, acc);
    }
    cp_wait<0>();
}

/// run_t with a hook called after the MMA of every K tile (flushes of
/// segmented accumulators).
template <int NS, int TBM, int TBN, class LA, class LB, class H>
__device__ __forceinline__ void run_t_hook(LA& la, LB& lb, int ktiles, double* smem,
                                           typename Shape<TBM, TBN>::Acc& acc, H&& hook) {
    static_assert(LA::ROWS == TBM && LB::ROWS == TBN, "loader extents must match the tile");
    constexpr int AE = stage_elems(TBM), BE = stage_elems(TBN);
    double* As = smem;
    double* Bs = smem + NS * AE;
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) {
        if (s < ktiles) {
            la.issue(As + s * AE, s);
            lb.issue(Bs + s * BE, s);
        }
        cp_commit();
    }
    for (int kt = 0; kt < ktiles; ++kt) {
        cp_wait<NS - 2>();
        __syncthreads();
        const int nk = kt + NS - 1;
        if (nk < ktiles) {
            la.issue(As + (nk % NS) * AE, nk);
            lb.issue(Bs + (nk % NS) * BE, nk);
        }
        cp_commit();
        const int st = kt % NS;
        mma_stage<LA::KC, LB::KC, TBM, TBN>(As + st * AE, Bs + st * BE, acc);
        hook(kt);
    }
    cp_wait<0>();
}

/// 64x64 shorthand (kernels written before the shape-adaptive engine).
template <int NS = STAGES, class LA, class LB>
__device__ __forceinline__ void run(LA& la, LB& lb, int ktiles, double* smem, Acc& acc) {
    run_t<NS, 64, 64>(la, lb, ktiles, smem, acc);
}

constexpr int smem_bytes_t(int ns, int tbm, int tbn) {
    return ns * (stage_elems(tbm) + stage_elems(tbn)) * int(sizeof(double));
}
constexpr int smem_bytes(int ns) { return smem_bytes_t(ns, 64, 64); }
constexpr int SMEM_BYTES = smem_bytes(STAGES);

/// Column-major operand whose rows are the reduction index k (k-contiguous):
/// element (k, m) at base[k + m * ld], valid for k < kmax, m < mmax.
template <int R, bool VEC = true>
struct LoadKCT {
    static constexpr bool KC = true;
    static constexpr int ROWS = R;
    const double* base;
    long long ld;
    int kmax, mmax;
    __device__ __forceinline__ void issue(double* S, int kt) const {
        if (VEC && pairs_aligned(base, ld)) {  // k pairs as 16-byte copies (half the copy instructions)
#pragma unroll
            for (int q = 0; q < (R * BK / 2 + THREADS - 1) / THREADS; ++q) {
                const int e = threadIdx.x + THREADS * q;
                if (R * BK / 2 % THREADS != 0 && e >= R * BK / 2) break;
                const int k2 = (e & (BK / 2 - 1)) * 2, m = e / (BK / 2);
                const int kk = kt * BK + k2;
                const int bytes = m < mmax ? (kk + 1 < kmax ? 16 : (kk < kmax ? 8 : 0)) : 0;
                cp_async16(S + m * LD_KC + k2, bytes ? base + kk + m * ld : base, bytes);
            }
            return;
        }
        const int k = threadIdx.x & 15;
        const int kk = kt * BK + k;
#pragma unroll
        for (int q = 0; q < R / 8; ++q) {
            const int m = (threadIdx.x >> 4) + 8 * q;
            const bool v = kk < kmax && m < mmax;
            cp_async8(S + m * LD_KC + k, v ? base + kk + m * ld : base, v);
        }
    }
};
using LoadKC = LoadKCT<64>;

/// Column-major operand whose rows are the output index m (m-contiguous):
/// element (m, k) at base[m + k * ld], valid for m < mmax, k < kmax.
template <int R, bool VEC = true>
struct LoadMCT {
    static constexpr bool KC = false;
    static constexpr int ROWS = R;
    const double* base;
    long long ld;
    int mmax, kmax;
    __device__ __forceinline__ void issue(double* S, int kt) const {
        if (VEC && pairs_aligned(base, ld)) {  // m pairs as 16-byte copies
#pragma unroll
            for (int q = 0; q < (R * BK / 2 + THREADS - 1) / THREADS; ++q) {
                const int e = threadIdx.x + THREADS * q;
                if (R * BK / 2 % THREADS != 0 && e >= R * BK / 2) break;
                const int m2 = (e % (R / 2)) * 2, k = e / (R / 2);
                const int kk = kt * BK + k;
                const int bytes = kk < kmax ? (m2 + 1 < mmax ? 16 : (m2 < mmax ? 8 : 0)) : 0;
                cp_async16(S + k * (R + 4) + m2, bytes ? base + m2 + kk * ld : base, bytes);
            }
            return;
        }
#pragma unroll
        for (int q = 0; q < R / 8; ++q) {
            const int e = threadIdx.x + THREADS * q;
            const int m = e % R, k = e / R;
            const int kk = kt * BK + k;
            const bool v = m < mmax && kk < kmax;
            cp_async8(S + k * (R + 4) + m, v ? base + m + kk * ld : base, v);
        }
    }
};
using LoadMC = LoadMCT<64>;

/// Visit every accumulator element owned by this thread: f(m, n, value).
template <int TBM, int TBN, class F>
__device__ __forceinline__ void for_each_t(const typename Shape<TBM, TBN>::Acc& acc, F&& f) {
    using S = Shape<TBM, TBN>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp / S::WGN) * (TBM / S::WGM), wn = (warp % S::WGN) * (TBN / S::WGN);
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int i = 0; i < S::WM; ++i)
#pragma unroll
        for (int j = 0; j < S::WN; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) f(wm + i * 8 + g, wn + j * 8 + 2 * t + e, acc.v[i][j][e]);
}
template <class F>
__device__ __forceinline__ void for_each(const Acc& acc, F&& f) {
    for_each_t<64, 64>(acc, f);
}

/// Same traversal as for_each_t, exposing the accumulator slot:
/// f(double& slot, m, n) for every element owned by this thread.
template <int TBM, int TBN, class F>
__device__ __forceinline__ void for_each_slot(typename Shape<TBM, TBN>::Acc& a, F&& f) {
    using S = Shape<TBM, TBN>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp / S::WGN) * (TBM / S::WGM), wn = (warp % S::WGN) * (TBN / S::WGN);
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int i = 0; i < S::WM; ++i)
#pragma unroll
        for (int j = 0; j < S::WN; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) f(a.v[i][j][e], wm + i * 8 + g, wn + j * 8 + 2 * t + e);
}

/// Paired traversal of two accumulator sets: f(a_slot, b_slot, m, n).
template <int TBM, int TBN, class F>
__device__ __forceinline__ void for_each_slot2(const typename Shape<TBM, TBN>::Acc& a,
                                               const typename Shape<TBM, TBN>::Acc& b, F&& f) {
    using S = Shape<TBM, TBN>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = (warp / S::WGN) * (TBM / S::WGM), wn = (warp % S::WGN) * (TBN / S::WGN);
    const int g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int i = 0; i < S::WM; ++i)
#pragma unroll
        for (int j = 0; j < S::WN; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) f(a.v[i][j][e], b.v[i][j][e], wm + i * 8 + g, wn + j * 8 + 2 * t + e);
}

/// Tile extent (16..96, multiple of 16) for a problem extent x: the smallest
/// single tile that covers x up to 96; beyond, 64 or 80, whichever pads less
/// (96-wide tiles over many column blocks cost occupancy: 48 accumulators).
inline int tile_for(int x) {
    if (x <= 96) return (x + 15) / 16 * 16 < 16 ? 16 : (x + 15) / 16 * 16;
    const int w64 = (x + 63) / 64 * 64 - x, w80 = (x + 79) / 80 * 80 - x;
    return w80 < w64 ? 80 : 64;
}

/// N extent when the M extent is fixed at tbm: like tile_for, plus 40 (a
/// 4 x 1 warp grid) for 33..40 columns when tbm is a multiple of 32.
inline int tile_for_n(int x, int tbm) {
    if (x > 32 && x <= 40 && tbm % 32 == 0) return 40;
    return tile_for(x);
}

}  // namespace tile

/// Host: run f(std::integral_constant<int, T>) for the tile extent t.
template <class F>
void with_tile(int t, F&& f) {
    switch (t) {
        case 16: f(std::integral_constant<int, 16>{}); break;
        case 32: f(std::integral_constant<int, 32>{}); break;
        case 40: f(std::integral_constant<int, 40>{}); break;
        case 48: f(std::integral_constant<int, 48>{}); break;
        case 64: f(std::integral_constant<int, 64>{}); break;
        case 80: f(std::integral_constant<int, 80>{}); break;
        case 96: f(std::integral_constant<int, 96>{}); break;
        default: throw std::logic_error("with_tile: unsupported tile extent");
    }
}

/// Host: opt the kernel KFN into `bytes` of dynamic shared memory (once).
template <auto KFN>
void attr_once(int bytes) {
    static DeviceOnce once;
    if (!once.first()) return;
    if (bytes > 48 * 1024)
        HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(KFN), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     bytes));
}

}  // namespace hg
