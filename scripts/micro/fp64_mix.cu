#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_mix(double* out, int iters, int mode) {
    double c[8][2] = {};
    double f[16];
    for (int j = 0; j < 16; ++j) f[j] = threadIdx.x + j;
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    const double fa = 1.0000001, fb = 1e-7;
    const bool dm = (mode == 0) || (mode == 2 && (threadIdx.x >> 5) % 2 == 0) || mode == 3;
    const bool df = (mode == 1) || (mode == 2 && (threadIdx.x >> 5) % 2 == 1) || mode == 3;
    for (int it = 0; it < iters; ++it) {
        if (dm) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
        }
        if (df) {
#pragma unroll
            for (int j = 0; j < 16; ++j) f[j] = fma(f[j], fa, fb);
        }
    }
    double s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
    for (int j = 0; j < 16; ++j) s += f[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[] = {"DMMA only", "DFMA only", "half warps each", "both in every warp"};
    for (int mode = 0; mode < 4; ++mode) {
        const int iters = 20000, blocks = sms * 2, threads = 512;
        k_mix<<<blocks, threads>>>(out, 10, mode);
        cudaEventRecord(e0); k_mix<<<blocks, threads>>>(out, iters, mode); cudaEventRecord(e1);
        cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double warps = double(blocks) * threads / 32;
        double fl = 0;
        if (mode == 0) fl = warps * iters * 8 * 512.0;
        if (mode == 1) fl = warps * 32 * iters * 16 * 2.0;
        if (mode == 2) fl = warps / 2 * iters * 8 * 512.0 + warps / 2 * 32 * iters * 16 * 2.0;
        if (mode == 3) fl = warps * iters * 8 * 512.0 + warps * 32 * iters * 16 * 2.0;
        printf("%-20s %.2f TFLOP/s (%.2f ms)\n", names[mode], fl / (ms * 1e-3) / 1e12, ms);
    }
    return 0;
}
