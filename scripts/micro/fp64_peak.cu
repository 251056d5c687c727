// FP64 ceilings on this GPU: DMMA m8n8k4 issue rate and DFMA rate
// (register-only loops, no memory traffic).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
    double c[8][2] = {};
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(double* out, int iters) {
    double c[16];
    for (int j = 0; j < 16; ++j) c[j] = threadIdx.x + j;
    const double a = 1.0000001, b = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) c[j] = fma(c[j], a, b);
    }
    double s = 0;
    for (int j = 0; j < 16; ++j) s += c[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        const int iters = 20000, blocks = sms * 2, threads = warps * 32 / 2;
        k_dmma<<<blocks, threads>>>(out, 10);
        cudaEventRecord(e0);
        k_dmma<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = double(blocks) * (threads / 32) * iters * 8 * 512.0;
        printf("DMMA m8n8k4: %2d warps/SM  %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
    }
    for (int warps : {8, 16, 32, 64}) {
        const int iters = 20000, blocks = sms * 2, threads = warps * 32 / 2;
        k_dfma<<<blocks, threads>>>(out, 10);
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = double(blocks) * threads * iters * 16 * 2.0;
        printf("DFMA:        %2d warps/SM  %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
    }
    return 0;
}
