// fp32_peak.cu -- measured FP32 (CUDA-core FFMA) peak of this B200, the denominator of bench.py's
// "fp32" roofline entry (north_star: kernel choices evidenced against the FP32 peak;
// MEASURED_PEAKS.json carries only HBM and bf16 tensor peaks).
//
// Every thread runs 8 independent FFMA chains (enough ILP to cover the 4-cycle FMA latency at
// 1024 threads per SM); grid = 148 x 8 CTAs of 256 threads, timed with CUDA events after a
// warm-up, best of 10.  flops = 2 per FFMA.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) ffma_kernel(float *out, int iters, float a, float b) {
    float x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; c++) x[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 16; k++) {
#pragma unroll
            for (int c = 0; c < kChains; c++) x[c] = fmaf(x[c], a, b);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; c++) s += x[c];
    if (s == 12345.678f) out[blockIdx.x] = s;   // keeps the chains live
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    float *out;
    cudaMalloc(&out, blocks * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    ffma_kernel<<<blocks, threads>>>(out, iters, 0.9999f, 1e-4f);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; r++) {
        cudaEventRecord(e0);
        ffma_kernel<<<blocks, threads>>>(out, iters, 0.9999f, 1e-4f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double flops = 2.0 * (double)blocks * threads * iters * 16 * kChains;
    cudaError_t err = cudaGetLastError();
    printf("{\"fp32_tflops\": %.3f, \"ms\": %.4f, \"sms\": %d, \"blocks\": %d, \"threads\": %d, \"ffma_per_thread\": %d, "
           "\"error\": \"%s\"}\n",
           flops / (best * 1e-3) / 1e12, best, sms, blocks, threads, iters * 16 * kChains, cudaGetErrorString(err));
    return err == cudaSuccess ? 0 : 1;
}
