// tools/fp32_peak.cu — measured FP32 issue peak on this B200: independent FFMA
// chains (8 per thread, register-only), 148 x 8 blocks x 256 threads, timed
// with CUDA events.  Writes profiles/fp32_peak.json when given a path.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_chains(float* out, int iters, float a, float b) {
    float x0 = threadIdx.x * 1e-7f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
          x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 20000;
    float* out;
    cudaMalloc(&out, sizeof(float) * blocks * threads);
    ffma_chains<<<blocks, threads>>>(out, 100, 0.999f, 1e-3f);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        ffma_chains<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double lane_ops = double(blocks) * threads * iters * 16 * 8;
    const double rate = lane_ops / (best * 1e-3);
    printf("{\"ffma_lane_ops_per_s\": %.6e, \"tflops_fma2\": %.3f, \"sms\": %d, \"ms\": %.3f, "
           "\"how\": \"8 independent FFMA chains/thread, %d blocks x %d threads, best of 5, CUDA events\"}\n",
           rate, 2 * rate / 1e12, sms, best, blocks, threads);
    return cudaGetLastError() != cudaSuccess;
}
