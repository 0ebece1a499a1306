// FP64 DFMA-chain microbenchmark: measures the sustained FP64 FMA rate of the
// B200 this runs on (the roofline denominator for the FP64-bound element
// kernels; MEASURED_PEAKS.json carries only HBM and bf16 figures).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_chain(double* out, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
#pragma unroll
            for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int threads : {256, 512, 1024}) {
        for (int bps : {1, 2, 4}) {
            if (threads * bps > 2048) continue;
            int blocks = sms * bps;
            dfma_chain<8><<<blocks, threads>>>(out, 16, 0.999999, 1e-7);
            cudaDeviceSynchronize();
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(e0);
                dfma_chain<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
            printf("{\"threads\": %d, \"blocks_per_sm\": %d, \"ms\": %.4f, \"fp64_tflops\": %.3f}\n",
                   threads, bps, best, flops / best / 1e9);
        }
    }
    printf("{\"sms\": %d, \"clock_khz\": %d, \"err\": \"%s\"}\n", sms, clk,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
