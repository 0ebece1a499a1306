// FP64 tensor-core (DMMA, mma.sync.m8n8k4.f64) throughput on this B200, for
// the tensor-core decision in DESIGN.md: independent accumulator chains per
// warp, all SMs, CUDA-event timing.  Prints JSON lines (TF/s counted as
// 2*8*8*4 flops per warp-level MMA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu
#include <cuda_runtime.h>

#include <cstdio>

template <int ILP>
__global__ void dmma_chain(double* out, int iters) {
  // a: 8x4 (one double per lane), b: 4x8 (one per lane), c/d: 8x8 (two per lane)
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5 - threadIdx.x * 1e-9;
  double c0[ILP], c1[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) c0[i] = c1[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c0[i]), "+d"(c1[i])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c0[i] + c1[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 8192;
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      if (threads * bps > 2048) continue;
      const int blocks = sms * bps;
      dmma_chain<8><<<blocks, threads>>>(out, 16);
      cudaDeviceSynchronize();
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dmma_chain<8><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const double mmas = 8.0 * iters * (threads / 32) * (double)blocks;
      printf("{\"threads\": %d, \"blocks_per_sm\": %d, \"ms\": %.4f, \"dmma_tflops\": %.3f}\n", threads, bps, best,
             mmas * 2 * 8 * 8 * 4 / best / 1e9);
    }
  }
  printf("{\"sms\": %d, \"clock_khz\": %d, \"err\": \"%s\"}\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
