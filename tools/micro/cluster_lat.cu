// Launch + barrier latency micro-benchmark (design aid for pcg_small.cuh):
// back-to-back launches of an (almost) empty kernel, as plain kernels and as
// 8-CTA clusters, with k cluster barriers, timed with CUDA events.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_plain(int* x, int nsync) {
  for (int i = 0; i < nsync; ++i) __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1;
}
__global__ void __cluster_dims__(8, 1, 1) k_cluster(int* x, int nsync) {
  cg::cluster_group cl = cg::this_cluster();
  for (int i = 0; i < nsync; ++i) cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1;
}
__global__ void __cluster_dims__(8, 1, 1) k_cluster_rd(int* x, const double* v, int n, int nsync) {
  cg::cluster_group cl = cg::this_cluster();
  double s = 0;
  for (int r = 0; r < nsync; ++r) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) s += v[i];
    cl.sync();
  }
  if (s == 12345.0) x[1] = 1;
  if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1;
}

int main() {
  int* x;
  double* v;
  cudaMalloc(&x, 8);
  cudaMalloc(&v, 1 << 20);
  cudaMemset(v, 0, 1 << 20);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 20; ++i) launch();
    cudaStreamSynchronize(st);
    // graph of 100 launches
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 100; ++i) launch();
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    cudaEventRecord(a, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %8.2f us/launch\n", name, ms * 10.0f);
  };
  for (int ns : {0, 4}) {
    char nm[64];
    snprintf(nm, 64, "plain 8x1024, %d syncthreads", ns);
    run(nm, [&] { k_plain<<<8, 1024, 0, st>>>(x, ns); });
    snprintf(nm, 64, "cluster 8x1024, %d cluster syncs", ns);
    run(nm, [&] { k_cluster<<<8, 1024, 0, st>>>(x, ns); });
    snprintf(nm, 64, "cluster 8x256, %d cluster syncs", ns);
    run(nm, [&] { k_cluster<<<8, 256, 0, st>>>(x, ns); });
  }
  for (int n : {15000, 110000}) {
    char nm[64];
    snprintf(nm, 64, "cluster 8x1024 read %d x4 + sync", n);
    run(nm, [&] { k_cluster_rd<<<8, 1024, 0, st>>>(x, v, n, 4); });
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
