// Constants, scalar-state layout and status words shared by the PCG kernels
// (vector_kernels.cuh) and the small-mesh cluster kernel (pcg_small.cuh).
// Header-only: no kernels here, so any translation unit may include it.
#pragma once
#include <cuda_runtime.h>

namespace sdme {

constexpr int kRedBlocks = 592;   // 4 x 148 SMs: fixed -> deterministic partials
constexpr int kRedThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}

// device scalar state of a PCG solve (ctx->d_scal)
enum {
  S_RZ0 = 0,   // r.z of the previous iterate, ping-pong by iteration parity
  S_RZ1,
  S_PAP,
  S_ALPHA,
  S_BETA,
  S_NB,        // ||b||
  S_TOL,
  S_RELPREV,   // relative residual of the previous iterate (PCGError stats)
  S_ITER,      // iterations completed
  S_STOPREL,   // relative residual at stop
  S_MAXIT,
  S_SCRATCH,   // generic dot result
  S_ITERB,     // number of the iteration in flight (fused sequence: written by k_pcg_update2, read by k_pcg_p2)
  S_COUNT
};

enum { PCG_RUNNING = 0, PCG_CONVERGED = 1, PCG_INDEFINITE = 2, PCG_MAXIT = 3, PCG_STOPPED = 4 };

__device__ __forceinline__ bool pcg_done(const int* status) { return status && *(volatile const int*)status != 0; }

// end the enclosing conditional while-node (no-op outside a graph)
__device__ __forceinline__ void set_cond(cudaGraphConditionalHandle cond, int has_cond) {
  if (has_cond) cudaGraphSetConditional(cond, 0);
}

}  // namespace sdme
