// Micro-test: TMA tensor load of an FP64 element box from a pitched lattice
// (box 6 x 5 x 5 x 3), TMA tensor reduce-add (f64) of the box back, and the
// non-tensor bulk reduce-add of 48-byte rows.  Prints PASS/FAIL per feature.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tma_f64.cu -o tma_f64
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#ifndef BXV
#define BXV 6
#define BYV 5
#endif
constexpr int Lx = 9, Px = 10, Ly = 9, Lz = 9, BX = BXV, BY = BYV, BZ = BYV;
constexpr long long Ns = (long long)Px * Ly * Lz;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k_tensor(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, int x0,
                         int y0, int z0) {
  __shared__ alignas(128) double box[(3 * BZ * BY * BX + 15) / 16 * 16];
  __shared__ alignas(8) unsigned long long bar;
  const int t = threadIdx.x;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (t == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                 "r"((int)(3 * BZ * BY * BX * 8)));
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(smem_u32(box)),
        "l"(&tin), "r"(x0), "r"(y0), "r"(z0), "r"(0), "r"(smem_u32(&bar))
        : "memory");
  }
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }" ::"r"(smem_u32(&bar))
      : "memory");
  for (int i = t; i < 3 * BZ * BY * BX; i += blockDim.x) box[i] = 2.0 * box[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (t == 0) {
    asm volatile("cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                     &tout),
                 "r"(x0), "r"(y0), "r"(z0), "r"(0), "r"(smem_u32(box))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// non-tensor: rows of 6 doubles (48 B) at 16-byte aligned addresses
__global__ void k_rows(const double* __restrict__ in, double* out, int x0, int y0, int z0) {
  __shared__ alignas(128) double rows[3 * BZ * BY * BX];
  __shared__ alignas(8) unsigned long long bar;
  const int t = threadIdx.x;
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (t == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                 "r"((int)sizeof(rows)));
  __syncthreads();
  if (t < 3 * BZ * BY) {
    const int c = t / (BZ * BY), k = (t / BY) % BZ, j = t % BY;
    const double* src = in + c * Ns + ((long long)(z0 + k) * Ly + y0 + j) * Px + x0;
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 48, [%2];" ::"r"(
            smem_u32(rows + t * BX)),
        "l"(src), "r"(smem_u32(&bar))
        : "memory");
  }
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W; }" ::"r"(smem_u32(&bar))
      : "memory");
  for (int i = t; i < 3 * BZ * BY * BX; i += blockDim.x) rows[i] = 2.0 * rows[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (t < 3 * BZ * BY) {
    const int c = t / (BZ * BY), k = (t / BY) % BZ, j = t % BY;
    double* dst = out + c * Ns + ((long long)(z0 + k) * Ly + y0 + j) * Px + x0;
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 48;" ::"l"(dst),
                 "r"(smem_u32(rows + t * BX))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

static int check(const char* what, const std::vector<double>& x, const std::vector<double>& y, int x0, int y0, int z0,
                 int xmax) {
  int bad = 0;
  for (int c = 0; c < 3; ++c)
    for (int Z = 0; Z < Lz; ++Z)
      for (int Y = 0; Y < Ly; ++Y)
        for (int X = 0; X < Px; ++X) {
          const long long i = c * Ns + ((long long)Z * Ly + Y) * Px + X;
          const bool in = X >= x0 && X < x0 + BX && X < xmax && Y >= y0 && Y < y0 + BY && Z >= z0 && Z < z0 + BZ;
          const double want = in ? 1.0 + 2.0 * x[i] : 1.0;
          if (y[i] != want) {
            if (bad < 5) printf("  %s mismatch c%d (%d,%d,%d): %g vs %g\n", what, c, X, Y, Z, y[i], want);
            ++bad;
          }
        }
  printf("%s: %s (%d bad)\n", what, bad ? "FAIL" : "PASS", bad);
  return bad;
}

int main() {
  const long long n = 3 * Ns;
  std::vector<double> x(n), one(n, 1.0), y(n);
  for (long long i = 0; i < n; ++i) x[i] = ((i * 7919) % 1000) * 1e-3 + 0.125;
  double *dx, *dy;
  cudaMalloc(&dx, n * 8);
  cudaMalloc(&dy, n * 8);
  cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
  auto enc = encode();
  CUtensorMap tin, tout;
  cuuint64_t dims[4] = {Lx, Ly, Lz, 3};
  cuuint64_t strides[3] = {Px * 8ull, (cuuint64_t)Px * Ly * 8ull, (cuuint64_t)Ns * 8ull};
  cuuint32_t box[4] = {BX, BY, BZ, 3}, es[4] = {1, 1, 1, 1};
  CUresult r1 = enc(&tin, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, dx, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, dy, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d %d\n", (int)r1, (int)r2);
  int bad = 0;
  // x0 = 4: box reaches X = 9 (out of bounds, dropped).  An odd x0 (a box
  // start 8 bytes off a 16-byte boundary) raises "illegal instruction" on B200
  // (measured), so the element kernels use the TMA path for even P only.
  for (int x0 : {0, 4}) {
    cudaMemcpy(dy, one.data(), n * 8, cudaMemcpyHostToDevice);
    k_tensor<<<1, 128>>>(tin, tout, x0, 4, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("tensor x0=%d: %s\n", x0, cudaGetErrorString(e));
    cudaMemcpy(y.data(), dy, n * 8, cudaMemcpyDeviceToHost);
    bad += check("tensor load + reduce-add f64", x, y, x0, 4, 0, Lx);
  }
  cudaMemcpy(dy, one.data(), n * 8, cudaMemcpyHostToDevice);
  k_rows<<<1, 128>>>(dx, dy, 4, 2, 4);
  cudaError_t e = cudaDeviceSynchronize();
  printf("rows: %s\n", cudaGetErrorString(e));
  cudaMemcpy(y.data(), dy, n * 8, cudaMemcpyDeviceToHost);
  bad += check("bulk rows load + reduce-add f64", x, y, 4, 2, 4, Px);
  return bad ? 1 : 0;
}
