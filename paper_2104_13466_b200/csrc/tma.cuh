// TMA (cp.async.bulk.tensor) helpers for the element kernels: one 4D box
// (x, y, z, component) of a pitched FP64 lattice vector per element and
// component, loaded into shared memory with mbarrier completion, and the
// transposed result added back with a bulk tensor reduce-add (f64).  The
// tensor maps (one per device vector, sdme_abi.cu) live in global memory.
// Verified on B200 by tools/micro/tma_f64.cu (load, OOB fill, f64 reduce-add);
// the box's x start must be 16-byte aligned (even lattice x), else the copy
// faults with "illegal instruction".  Boxes therefore start at the even
// lattice x at or below the element's first point and are BoxW = (n + 2) & ~1
// points wide: n + 1 for even P, n + 2 for odd P, whose elements starting at
// an odd x read their rows shifted by one (make_tmap / launch_col).
#pragma once
#include <cuda.h>

#include "check.cuh"

namespace sdme {

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  SDME_CHECK(smem_ok(bar, 8, 8));
  asm volatile(
      "{\n .reg .pred p;\n W%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(
          smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// box load of lattice block (x0, y0, z0) of component c
__device__ __forceinline__ void tma_load_box(double* dst, const CUtensorMap* map, int x0, int y0, int z0, int c,
                                             unsigned long long* bar) {
  SDME_CHECK(smem_ok(dst, 128, 128) && smem_ok(bar, 8, 8) && (x0 & 1) == 0);
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(x0), "r"(y0), "r"(z0), "r"(c), "r"(smem_addr(bar))
      : "memory");
}

// the same box on its way into L2 (no shared-memory destination, no barrier)
__device__ __forceinline__ void tma_prefetch_box(const CUtensorMap* map, int x0, int y0, int z0, int c) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(map), "r"(x0),
               "r"(y0), "r"(z0), "r"(c)
               : "memory");
}

// y[box] += src  (bulk tensor reduce-add; elements outside the tensor are dropped)
__device__ __forceinline__ void tma_reduce_add_box(const CUtensorMap* map, const double* src, int x0, int y0, int z0,
                                                   int c) {
  SDME_CHECK(smem_ok(src, 128, 128) && (x0 & 1) == 0);
  asm volatile(
      "cp.reduce.async.bulk.tensor.4d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
          map),
      "r"(x0), "r"(y0), "r"(z0), "r"(c), "r"(smem_addr(src))
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// the source shared memory of every committed bulk op has been read
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// every committed bulk op has completed (global writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// generic-proxy shared writes -> visible to a following async-proxy (TMA) read
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// programmatic dependent launch (colour passes, ops.cu launch_col_k): the
// next launch on the stream may start as soon as every CTA of this grid has
// issued launch_dependents; it must wait (griddepcontrol.wait: the previous
// grid has completed and its memory is visible) before touching the output.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

}  // namespace sdme
