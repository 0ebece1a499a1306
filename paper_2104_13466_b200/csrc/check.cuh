// Device-side bounds / alignment checks of the checked build (-DSDME_CHECKED,
// `python -m paper_2104_13466_b200.build --checked` -> libsdme_checked.so).
// compute-sanitizer is not available on the GPU pool this is measured on, so
// the checked build is the memory-safety evidence: every TMA box / mbarrier /
// vector shared access and every shared-layout index is verified at run time,
// and a violation traps with the kernel's file:line.  Compiled out otherwise.
#pragma once
#include <cstdio>

#ifdef SDME_CHECKED
#define SDME_CHECK(cond)                                                                          \
  do {                                                                                            \
    if (!(cond)) {                                                                                \
      printf("SDME_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                                  \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define SDME_CHECK(cond) \
  do {                   \
  } while (0)
#endif

namespace sdme {

__device__ __forceinline__ unsigned dyn_smem_bytes() {
  unsigned v;
  asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
  return v;
}

// p .. p + bytes lies in this CTA's dynamic shared memory and is `align`-aligned
__device__ __forceinline__ bool smem_ok(const void* p, unsigned bytes, unsigned align) {
  extern __shared__ __align__(128) double smem[];
  const unsigned a = (unsigned)__cvta_generic_to_shared(p), base = (unsigned)__cvta_generic_to_shared(smem);
  return a >= base && a + bytes <= base + dyn_smem_bytes() && (a % align) == 0;
}

}  // namespace sdme
