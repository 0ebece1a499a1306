// One-launch PCG iteration tail for small meshes (E-vector mode).
//
// After the element kernel has written the element boxes of A p into the
// E-vector, a single 8-CTA thread-block cluster does the rest of the
// iteration (solver.py:140-165): gather A p, p.Ap, the indefinite test, alpha,
// the x / r update with (r.r, r.z), the convergence and maxit tests, beta and
// the p update.  Reductions go CTA -> distributed shared memory of the
// cluster, summed by every CTA in rank order, so every CTA takes the same
// decisions and the result is bit-reproducible.  The kernel also drives the
// conditional while-node of the PCG graph (cond = 0 once stopped).
//
// Replaces 6 launches (zero, pap, alpha, update, check, p) by one; for the
// BASELINE config-1 mesh (14.7K lattice entries) the whole vector state fits
// the cluster's L1/L2 working set.
#pragma once
#include <cooperative_groups.h>

#include "element_kernels.cuh"
#include "pcg_state.cuh"

namespace sdme {

#ifndef SDME_SMALL_CTA
#define SDME_SMALL_CTA 16
#endif
#ifndef SDME_SMALL_THREADS
#define SDME_SMALL_THREADS 1024
#endif
constexpr int kSmallCta = SDME_SMALL_CTA;  // non-portable cluster size above 8 (attribute set at launch)
constexpr int kSmallThreads = SDME_SMALL_THREADS;
constexpr long long kSmallPcgMax = 1LL << 18;  // lattice entries (3 Ns) for this path

// Cluster-wide sum of NV values: warp trees -> CTA tree (warp 0) -> the
// kSmallCta CTA partials read from distributed shared memory by lanes 0..7 of
// warp 0 and combined by the same fixed tree, so every CTA obtains the same
// bit-identical totals in tot[] (shared).  part[] must not be rewritten
// until every CTA has passed a later cluster barrier.
template <int NV>
__device__ __forceinline__ void cluster_sum(cooperative_groups::cluster_group& cl, double (&v)[NV],
                                            double (*red)[kSmallThreads / 32], double* part, double* tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const double s = warp_sum(v[k]);
    if (lane == 0) red[k][wid] = s;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double s = warp_sum(lane < kSmallThreads / 32 ? red[k][lane] : 0.0);
      if (lane == 0) part[k] = s;
    }
  }
  cl.sync();
  if (wid == 0) {
    const double* rp = cl.map_shared_rank(part, lane < kSmallCta ? lane : 0);
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const double s = warp_sum(lane < kSmallCta ? rp[k] : 0.0);
      if (lane == 0) tot[k] = s;
    }
  }
  __syncthreads();
}

template <int N>
__global__ void __launch_bounds__(kSmallThreads)
    k_pcg_small(double* __restrict__ x, double* __restrict__ r, double* __restrict__ p, double* __restrict__ ap,
                const double* __restrict__ dinv, const double* __restrict__ ev, const __grid_constant__ Geo g,
                double* s, int* status, cudaGraphConditionalHandle cond, int has_cond) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double red[2][kSmallThreads / 32];
  __shared__ double part[3], tot[3];
  const bool lead = cl.block_rank() == 0 && threadIdx.x == 0;
  // every read of the scalar state happens before any write (first cluster barrier)
  const bool done = pcg_done(status);
  const long long k = (long long)s[S_ITER] + 1;
  const double rz_old = s[S_RZ0 + ((k - 1) & 1)], nb = s[S_NB], tol = s[S_TOL], maxit = s[S_MAXIT],
               relprev = s[S_RELPREV];
  cl.sync();
  if (done) {
    if (lead) set_cond(cond, has_cond);
    return;
  }
  // launched as a programmatic dependent of the element kernel (which wrote
  // the E-vector): everything above overlapped it
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const long long n = 3 * g.Ns;
  const long long i0 = (long long)cl.block_rank() * kSmallThreads + threadIdx.x;
  constexpr long long stride = (long long)kSmallCta * kSmallThreads;
  // A p (gathered) and p.Ap
  double a1[1] = {0.0};
  for (long long i = i0; i < n; i += stride) {
    double v = 0.0;
    if (!ev_point<N>(ev, g, i, v)) v = 0.0;
    ap[i] = v;
    a1[0] = fma(p[i], v, a1[0]);
  }
  cluster_sum<1>(cl, a1, red, part, tot);
  const double pap = tot[0];
  if (!(pap > 0.0)) {
    if (lead) {
      s[S_PAP] = pap;
      s[S_ITER] = (double)k;
      s[S_STOPREL] = relprev;
      *status = PCG_INDEFINITE;
      set_cond(cond, has_cond);
    }
    cl.sync();
    return;
  }
  const double alpha = rz_old / pap;
  if (lead) {
    s[S_PAP] = pap;
    s[S_ALPHA] = alpha;
  }
  // x += alpha p ; r -= alpha Ap ; (r.r, r.z)
  double a2[2] = {0.0, 0.0};
  for (long long i = i0; i < n; i += stride) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, ap[i], r[i]);
    r[i] = ri;
    a2[0] = fma(ri, ri, a2[0]);
    a2[1] = fma(ri, dinv[i] * ri, a2[1]);
  }
  cluster_sum<2>(cl, a2, red, part + 1, tot + 1);
  const double rr = tot[1], rz = tot[2];
  cl.sync();  // remote reads done before any CTA exits
  const double rel = sqrt(rr) / nb;
  if (rel <= tol || (double)k >= maxit) {
    if (lead) {
      s[S_ITER] = (double)k;
      s[S_STOPREL] = rel;
      *status = rel <= tol ? PCG_CONVERGED : PCG_MAXIT;
      set_cond(cond, has_cond);
    }
    return;
  }
  const double beta = rz / rz_old;
  if (lead) {
    s[S_ITER] = (double)k;
    s[S_RELPREV] = rel;
    s[S_BETA] = beta;
    s[S_RZ0 + (k & 1)] = rz;
  }
  for (long long i = i0; i < n; i += stride) p[i] = fma(beta, p[i], dinv[i] * r[i]);
}

}  // namespace sdme
