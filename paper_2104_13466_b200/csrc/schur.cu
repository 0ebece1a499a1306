// Assembled linear-solve path of the reference's default solver configuration
// (SolverConfig(precond="sgs", condense=True), dynamics.py:38-43): dense
// element matrices of c_k K_T(u) + c_m M on the device, per-element static
// condensation of the interior modes (condense_elements, solver.py:258-293:
// Cholesky of K_ii, Schur K_bb - K_ib^T K_ii^-1 K_ib), deterministic assembly
// of the boundary Schur complement in CSR, PCG (solver.py:129-170) on it with
// the symmetric Gauss-Seidel preconditioner (solver.py:78-120) run as
// level-scheduled triangular sweeps, and the interior recovery
// (CondensedSystem.reduce_rhs / recover, solver.py:186-203).  With no interior
// modes (condense=False) the same machinery assembles the full free-DOF
// operator (make_solver's CSR branch, dynamics.py:118-126).
//
// Element matrix (box meshes, identical element geometry): with G_f(q) the
// physical gradient of local function f at point q, K = F^-T, kappa = mu -
// lam ln J, the tangent's bilinear form is
//   K_e[(f,c),(g,c')] = sum_q w_q detJ [ mu d_cc' G_f.G_g + lam (K_c.G_f)(K_c'.G_g)
//                                        + kappa (K_c.G_g)(K_c'.G_f) ]
// (the same dP = mu Hp + lam (K:Hp) K + kappa K Hp^T K as the matrix-free
// kernels, i.e. the reference's B^T D B + geometric term, material.py:84-105,
// femcore.py:130-146), so with S[q][(f,c)] = K_c.G_f(q) the u-dependent part is
// two weighted Gram products of S; mu sum_q w G_f.G_g and the mass
// rho sum_q w N_f N_g are u-independent and tabulated once.
//
// Everything here is sized for the meshes the reference itself can assemble
// (dense element matrices, 1.1 MB per element at P = 4); the matrix-free path
// is the one for large meshes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "sdme.h"

namespace {

constexpr unsigned long long kNone = ~0ull;
constexpr int kTF = 16;        // element-matrix tile: 16 x 16 functions (48 x 48 dofs)
constexpr int kQC = 8;         // quadrature points per smem chunk
constexpr int kSolveThreads = 1024;
constexpr int kRed = 256;      // reduction block
constexpr int kRedGrid = 296;  // fixed grid -> deterministic partial sums

// ------------------------------------------------------------ device kernels

// per element and point: S[e][q][f*3+c] = K_c . G_f(q), wk[e][q] = w detJ (mu - lam lnJ)
__global__ void k_point_state(const double* __restrict__ u, const long long* __restrict__ addr, int nd, int nq,
                              const double* __restrict__ G, const double* __restrict__ wdet, double mu, double lam,
                              double* __restrict__ S, double* __restrict__ wk, unsigned long long* flag) {
  extern __shared__ double ue[];
  const long long e = blockIdx.x;
  for (int l = threadIdx.x; l < nd; l += blockDim.x) {
    const long long a = addr[e * nd + l];
    ue[l] = a >= 0 ? u[a] : 0.0;
  }
  __syncthreads();
  const int nf = nd / 3;
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    double H[3][3] = {};
    const double* gq = G + (long long)q * nf * 3;
    for (int f = 0; f < nf; ++f)
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) H[c][d] = fma(ue[f * 3 + c], gq[f * 3 + d], H[c][d]);
    const double F00 = 1.0 + H[0][0], F01 = H[0][1], F02 = H[0][2];
    const double F10 = H[1][0], F11 = 1.0 + H[1][1], F12 = H[1][2];
    const double F20 = H[2][0], F21 = H[2][1], F22 = 1.0 + H[2][2];
    const double c00 = F11 * F22 - F12 * F21, c01 = F12 * F20 - F10 * F22, c02 = F10 * F21 - F11 * F20;
    const double det = F00 * c00 + F01 * c01 + F02 * c02;
    if (!(det > 0.0)) {
      atomicMin(flag, (unsigned long long)e * nq + q);
      continue;
    }
    const double inv = 1.0 / det;
    double K[3][3];  // cof(F) / det = F^-T
    K[0][0] = c00 * inv, K[0][1] = c01 * inv, K[0][2] = c02 * inv;
    K[1][0] = (F02 * F21 - F01 * F22) * inv, K[1][1] = (F00 * F22 - F02 * F20) * inv,
    K[1][2] = (F01 * F20 - F00 * F21) * inv;
    K[2][0] = (F01 * F12 - F02 * F11) * inv, K[2][1] = (F02 * F10 - F00 * F12) * inv,
    K[2][2] = (F00 * F11 - F01 * F10) * inv;
    wk[e * nq + q] = wdet[q] * (mu - lam * log(det));
    double* sq = S + (e * nq + q) * nd;
    for (int f = 0; f < nf; ++f)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        sq[f * 3 + c] = fma(K[c][0], gq[f * 3], fma(K[c][1], gq[f * 3 + 1], K[c][2] * gq[f * 3 + 2]));
  }
}

// Ke[e] = c_k (mu L (x) I + sum_q wl S S^T + swap(sum_q wk S S^T)) + c_m rho Mref (x) I
// one 16 x 16 function tile per block (256 threads, a 3 x 3 dof block each)
__global__ void __launch_bounds__(kTF* kTF) k_elem_matrix(const double* __restrict__ S, const double* __restrict__ wk,
                                                          const double* __restrict__ wdet, const double* __restrict__ Lg,
                                                          const double* __restrict__ Mr, int nf, int nq, double ck,
                                                          double cm, double mu, double lam, double rho,
                                                          double* __restrict__ Ke) {
  __shared__ double sr[kQC][3 * kTF], sc[kQC][3 * kTF], wl_s[kQC], wk_s[kQC];
  const long long e = blockIdx.z;
  const int nd = 3 * nf;
  const int fr = blockIdx.y * kTF + threadIdx.y, fc = blockIdx.x * kTF + threadIdx.x;
  const int tid = threadIdx.y * kTF + threadIdx.x;
  double t2[3][3] = {}, t3[3][3] = {};
  if (ck != 0.0) {
    for (int q0 = 0; q0 < nq; q0 += kQC) {
      __syncthreads();
      for (int i = tid; i < kQC * 3 * kTF; i += kTF * kTF) {
        const int qq = i / (3 * kTF), l = i % (3 * kTF), q = q0 + qq;
        const int rr = blockIdx.y * kTF * 3 + l, cc = blockIdx.x * kTF * 3 + l;
        const bool okq = q < nq;
        sr[qq][l] = okq && rr < nd ? S[(e * nq + q) * nd + rr] : 0.0;
        sc[qq][l] = okq && cc < nd ? S[(e * nq + q) * nd + cc] : 0.0;
      }
      if (tid < kQC) {
        const int q = q0 + tid;
        wl_s[tid] = q < nq ? wdet[q] * lam : 0.0;
        wk_s[tid] = q < nq ? wk[e * nq + q] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int qq = 0; qq < kQC; ++qq) {
        const double a0 = sr[qq][threadIdx.y * 3], a1 = sr[qq][threadIdx.y * 3 + 1], a2 = sr[qq][threadIdx.y * 3 + 2];
        const double b0 = sc[qq][threadIdx.x * 3], b1 = sc[qq][threadIdx.x * 3 + 1], b2 = sc[qq][threadIdx.x * 3 + 2];
        const double A[3] = {a0, a1, a2}, B[3] = {b0, b1, b2};
        const double wl = wl_s[qq], wq = wk_s[qq];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            t2[i][j] = fma(wl * A[i], B[j], t2[i][j]);
            t3[i][j] = fma(wq * A[j], B[i], t3[i][j]);
          }
      }
    }
  }
  if (fr >= nf || fc >= nf) return;
  const double lg = Lg[(long long)fr * nf + fc], mr = Mr[(long long)fr * nf + fc];
  double* out = Ke + e * (long long)nd * nd;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double v = ck * (t2[i][j] + t3[i][j] + (i == j ? mu * lg : 0.0));
      if (i == j) v += cm * rho * mr;
      out[(long long)(fr * 3 + i) * nd + fc * 3 + j] = v;
    }
}

// per element (one CTA): Cholesky of K_ii (lower, in place), X = K_ii^-1 K_ib,
// Schur_e = K_bb - K_ib^T X.  Workspace per element: Lw (ni^2), X (ni*nbe),
// Sch (nbe^2); bl / il: local dof lists (ascending local order).
__global__ void __launch_bounds__(kSolveThreads) k_condense(const double* __restrict__ Ke, int nd,
                                                            const int* __restrict__ loc, const long long* __restrict__ off,
                                                            const int* __restrict__ nbe_a, const int* __restrict__ ni_a,
                                                            double* __restrict__ Lw, double* __restrict__ Xw,
                                                            double* __restrict__ Sch, const long long* __restrict__ woff,
                                                            const long long* __restrict__ soff,
                                                            unsigned long long* flag) {
  const long long e = blockIdx.x;
  const int nbe = nbe_a[e], ni = ni_a[e];
  const int* bl = loc + off[e];
  const int* il = bl + nbe;
  const double* K = Ke + e * (long long)nd * nd;
  double* L = Lw + woff[e];
  double* X = Xw + woff[e] + (long long)ni * ni;
  double* Sc = Sch + soff[e];
  const int t = threadIdx.x, T = blockDim.x;
  __shared__ int fail;
  if (t == 0) fail = 0;
  for (long long i = t; i < (long long)ni * ni; i += T) L[i] = K[(long long)il[i / ni] * nd + il[i % ni]];
  for (long long i = t; i < (long long)ni * nbe; i += T) X[i] = K[(long long)il[i / nbe] * nd + bl[i % nbe]];
  __syncthreads();
  // right-looking Cholesky, column j at a time (lower triangle used)
  for (int j = 0; j < ni; ++j) {
    const double piv = L[(long long)j * ni + j];
    if (!(piv > 0.0)) {
      if (t == 0) fail = 1;
      break;
    }
    const double d = sqrt(piv);
    __syncthreads();
    if (t == 0) L[(long long)j * ni + j] = d;
    for (int i = j + 1 + t; i < ni; i += T) L[(long long)i * ni + j] /= d;
    __syncthreads();
    const int m = ni - j - 1;
    for (long long w = t; w < (long long)m * m; w += T) {
      // trailing lower triangle: (i, k) with j < k <= i
      const int i = j + 1 + (int)(w / m), k = j + 1 + (int)(w % m);
      if (k <= i) L[(long long)i * ni + k] -= L[(long long)i * ni + j] * L[(long long)k * ni + j];
    }
    __syncthreads();
  }
  __syncthreads();
  if (fail) {
    if (t == 0) atomicMin(flag, (unsigned long long)e);
    return;
  }
  // X = L^-T L^-1 K_ib, one column per thread
  for (int k = t; k < nbe; k += T) {
    for (int i = 0; i < ni; ++i) {
      double s = X[(long long)i * nbe + k];
      for (int jj = 0; jj < i; ++jj) s -= L[(long long)i * ni + jj] * X[(long long)jj * nbe + k];
      X[(long long)i * nbe + k] = s / L[(long long)i * ni + i];
    }
    for (int i = ni - 1; i >= 0; --i) {
      double s = X[(long long)i * nbe + k];
      for (int jj = i + 1; jj < ni; ++jj) s -= L[(long long)jj * ni + i] * X[(long long)jj * nbe + k];
      X[(long long)i * nbe + k] = s / L[(long long)i * ni + i];
    }
  }
  __syncthreads();
  // Sc = K_bb - K_ib^T X
  for (long long w = t; w < (long long)nbe * nbe; w += T) {
    const int a = (int)(w / nbe), b = (int)(w % nbe);
    double s = K[(long long)bl[a] * nd + bl[b]];
    for (int i = 0; i < ni; ++i) s -= K[(long long)il[i] * nd + bl[a]] * X[(long long)i * nbe + b];
    Sc[w] = s;
  }
}

// vals[s] = sum of the slot's contributions in element order (deterministic)
__global__ void k_gather_sum(const long long* __restrict__ ptr, const long long* __restrict__ src,
                             const double* __restrict__ from, double* __restrict__ vals, long long n) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < n; s += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (long long k = ptr[s]; k < ptr[s + 1]; ++k) acc += from[src[k]];
    vals[s] = acc;
  }
}

// y = A x (CSR), one warp per row, fixed lane order and tree
__global__ void k_spmv(const long long* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                       const double* __restrict__ x, double* __restrict__ y, long long n) {
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * blockDim.x / 32;
  for (long long i = w; i < n; i += nw) {
    double s = 0.0;
    for (long long k = rp[i] + lane; k < rp[i + 1]; k += 32) s = fma(v[k], x[ci[k]], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) y[i] = s;
  }
}

// symmetric Gauss-Seidel z = (D+U)^-1 D (D+L)^-1 r (solver.py:78-120), as two
// level-scheduled sweeps in one CTA; rows of one level are independent
__global__ void __launch_bounds__(kSolveThreads) k_sgs(const long long* __restrict__ rp, const int* __restrict__ ci,
                                                       const double* __restrict__ v, const double* __restrict__ dg,
                                                       const int* __restrict__ frow, const int* __restrict__ fptr,
                                                       int nfl, const int* __restrict__ brow,
                                                       const int* __restrict__ bptr, int nbl,
                                                       const double* __restrict__ r, double* __restrict__ z) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  for (int lv = 0; lv < nfl; ++lv) {
    for (int k = fptr[lv] + warp; k < fptr[lv + 1]; k += nwarp) {
      const int i = frow[k];
      double s = 0.0;
      for (long long q = rp[i] + lane; q < rp[i + 1]; q += 32) {
        const int j = ci[q];
        if (j < i) s = fma(v[q], z[j], s);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) z[i] = (r[i] - s) / dg[i];
    }
    __syncthreads();
  }
  for (int lv = 0; lv < nbl; ++lv) {
    for (int k = bptr[lv] + warp; k < bptr[lv + 1]; k += nwarp) {
      const int i = brow[k];
      double s = 0.0;
      for (long long q = rp[i] + lane; q < rp[i + 1]; q += 32) {
        const int j = ci[q];
        if (j != i) s = fma(v[q], z[j], s);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) z[i] = (r[i] - s) / dg[i];
    }
    __syncthreads();
  }
}

__global__ void k_diag_of(const long long* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ v,
                          double* __restrict__ dg, long long n, unsigned long long* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double d = 0.0;
    for (long long k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] == i) d = v[k];
    dg[i] = d;
    if (!(d > 0.0)) atomicMin(flag, (unsigned long long)i);
  }
}

// deterministic dot: fixed grid, fixed in-block tree, partials summed in order
__global__ void __launch_bounds__(kRed) k_dot2(const double* __restrict__ a, const double* __restrict__ b, long long n,
                                               double* __restrict__ part) {
  __shared__ double red[kRed / 32];
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)kRed + threadIdx.x; i < n; i += (long long)kRedGrid * kRed)
    s = fma(a[i], b[i], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRed / 32; ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void k_dot_finish(const double* __restrict__ part, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < kRedGrid; ++k) t += part[k];
    *out = t;
  }
}

// y = a x + b y
__global__ void k_axpby(double a, const double* __restrict__ x, double b, double* __restrict__ y, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = fma(a, x[i], b * y[i]);
}

__global__ void k_scale_copy(double* __restrict__ z, const double* __restrict__ d, const double* __restrict__ r,
                             long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    z[i] = d ? r[i] / d[i] : r[i];
}

// b_sc[k] = b[addr_b[k]] - sum over (element order) of v_e contributions
__global__ void k_reduce_v(const double* __restrict__ b, const long long* __restrict__ addr, const int* __restrict__ loc,
                           const long long* __restrict__ off, const int* __restrict__ nbe_a,
                           const int* __restrict__ ni_a, const double* __restrict__ Xw,
                           const long long* __restrict__ woff, double* __restrict__ v, const long long* __restrict__ voff,
                           int nd) {
  const long long e = blockIdx.x;
  const int nbe = nbe_a[e], ni = ni_a[e];
  const int* il = loc + off[e] + nbe;
  const double* X = Xw + woff[e] + (long long)ni * ni;
  for (int k = threadIdx.x; k < nbe; k += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < ni; ++i) s = fma(X[(long long)i * nbe + k], b[addr[e * nd + il[i]]], s);
    v[voff[e] + k] = s;
  }
}

__global__ void k_reduce_rhs(const double* __restrict__ b, const long long* __restrict__ addr_b,
                             const long long* __restrict__ ptr, const long long* __restrict__ src,
                             const double* __restrict__ v, double* __restrict__ bsc, long long nb) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nb; k += (long long)gridDim.x * blockDim.x) {
    double acc = b[addr_b[k]];
    for (long long j = ptr[k]; j < ptr[k + 1]; ++j) acc -= v[src[j]];
    bsc[k] = acc;
  }
}

// x[addr_b] = u_b; per element x_i = K_ii^-1 (b_i - K_ib u_b)
__global__ void k_scatter_b(const double* __restrict__ ub, const long long* __restrict__ addr_b, double* __restrict__ x,
                            long long nb) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nb; k += (long long)gridDim.x * blockDim.x)
    x[addr_b[k]] = ub[k];
}

__global__ void k_recover(const double* __restrict__ b, const double* __restrict__ ub, const double* __restrict__ Ke,
                          int nd, const long long* __restrict__ addr, const int* __restrict__ loc,
                          const long long* __restrict__ off, const int* __restrict__ nbe_a, const int* __restrict__ ni_a,
                          const int* __restrict__ bidx, const double* __restrict__ Lw, const long long* __restrict__ woff,
                          double* __restrict__ tmp, const long long* __restrict__ toff, double* __restrict__ x) {
  const long long e = blockIdx.x;
  const int nbe = nbe_a[e], ni = ni_a[e];
  const int* bl = loc + off[e];
  const int* il = bl + nbe;
  const int* bi = bidx + off[e];
  const double* K = Ke + e * (long long)nd * nd;
  const double* L = Lw + woff[e];
  double* y = tmp + toff[e];
  for (int i = threadIdx.x; i < ni; i += blockDim.x) {
    double s = b[addr[e * nd + il[i]]];
    for (int k = 0; k < nbe; ++k) s -= K[(long long)il[i] * nd + bl[k]] * ub[bi[k]];
    y[i] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < ni; ++i) {
      double s = y[i];
      for (int j = 0; j < i; ++j) s -= L[(long long)i * ni + j] * y[j];
      y[i] = s / L[(long long)i * ni + i];
    }
    for (int i = ni - 1; i >= 0; --i) {
      double s = y[i];
      for (int j = i + 1; j < ni; ++j) s -= L[(long long)j * ni + i] * y[j];
      y[i] = s / L[(long long)i * ni + i];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ni; i += blockDim.x) x[addr[e * nd + il[i]]] = y[i];
}

template <class T>
T* dev_copy(const std::vector<T>& h) {
  T* d = nullptr;
  if (h.empty()) return nullptr;
  if (cudaMalloc(&d, h.size() * sizeof(T)) != cudaSuccess) return nullptr;
  cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
  return d;
}

}  // namespace

struct sdme_schur {
  sdme_ctx* ctx = nullptr;
  int nd = 0, nf = 0, nq = 0;
  long long ne = 0, nb = 0, nnz = 0;
  double mu = 0, lam = 0, rho = 0;
  // element tables (device)
  long long* addr = nullptr;   // [e][nd] lattice address or -1
  int* loc = nullptr;          // per element: bl (nbe) then il (ni), local dof indices
  int* bidx = nullptr;         // per element, aligned with loc: boundary index of bl[k]
  long long* off = nullptr;    // per element start in loc / bidx
  int *nbe = nullptr, *ni = nullptr;
  long long *woff = nullptr, *soff = nullptr, *voff = nullptr, *toff = nullptr;
  long long* addr_b = nullptr;  // [nb]
  double *G = nullptr, *wdet = nullptr, *Lg = nullptr, *Mr = nullptr;
  // work
  double *S = nullptr, *wk = nullptr, *Ke = nullptr, *Lw = nullptr, *Sch = nullptr, *V = nullptr, *T = nullptr;
  // CSR of the Schur complement (rows = boundary free indices, sorted columns)
  long long* rp = nullptr;
  int* ci = nullptr;
  double *vals = nullptr, *dg = nullptr;
  long long *aptr = nullptr, *asrc = nullptr;  // slot -> contributions (element order)
  long long *rptr = nullptr, *rsrc = nullptr;  // boundary dof -> reduce_rhs contributions
  // SGS level schedules
  int *frow = nullptr, *fptr = nullptr, *brow = nullptr, *bptr = nullptr;
  int nfl = 0, nbl = 0;
  // PCG vectors
  double *xb = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *ap = nullptr, *bsc = nullptr;
  double *part = nullptr, *dscal = nullptr, *hscal = nullptr;
  unsigned long long *dflag = nullptr, *hflag = nullptr;
  bool factored = false;
  std::vector<long long> h_rp;
  std::vector<int> h_ci;
};

namespace {

int serr(sdme_schur* s, int code, const std::string& msg, int64_t elem = -1) {
  if (s && s->ctx) {
    s->ctx->err_code = code;
    s->ctx->err_msg = msg;
    s->ctx->err_elem = elem;
    s->ctx->err_qp = -1;
  }
  return code;
}

#define SCK(call)                                                                           \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) return serr(s, SDME_CUDA_ERROR, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

inline int blocks_for(long long n, int t = 256) { return (int)std::max<long long>(1, std::min<long long>((n + t - 1) / t, 148LL * 8)); }

double* ctx_vec(sdme_ctx* c, int id) {
  if (!c || id < 0 || id >= (int)c->vecs.size()) return nullptr;
  return c->vecs[id];
}

int dot(sdme_schur* s, const double* a, const double* b, double* out) {
  cudaStream_t st = s->ctx->st;
  k_dot2<<<kRedGrid, kRed, 0, st>>>(a, b, s->nb, s->part);
  k_dot_finish<<<1, 32, 0, st>>>(s->part, s->dscal);
  SCK(cudaMemcpyAsync(s->hscal, s->dscal, sizeof(double), cudaMemcpyDeviceToHost, st));
  SCK(cudaStreamSynchronize(st));
  s->ctx->launches += 2;
  *out = *s->hscal;
  return SDME_OK;
}

int precond(sdme_schur* s, int kind, const double* rr, double* zz) {
  cudaStream_t st = s->ctx->st;
  if (kind == 2) {
    SCK(cudaMemsetAsync(zz, 0, s->nb * sizeof(double), st));
    k_sgs<<<1, kSolveThreads, 0, st>>>(s->rp, s->ci, s->vals, s->dg, s->frow, s->fptr, s->nfl, s->brow, s->bptr,
                                       s->nbl, rr, zz);
  } else {
    k_scale_copy<<<blocks_for(s->nb), 256, 0, st>>>(zz, kind == 1 ? s->dg : nullptr, rr, s->nb);
  }
  ++s->ctx->launches;
  return SDME_OK;
}

// level schedule of the lower (fwd) / upper (bwd) triangle of a CSR pattern
void levels(const std::vector<long long>& rp, const std::vector<int>& ci, long long n, bool fwd, std::vector<int>& rows,
            std::vector<int>& ptr) {
  std::vector<int> lv(n, 0);
  int maxl = 0;
  for (long long t = 0; t < n; ++t) {
    const long long i = fwd ? t : n - 1 - t;
    int l = 0;
    for (long long k = rp[i]; k < rp[i + 1]; ++k) {
      const long long j = ci[k];
      if ((fwd && j < i) || (!fwd && j > i)) l = std::max(l, lv[j] + 1);
    }
    lv[i] = l;
    maxl = std::max(maxl, l);
  }
  ptr.assign(maxl + 2, 0);
  for (long long i = 0; i < n; ++i) ++ptr[lv[i] + 1];
  for (int l = 0; l <= maxl; ++l) ptr[l + 1] += ptr[l];
  rows.assign(n, 0);
  std::vector<int> fill(ptr.begin(), ptr.end() - 1);
  for (long long i = 0; i < n; ++i) rows[fill[lv[i]]++] = (int)i;
}

}  // namespace

extern "C" {

int sdme_schur_create(sdme_ctx* ctx, const sdme_schur_desc* d, sdme_schur** out) {
  if (!ctx || !d || !out || d->n_elems < 1 || d->nd < 3 || d->nq < 1 || d->nb < 0) return SDME_BAD_ARGUMENT;
  auto* s = new sdme_schur();
  s->ctx = ctx;
  s->ne = d->n_elems, s->nd = d->nd, s->nf = d->nd / 3, s->nq = d->nq, s->nb = d->nb;
  s->mu = d->mu, s->lam = d->lambda_lame, s->rho = d->rho0;
  const long long ne = s->ne, nd = s->nd;
  // per-element boundary / interior local dof lists (ascending local order)
  std::vector<int> loc, bidx, nbe(ne), ni(ne);
  std::vector<long long> off(ne + 1, 0), woff(ne + 1, 0), soff(ne + 1, 0), voff(ne + 1, 0), toff(ne + 1, 0);
  for (long long e = 0; e < ne; ++e) {
    off[e] = (long long)loc.size();
    std::vector<int> il;
    for (int l = 0; l < nd; ++l) {
      const int r = d->role[e * nd + l];
      if (r >= 0) {
        if (r >= s->nb) {
          delete s;
          return SDME_BAD_ARGUMENT;
        }
        loc.push_back(l);
        bidx.push_back(r);
      } else if (r == -2) {
        il.push_back(l);
      }
    }
    nbe[e] = (int)(loc.size() - off[e]);
    ni[e] = (int)il.size();
    for (int l : il) {
      loc.push_back(l);
      bidx.push_back(-1);
    }
    woff[e + 1] = woff[e] + (long long)ni[e] * ni[e] + (long long)ni[e] * nbe[e];
    soff[e + 1] = soff[e] + (long long)nbe[e] * nbe[e];
    voff[e + 1] = voff[e] + nbe[e];
    toff[e + 1] = toff[e] + ni[e];
  }
  off[ne] = (long long)loc.size();
  // Schur CSR pattern and the per-slot contribution lists (element order)
  std::vector<std::vector<std::pair<int, long long>>> rows(s->nb);
  std::vector<std::vector<long long>> rcontrib(s->nb);
  for (long long e = 0; e < ne; ++e) {
    const int nb_e = nbe[e];
    for (int a = 0; a < nb_e; ++a) {
      const int ra = bidx[off[e] + a];
      rcontrib[ra].push_back(voff[e] + a);
      for (int b = 0; b < nb_e; ++b) rows[ra].push_back({bidx[off[e] + b], soff[e] + (long long)a * nb_e + b});
    }
  }
  std::vector<long long> rp(s->nb + 1, 0), aptr(1, 0), asrc, rptr(s->nb + 1, 0), rsrc;
  std::vector<int> ci;
  for (long long i = 0; i < s->nb; ++i) {
    auto& v = rows[i];
    std::stable_sort(v.begin(), v.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    for (size_t k = 0; k < v.size(); ++k) {
      if (k == 0 || v[k].first != v[k - 1].first) {
        ci.push_back(v[k].first);
        aptr.push_back(aptr.back());
      }
      asrc.push_back(v[k].second);
      ++aptr.back();
    }
    rp[i + 1] = (long long)ci.size();
    std::vector<std::pair<int, long long>>().swap(v);
    for (long long c : rcontrib[i]) rsrc.push_back(c);
    rptr[i + 1] = (long long)rsrc.size();
  }
  s->nnz = (long long)ci.size();
  std::vector<int> frow, fptr, brow, bptr;
  levels(rp, ci, s->nb, true, frow, fptr);
  levels(rp, ci, s->nb, false, brow, bptr);
  s->nfl = (int)fptr.size() - 1, s->nbl = (int)bptr.size() - 1;
  s->h_rp = rp;
  s->h_ci = ci;
  // tables
  std::vector<long long> addr(d->addr, d->addr + ne * nd), addr_b(d->addr_b, d->addr_b + s->nb);
  const int nf = s->nf, nq = s->nq;
  std::vector<double> G(d->G, d->G + (long long)nq * nf * 3), wdet(d->wdet, d->wdet + nq);
  std::vector<double> N(d->N, d->N + (long long)nq * nf), Lg((long long)nf * nf, 0.0), Mr((long long)nf * nf, 0.0);
  for (int f = 0; f < nf; ++f)
    for (int g = 0; g < nf; ++g) {
      double l = 0.0, m = 0.0;
      for (int q = 0; q < nq; ++q) {
        const double* gf = &G[((long long)q * nf + f) * 3];
        const double* gg = &G[((long long)q * nf + g) * 3];
        l += wdet[q] * (gf[0] * gg[0] + gf[1] * gg[1] + gf[2] * gg[2]);
        m += wdet[q] * N[(long long)q * nf + f] * N[(long long)q * nf + g];
      }
      Lg[(long long)f * nf + g] = l;
      Mr[(long long)f * nf + g] = m;
    }
  s->addr = dev_copy(addr);
  s->loc = dev_copy(loc);
  s->bidx = dev_copy(bidx);
  s->off = dev_copy(off);
  s->nbe = dev_copy(nbe);
  s->ni = dev_copy(ni);
  s->woff = dev_copy(woff);
  s->soff = dev_copy(soff);
  s->voff = dev_copy(voff);
  s->toff = dev_copy(toff);
  s->addr_b = dev_copy(addr_b);
  s->G = dev_copy(G);
  s->wdet = dev_copy(wdet);
  s->Lg = dev_copy(Lg);
  s->Mr = dev_copy(Mr);
  s->rp = dev_copy(rp);
  s->ci = dev_copy(ci);
  s->aptr = dev_copy(aptr);
  s->asrc = dev_copy(asrc);
  s->rptr = dev_copy(rptr);
  s->rsrc = dev_copy(rsrc);
  s->frow = dev_copy(frow);
  s->fptr = dev_copy(fptr);
  s->brow = dev_copy(brow);
  s->bptr = dev_copy(bptr);
  const long long nbv = std::max<long long>(1, s->nb);
  bool ok = cudaMalloc(&s->S, (size_t)ne * nq * nd * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->wk, (size_t)ne * nq * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->Ke, (size_t)ne * nd * nd * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->Lw, (size_t)std::max<long long>(1, woff[ne]) * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->Sch, (size_t)std::max<long long>(1, soff[ne]) * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->V, (size_t)std::max<long long>(1, voff[ne]) * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->T, (size_t)std::max<long long>(1, toff[ne]) * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->vals, (size_t)std::max<long long>(1, s->nnz) * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->dg, nbv * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->xb, nbv * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->r, nbv * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->z, nbv * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->p, nbv * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->ap, nbv * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->bsc, nbv * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->part, kRedGrid * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->dscal, 4 * sizeof(double)) == cudaSuccess &&
            cudaMallocHost(&s->hscal, 4 * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->dflag, sizeof(unsigned long long)) == cudaSuccess &&
            cudaMallocHost(&s->hflag, sizeof(unsigned long long)) == cudaSuccess;
  if (!ok || (s->nb > 0 && (!s->rp || !s->addr_b))) {
    cudaGetLastError();
    sdme_schur_destroy(s);
    return SDME_CUDA_ERROR;
  }
  *out = s;
  return SDME_OK;
}

int sdme_schur_destroy(sdme_schur* s) {
  if (!s) return SDME_OK;
  void* ptrs[] = {s->addr, s->loc,  s->bidx, s->off,   s->nbe,  s->ni,   s->woff,  s->soff,  s->voff, s->toff,
                  s->addr_b, s->G,  s->wdet, s->Lg,    s->Mr,   s->S,    s->wk,    s->Ke,    s->Lw,   s->Sch,
                  s->V,    s->T,    s->rp,   s->ci,    s->vals, s->dg,   s->aptr,  s->asrc,  s->rptr, s->rsrc,
                  s->frow, s->fptr, s->brow, s->bptr,  s->xb,   s->r,    s->z,     s->p,     s->ap,   s->bsc,
                  s->part, s->dscal, s->dflag};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (s->hscal) cudaFreeHost(s->hscal);
  if (s->hflag) cudaFreeHost(s->hflag);
  delete s;
  return SDME_OK;
}

int sdme_schur_info(const sdme_schur* s, int64_t* nb, int64_t* nnz, int* fwd_levels, int* bwd_levels) {
  if (!s) return SDME_BAD_ARGUMENT;
  if (nb) *nb = s->nb;
  if (nnz) *nnz = s->nnz;
  if (fwd_levels) *fwd_levels = s->nfl;
  if (bwd_levels) *bwd_levels = s->nbl;
  return SDME_OK;
}

int sdme_schur_factor(sdme_schur* s, int u, double c_k, double c_m) {
  if (!s) return SDME_BAD_ARGUMENT;
  sdme_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->st;
  const double* pu = nullptr;
  if (c_k != 0.0) {
    pu = ctx_vec(ctx, u);
    if (!pu) return serr(s, SDME_BAD_ARGUMENT, "schur factor: bad u vector");
  }
  s->factored = false;
  SCK(cudaMemsetAsync(s->dflag, 0xFF, sizeof(unsigned long long), st));
  if (c_k != 0.0) {
    const int thr = std::min(1024, ((s->nq + 31) / 32) * 32);
    k_point_state<<<(unsigned)s->ne, thr, s->nd * sizeof(double), st>>>(pu, s->addr, s->nd, s->nq, s->G, s->wdet,
                                                                         s->mu, s->lam, s->S, s->wk, s->dflag);
    ++ctx->launches;
    SCK(cudaMemcpyAsync(s->hflag, s->dflag, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    if (*s->hflag != kNone) {
      const unsigned long long f = *s->hflag;
      const int64_t e = (int64_t)(f / s->nq);
      const int q = (int)(f % s->nq);
      ctx->err_code = SDME_INVERSION;
      ctx->err_msg = "element " + std::to_string(e) + " inverted at quadrature point " + std::to_string(q);
      ctx->err_elem = e;
      ctx->err_qp = q;
      return SDME_INVERSION;
    }
  }
  const int tiles = (s->nf + kTF - 1) / kTF;
  k_elem_matrix<<<dim3(tiles, tiles, (unsigned)s->ne), dim3(kTF, kTF), 0, st>>>(
      s->S, s->wk, s->wdet, s->Lg, s->Mr, s->nf, s->nq, c_k, c_m, s->mu, s->lam, s->rho, s->Ke);
  k_condense<<<(unsigned)s->ne, kSolveThreads, 0, st>>>(s->Ke, s->nd, s->loc, s->off, s->nbe, s->ni, s->Lw, s->Lw,
                                                         s->Sch, s->woff, s->soff, s->dflag);
  ctx->launches += 2;
  SCK(cudaGetLastError());
  SCK(cudaMemcpyAsync(s->hflag, s->dflag, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  SCK(cudaStreamSynchronize(st));
  if (*s->hflag != kNone)
    return serr(s, SDME_BAD_ARGUMENT, "element interior block is not SPD", (int64_t)*s->hflag);
  if (s->nb > 0) {
    k_gather_sum<<<blocks_for(s->nnz), 256, 0, st>>>(s->aptr, s->asrc, s->Sch, s->vals, s->nnz);
    k_diag_of<<<blocks_for(s->nb), 256, 0, st>>>(s->rp, s->ci, s->vals, s->dg, s->nb, s->dflag);
    ctx->launches += 2;
  }
  SCK(cudaGetLastError());
  s->factored = true;
  return SDME_OK;
}

int sdme_schur_solve(sdme_schur* s, int b, int x, int prec, double tol, int maxit, int* iters, double* relres) {
  if (!s || !s->factored) return SDME_BAD_ARGUMENT;
  sdme_ctx* ctx = s->ctx;
  cudaStream_t st = ctx->st;
  const double* pb = ctx_vec(ctx, b);
  double* px = ctx_vec(ctx, x);
  if (!pb || !px || prec < 0 || prec > 2 || !(tol > 0.0 && tol < 1.0)) return serr(s, SDME_BAD_ARGUMENT, "schur solve: bad argument");
  if (iters) *iters = 0;
  if (relres) *relres = 0.0;
  if (prec >= 1) {
    SCK(cudaMemcpyAsync(s->hflag, s->dflag, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    SCK(cudaStreamSynchronize(st));
    if (*s->hflag != kNone)
      return serr(s, SDME_BAD_DIAGONAL, prec == 2 ? "Gauss-Seidel preconditioner needs positive diagonal entries"
                                                  : "diagonal preconditioner needs positive diagonal entries");
  }
  const long long nb = s->nb;
  // b_sc = reduce_rhs(b)
  if (nb > 0) {
    k_reduce_v<<<(unsigned)s->ne, 256, 0, st>>>(pb, s->addr, s->loc, s->off, s->nbe, s->ni, s->Lw, s->woff, s->V,
                                               s->voff, s->nd);
    k_reduce_rhs<<<blocks_for(nb), 256, 0, st>>>(pb, s->addr_b, s->rptr, s->rsrc, s->V, s->bsc, nb);
    ctx->launches += 2;
  }
  SCK(cudaMemsetAsync(s->xb, 0, std::max<long long>(1, nb) * sizeof(double), st));
  int it = 0;
  double rel = 0.0;
  int status = SDME_OK;
  double nrm_b2 = 0.0;
  if (nb > 0 && (status = dot(s, s->bsc, s->bsc, &nrm_b2))) return status;
  const double nrm_b = std::sqrt(nrm_b2);
  if (nb > 0 && nrm_b > 0.0) {
    // x0 = 0: r = b ; z = M r ; p = z ; rz = r.z   (solver.py:143-147)
    SCK(cudaMemcpyAsync(s->r, s->bsc, nb * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if ((status = precond(s, prec, s->r, s->z))) return status;
    SCK(cudaMemcpyAsync(s->p, s->z, nb * sizeof(double), cudaMemcpyDeviceToDevice, st));
    double rz = 0.0;
    if ((status = dot(s, s->r, s->z, &rz))) return status;
    const int spmv_grid = blocks_for(nb * 32, 256);
    bool done = false;
    for (it = 1; it <= maxit; ++it) {
      k_spmv<<<spmv_grid, 256, 0, st>>>(s->rp, s->ci, s->vals, s->p, s->ap, nb);
      ++ctx->launches;
      double pap = 0.0;
      if ((status = dot(s, s->p, s->ap, &pap))) return status;
      if (pap <= 0.0) {
        double rr = 0.0;
        if ((status = dot(s, s->r, s->r, &rr))) return status;
        rel = std::sqrt(rr) / nrm_b;
        char msg[160];
        snprintf(msg, sizeof msg, "indefinite operator detected at iteration %d (p^T A p = %.3e)", it, pap);
        if (iters) *iters = it;
        if (relres) *relres = rel;
        return serr(s, SDME_INDEFINITE, msg);
      }
      const double alpha = rz / pap;
      k_axpby<<<blocks_for(nb), 256, 0, st>>>(alpha, s->p, 1.0, s->xb, nb);
      k_axpby<<<blocks_for(nb), 256, 0, st>>>(-alpha, s->ap, 1.0, s->r, nb);
      ctx->launches += 2;
      double rr = 0.0;
      if ((status = dot(s, s->r, s->r, &rr))) return status;
      rel = std::sqrt(rr) / nrm_b;
      if (rel <= tol) {
        done = true;
        break;
      }
      if ((status = precond(s, prec, s->r, s->z))) return status;
      double rzn = 0.0;
      if ((status = dot(s, s->r, s->z, &rzn))) return status;
      k_axpby<<<blocks_for(nb), 256, 0, st>>>(1.0, s->z, rzn / rz, s->p, nb);
      ++ctx->launches;
      rz = rzn;
    }
    if (!done) {
      // true residual of the final iterate (solver.py:166-170)
      k_spmv<<<spmv_grid, 256, 0, st>>>(s->rp, s->ci, s->vals, s->xb, s->ap, nb);
      k_axpby<<<blocks_for(nb), 256, 0, st>>>(1.0, s->bsc, -1.0, s->ap, nb);
      ctx->launches += 2;
      double rr = 0.0;
      if ((status = dot(s, s->ap, s->ap, &rr))) return status;
      rel = std::sqrt(rr) / nrm_b;
      if (iters) *iters = maxit;
      if (relres) *relres = rel;
      char msg[160];
      snprintf(msg, sizeof msg, "PCG did not converge in %d iterations (relative residual %.3e)", maxit, rel);
      return serr(s, SDME_MAXIT, msg);
    }
  } else {
    it = 0;
  }
  // recover the full vector: x = 0 on Dirichlet points, boundary from x_b, interior per element
  SCK(cudaMemsetAsync(px, 0, ctx->nvec * sizeof(double), st));
  if (nb > 0) k_scatter_b<<<blocks_for(nb), 256, 0, st>>>(s->xb, s->addr_b, px, nb);
  k_recover<<<(unsigned)s->ne, 128, 0, st>>>(pb, s->xb, s->Ke, s->nd, s->addr, s->loc, s->off, s->nbe, s->ni, s->bidx,
                                             s->Lw, s->woff, s->T, s->toff, px);
  ctx->launches += 2;
  SCK(cudaGetLastError());
  SCK(cudaStreamSynchronize(st));
  if (iters) *iters = it;
  if (relres) *relres = rel;
  return SDME_OK;
}

int sdme_schur_matrix(const sdme_schur* s, int64_t* rowptr, int32_t* cols, double* vals, double* element_matrix0) {
  if (!s || !s->factored) return SDME_BAD_ARGUMENT;
  if (rowptr) std::copy(s->h_rp.begin(), s->h_rp.end(), rowptr);
  if (cols) std::copy(s->h_ci.begin(), s->h_ci.end(), cols);
  if (vals && s->nnz) cudaMemcpy(vals, s->vals, s->nnz * sizeof(double), cudaMemcpyDeviceToHost);
  if (element_matrix0) cudaMemcpy(element_matrix0, s->Ke, (size_t)s->nd * s->nd * sizeof(double), cudaMemcpyDeviceToHost);
  return cudaGetLastError() == cudaSuccess ? SDME_OK : SDME_CUDA_ERROR;
}

}  // extern "C"
