// Sum-factorised FP64 element kernels for order-P hexahedra (sm_100a).
//
// Replaces the dense per-element path of the reference
//   femcore.py:87-106  deformation_state / element_internal_force   (K1 fint)
//   femcore.py:116-146 _b_matrix / element_tangent, consumer a@p     (K2 apply)
//   femcore.py:149-156 element_mass, mass_full @ a_trial             (K3 mass)
//   solver.py:105-110  diagonal of the assembled effective operator  (K4 diag)
// by O(n^4) tensor contractions plus O(m^3) point work, matrix-free.
//
// Data layout: every global vector is a lattice of
// Lx*Ly*Lz points per displacement component, component-major, x fastest.
// Element (i,j,k) owns the (P+1)^3 box starting at (P*i, P*j, P*k).  The 1D
// tables arrive permuted to *lattice-local* order (column l = lattice offset l),
// so an element gather is a strided box with no index table.
//
// Assembly is deterministic: elements are processed in 8 colour passes (parity
// of i, j, k); elements of one colour share no lattice point, so each pass does
// a plain read-modify-write and the summation order at every point is fixed by
// the colour order.  No floating-point atomics anywhere.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sdme {

template <int N, int M>
struct Tab {
  double B[M][N];  // value of lattice-local function l at 1D point a
  double D[M][N];  // derivative d/dxi
  double W[M];     // 1D weights
};

struct Geo {
  int nx, ny, nz;     // elements per axis
  int Lx, Ly, Lz;     // lattice points per axis (P*n+1)
  long long Ns;       // points per component plane
  double s[3];        // dxi/dX = 2/h per axis
  double detJ;        // h_x h_y h_z / 8
  double mu, lam, rho;
  int dmask[3];       // Dirichlet face bits per component (xmin,xmax,ymin,ymax,zmin,zmax)
};

// MODE_SETUP stores K = F^-T and ln J at every quadrature point (OpArgs::qpd);
// MODE_PA is K.p from those stored values (the PCG operator: u is fixed
// during a solve, so the u pass and the point inverse/log are done once).
enum Mode { MODE_FINT = 0, MODE_APPLY = 1, MODE_MASS = 2, MODE_PA = 3, MODE_SETUP = 4 };
constexpr int kQpSlots = 10;  // K (9) + ln J per point, [elem][slot][q]

struct OpArgs {
  const double* u;    // linearisation point (FINT, APPLY, DIAG)
  const double* p;    // direction (APPLY) or field (MASS)
  double* y;          // accumulated output (RMW per colour pass)
  double c_k, c_m;    // y += c_k K p + c_m M p   (APPLY); y += c_m M p (MASS)
  int colour;         // bit0: i parity, bit1: j parity, bit2: k parity
  unsigned long long* inv_flag;  // atomicMin(elem*nq + qp) on det F <= 0
  const int* skip = nullptr;     // if set and non-zero: return at once (stopped PCG graph)
  double* ev = nullptr;          // E-vector mode (colour < 0): element boxes stored, not scattered
  double* qpd = nullptr;         // quadrature data (MODE_SETUP writes, MODE_PA reads)
};

__device__ __forceinline__ bool constrained(const Geo& g, int comp, int X, int Y, int Z) {
  const int m = g.dmask[comp];
  return ((m & 1) && X == 0) || ((m & 2) && X == g.Lx - 1) || ((m & 4) && Y == 0) ||
         ((m & 8) && Y == g.Ly - 1) || ((m & 16) && Z == 0) || ((m & 32) && Z == g.Lz - 1);
}

// True when the element box starting at (X0, Y0, Z0) with N points per edge
// touches a Dirichlet plane of component comp (warp-uniform fast path).
__device__ __forceinline__ bool touches_dirichlet(const Geo& g, int comp, int X0, int Y0, int Z0, int N) {
  const int m = g.dmask[comp];
  if (!m) return false;
  return ((m & 1) && X0 == 0) || ((m & 2) && X0 + N - 1 == g.Lx - 1) || ((m & 4) && Y0 == 0) ||
         ((m & 8) && Y0 + N - 1 == g.Ly - 1) || ((m & 16) && Z0 == 0) || ((m & 32) && Z0 + N - 1 == g.Lz - 1);
}

// Element of this block slot, for the given colour pass.  Returns false past the end.
// colour >= 0: the elements of one parity class (8-colour passes);
// colour < 0: every element in lexicographic order (E-vector mode).
__device__ __forceinline__ bool colour_element(const Geo& g, int colour, long long idx,
                                               int& ei, int& ej, int& ek) {
  if (colour < 0) {
    if (idx >= (long long)g.nx * g.ny * g.nz) return false;
    ei = (int)(idx % g.nx);
    const long long r = idx / g.nx;
    ej = (int)(r % g.ny);
    ek = (int)(r / g.ny);
    return true;
  }
  const int cx = colour & 1, cy = (colour >> 1) & 1, cz = (colour >> 2) & 1;
  const int nex = (g.nx - cx + 1) >> 1, ney = (g.ny - cy + 1) >> 1, nez = (g.nz - cz + 1) >> 1;
  if (nex <= 0 || ney <= 0 || nez <= 0) return false;
  if (idx >= (long long)nex * ney * nez) return false;
  const int ix = (int)(idx % nex);
  const long long r = idx / nex;
  const int iy = (int)(r % ney);
  const int iz = (int)(r / ney);
  ei = 2 * ix + cx;
  ej = 2 * iy + cy;
  ek = 2 * iz + cz;
  return true;
}

__host__ __device__ inline long long colour_count(const Geo& g, int colour) {
  if (colour < 0) return (long long)g.nx * g.ny * g.nz;
  const int cx = colour & 1, cy = (colour >> 1) & 1, cz = (colour >> 2) & 1;
  const long long nex = (g.nx - cx + 1) >> 1, ney = (g.ny - cy + 1) >> 1, nez = (g.nz - cz + 1) >> 1;
  if (nex <= 0 || ney <= 0 || nez <= 0) return 0;
  return nex * ney * nez;
}

// ---------------------------------------------------------------------------
// Per-qp constitutive work (neo-Hookean, material.py:65-105).

struct QpState {
  double F[3][3];
  double Ci[3][3];
  double S[3][3];
  double lnJ;
  double detF;
};

__device__ __forceinline__ void qp_state(const double H[3][3], double mu, double lam, QpState& st) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) st.F[i][j] = H[i][j] + (i == j ? 1.0 : 0.0);
  const double(&F)[3][3] = st.F;
  st.detF = F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) -
            F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
            F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
  // C = F^T F (symmetric)
  double C00 = F[0][0] * F[0][0] + F[1][0] * F[1][0] + F[2][0] * F[2][0];
  double C11 = F[0][1] * F[0][1] + F[1][1] * F[1][1] + F[2][1] * F[2][1];
  double C22 = F[0][2] * F[0][2] + F[1][2] * F[1][2] + F[2][2] * F[2][2];
  double C01 = F[0][0] * F[0][1] + F[1][0] * F[1][1] + F[2][0] * F[2][1];
  double C12 = F[0][1] * F[0][2] + F[1][1] * F[1][2] + F[2][1] * F[2][2];
  double C02 = F[0][0] * F[0][2] + F[1][0] * F[1][2] + F[2][0] * F[2][2];
  // adjugate / det
  double A00 = C11 * C22 - C12 * C12;
  double A01 = C02 * C12 - C01 * C22;
  double A02 = C01 * C12 - C02 * C11;
  double A11 = C00 * C22 - C02 * C02;
  double A12 = C01 * C02 - C00 * C12;
  double A22 = C00 * C11 - C01 * C01;
  double detC = C00 * A00 + C01 * A01 + C02 * A02;
  double inv = 1.0 / detC;
  st.Ci[0][0] = A00 * inv; st.Ci[1][1] = A11 * inv; st.Ci[2][2] = A22 * inv;
  st.Ci[0][1] = st.Ci[1][0] = A01 * inv;
  st.Ci[1][2] = st.Ci[2][1] = A12 * inv;
  st.Ci[0][2] = st.Ci[2][0] = A02 * inv;
  st.lnJ = 0.5 * log(detC);
  const double a = lam * st.lnJ - mu;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) st.S[i][j] = a * st.Ci[i][j] + (i == j ? mu : 0.0);
}

// dP = H_p S + F dS,  dS = lam (Ci:dE) Ci + 2 (mu - lam lnJ) Ci dE Ci,  dE = sym(F^T H_p)
// (matrix-free form of B^T D B + geometric term).
__device__ __forceinline__ void qp_dP(const QpState& st, const double Hp[3][3], double mu, double lam,
                                      double dP[3][3]) {
  double A[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      A[i][j] = st.F[0][i] * Hp[0][j] + st.F[1][i] * Hp[1][j] + st.F[2][i] * Hp[2][j];
  double E[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) E[i][j] = 0.5 * (A[i][j] + A[j][i]);
  double tr = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) tr += st.Ci[i][j] * E[i][j];
  double T1[3][3];  // Ci E
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      T1[i][j] = st.Ci[i][0] * E[0][j] + st.Ci[i][1] * E[1][j] + st.Ci[i][2] * E[2][j];
  const double c2 = 2.0 * (mu - lam * st.lnJ);
  const double c1 = lam * tr;
  double dS[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      dS[i][j] = c1 * st.Ci[i][j] +
                 c2 * (T1[i][0] * st.Ci[0][j] + T1[i][1] * st.Ci[1][j] + T1[i][2] * st.Ci[2][j]);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      dP[i][j] = Hp[i][0] * st.S[0][j] + Hp[i][1] * st.S[1][j] + Hp[i][2] * st.S[2][j] +
                 st.F[i][0] * dS[0][j] + st.F[i][1] * dS[1][j] + st.F[i][2] * dS[2][j];
}

// ---------------------------------------------------------------------------
// Shared-memory layout per element slot (doubles):
//   sX0, sX1 : n*n*m   (after x contraction: [k][j][a])
//   sY0..sY2 : n*m*m   (after y contraction: [k][b][a])
//   sGu      : 9*m^3   grad u   [comp][d][c][b][a]
//   sGp      : 12*m^3  grad p (+ value) [comp][d(0..3)][c][b][a]; reused as flux
template <int N, int M>
struct Smem {
  static constexpr int X = N * N * M;
  static constexpr int Y = N * M * M;
  static constexpr int Q = M * M * M;
  static constexpr int kX0 = 0, kX1 = X, kY0 = 2 * X, kY1 = 2 * X + Y, kY2 = 2 * X + 2 * Y;
  static constexpr int kGu = 2 * X + 3 * Y;
  static constexpr int kGp = kGu + 9 * Q;
  static constexpr int per_elem = kGp + 12 * Q;
};

// Forward: one scalar field (one component) from the global lattice to point
// values and/or reference gradients.  WANT_GRAD: gx,gy,gz; WANT_VAL: value.
// Output written to dst[d][c][b][a] for d in {0,1,2} (grad, scaled by s_d) and
// dst[3] (value) when requested.
template <int N, int M, bool WANT_GRAD, bool WANT_VAL, int EB>
__device__ __forceinline__ void forward_field(const Tab<N, M>& tb, const Geo& g, double* sm,
                                              const double* __restrict__ src, const int (*base)[3],
                                              const bool* valid, double* const* dst) {
  using L = Smem<N, M>;
  const int tid = threadIdx.x, nt = blockDim.x;
  // stage X: pencils (k, j) along x from global memory
  for (int w = tid; w < EB * N * N; w += nt) {
    const int el = w / (N * N), it = w % (N * N);
    const int k = it / N, j = it % N;
    double* s = sm + el * L::per_elem;
    double v[N];
    if (valid[el]) {
      const double* row = src + ((long long)(base[el][2] + k) * g.Ly + (base[el][1] + j)) * g.Lx + base[el][0];
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = __ldg(row + i);
    } else {
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = 0.0;
    }
#pragma unroll
    for (int a = 0; a < M; ++a) {
      double b0 = 0.0, b1 = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        b0 = fma(tb.B[a][i], v[i], b0);
        if (WANT_GRAD) b1 = fma(tb.D[a][i], v[i], b1);
      }
      s[L::kX0 + it * M + a] = b0;
      if (WANT_GRAD) s[L::kX1 + it * M + a] = b1;
    }
  }
  __syncthreads();
  // stage Y: pencils (k, a) along y
  for (int w = tid; w < EB * N * M; w += nt) {
    const int el = w / (N * M), it = w % (N * M);
    const int k = it / M, a = it % M;
    double* s = sm + el * L::per_elem;
    double x0[N], x1[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      x0[j] = s[L::kX0 + (k * N + j) * M + a];
      if (WANT_GRAD) x1[j] = s[L::kX1 + (k * N + j) * M + a];
    }
#pragma unroll
    for (int b = 0; b < M; ++b) {
      double bb = 0.0, db = 0.0, bd = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        bb = fma(tb.B[b][j], x0[j], bb);
        if (WANT_GRAD) {
          db = fma(tb.D[b][j], x0[j], db);
          bd = fma(tb.B[b][j], x1[j], bd);
        }
      }
      const int o = (k * M + b) * M + a;
      s[L::kY0 + o] = bb;   // B_y B_x
      if (WANT_GRAD) {
        s[L::kY1 + o] = db;  // D_y B_x
        s[L::kY2 + o] = bd;  // B_y D_x
      }
    }
  }
  __syncthreads();
  // stage Z: pencils (b, a) along z -> point values
  for (int w = tid; w < EB * M * M; w += nt) {
    const int el = w / (M * M), it = w % (M * M);
    double* s = sm + el * L::per_elem;
    double y0[N], y1[N], y2[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      y0[k] = s[L::kY0 + k * M * M + it];
      if (WANT_GRAD) {
        y1[k] = s[L::kY1 + k * M * M + it];
        y2[k] = s[L::kY2 + k * M * M + it];
      }
    }
    double* o = dst[el];
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double gx = 0.0, gy = 0.0, gz = 0.0, vv = 0.0;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        if (WANT_GRAD) {
          gx = fma(tb.B[c][k], y2[k], gx);
          gy = fma(tb.B[c][k], y1[k], gy);
          gz = fma(tb.D[c][k], y0[k], gz);
        }
        if (WANT_VAL) vv = fma(tb.B[c][k], y0[k], vv);
      }
      const int q = c * M * M + it;
      if (WANT_GRAD) {
        o[0 * L::Q + q] = gx * g.s[0];
        o[1 * L::Q + q] = gy * g.s[1];
        o[2 * L::Q + q] = gz * g.s[2];
      }
      if (WANT_VAL) o[3 * L::Q + q] = vv;
    }
  }
  __syncthreads();
}

// Backward: fluxes at points -> element vector of one component, then
// masked read-modify-write into the global lattice (colour pass).
//   y_l = sum_q [ Dx By Bz Qx + Bx Dy Bz Qy + Bx By Dz Qz + Bx By Bz V ]
template <int N, int M, bool HAS_GRAD, bool HAS_VAL, int EB>
__device__ __forceinline__ void backward_field(const Tab<N, M>& tb, const Geo& g, double* sm,
                                               double* const* flux, double* __restrict__ dstv,
                                               int comp, const int (*base)[3], const bool* valid) {
  using L = Smem<N, M>;
  const int tid = threadIdx.x, nt = blockDim.x;
  // stage Z': pencils (b, a), contract over c
  for (int w = tid; w < EB * M * M; w += nt) {
    const int el = w / (M * M), it = w % (M * M);
    double* s = sm + el * L::per_elem;
    const double* f = flux[el];
    double qx[M], qy[M], qz[M], qv[M];
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const int q = c * M * M + it;
      if (HAS_GRAD) {
        qx[c] = f[0 * L::Q + q];
        qy[c] = f[1 * L::Q + q];
        qz[c] = f[2 * L::Q + q];
      }
      if (HAS_VAL) qv[c] = f[3 * L::Q + q];
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double hx = 0.0, hy = 0.0, hz = 0.0;
#pragma unroll
      for (int c = 0; c < M; ++c) {
        if (HAS_GRAD) {
          hx = fma(tb.B[c][k], qx[c], hx);
          hy = fma(tb.B[c][k], qy[c], hy);
          hz = fma(tb.D[c][k], qz[c], hz);
        }
        if (HAS_VAL) hz = fma(tb.B[c][k], qv[c], hz);
      }
      const int o = k * M * M + it;
      if (HAS_GRAD) {
        s[L::kY0 + o] = hx;
        s[L::kY1 + o] = hy;
      }
      s[L::kY2 + o] = hz;
    }
  }
  __syncthreads();
  // stage Y': pencils (k, a), contract over b
  for (int w = tid; w < EB * N * M; w += nt) {
    const int el = w / (N * M), it = w % (N * M);
    const int k = it / M, a = it % M;
    double* s = sm + el * L::per_elem;
    double hx[M], hy[M], hz[M];
#pragma unroll
    for (int b = 0; b < M; ++b) {
      const int o = (k * M + b) * M + a;
      if (HAS_GRAD) {
        hx[b] = s[L::kY0 + o];
        hy[b] = s[L::kY1 + o];
      }
      hz[b] = s[L::kY2 + o];
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double jx = 0.0, jyz = 0.0;
#pragma unroll
      for (int b = 0; b < M; ++b) {
        if (HAS_GRAD) {
          jx = fma(tb.B[b][j], hx[b], jx);
          jyz = fma(tb.D[b][j], hy[b], jyz);
        }
        jyz = fma(tb.B[b][j], hz[b], jyz);
      }
      const int o = (k * N + j) * M + a;
      if (HAS_GRAD) s[L::kX0 + o] = jx;
      s[L::kX1 + o] = jyz;
    }
  }
  __syncthreads();
  // stage X': pencils (k, j), contract over a, scatter along x
  for (int w = tid; w < EB * N * N; w += nt) {
    const int el = w / (N * N), it = w % (N * N);
    const int k = it / N, j = it % N;
    if (!valid[el]) continue;
    double* s = sm + el * L::per_elem;
    double jx[M], jyz[M];
#pragma unroll
    for (int a = 0; a < M; ++a) {
      if (HAS_GRAD) jx[a] = s[L::kX0 + it * M + a];
      jyz[a] = s[L::kX1 + it * M + a];
    }
    const int Z = base[el][2] + k, Y = base[el][1] + j;
    double* row = dstv + ((long long)Z * g.Ly + Y) * g.Lx + base[el][0];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < M; ++a) {
        if (HAS_GRAD) acc = fma(tb.D[a][i], jx[a], acc);
        acc = fma(tb.B[a][i], jyz[a], acc);
      }
      if (!constrained(g, comp, base[el][0] + i, Y, Z)) row[i] += acc;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// K1 / K2 / K3: one colour pass of f_int, (c_k K + c_m M) p, or c_m M p.
template <int N, int M, int EB, int MODE>
__global__ void __launch_bounds__(128) element_op(const __grid_constant__ Tab<N, M> tb,
                                                  const __grid_constant__ Geo g, OpArgs args) {
  using L = Smem<N, M>;
  extern __shared__ double smem[];
  __shared__ int base[EB][3];
  __shared__ bool valid[EB];
  __shared__ long long eid[EB];
  if (threadIdx.x < EB) {
    int ei = 0, ej = 0, ek = 0;
    const long long idx = (long long)blockIdx.x * EB + threadIdx.x;
    const bool ok = colour_element(g, args.colour, idx, ei, ej, ek);
    valid[threadIdx.x] = ok;
    base[threadIdx.x][0] = (N - 1) * ei;
    base[threadIdx.x][1] = (N - 1) * ej;
    base[threadIdx.x][2] = (N - 1) * ek;
    eid[threadIdx.x] = ((long long)ek * g.ny + ej) * g.nx + ei;
  }
  __syncthreads();

  double* gu[EB];
  double* gp[EB];
#pragma unroll
  for (int e = 0; e < EB; ++e) {
    gu[e] = smem + e * L::per_elem + L::kGu;
    gp[e] = smem + e * L::per_elem + L::kGp;
  }

  if (MODE == MODE_FINT || MODE == MODE_APPLY) {
#pragma unroll 1
    for (int comp = 0; comp < 3; ++comp) {
      double* dst[EB];
#pragma unroll
      for (int e = 0; e < EB; ++e) dst[e] = gu[e] + comp * 3 * L::Q;
      forward_field<N, M, true, false, EB>(tb, g, smem, args.u + comp * g.Ns, base, valid, dst);
    }
  }
  if (MODE == MODE_APPLY || MODE == MODE_MASS) {
    const bool want_val = (args.c_m != 0.0);
#pragma unroll 1
    for (int comp = 0; comp < 3; ++comp) {
      double* dst[EB];
#pragma unroll
      for (int e = 0; e < EB; ++e) dst[e] = gp[e] + comp * 4 * L::Q;
      if (MODE == MODE_MASS)
        forward_field<N, M, false, true, EB>(tb, g, smem, args.p + comp * g.Ns, base, valid, dst);
      else if (want_val)
        forward_field<N, M, true, true, EB>(tb, g, smem, args.p + comp * g.Ns, base, valid, dst);
      else
        forward_field<N, M, true, false, EB>(tb, g, smem, args.p + comp * g.Ns, base, valid, dst);
    }
  }

  // point work
  for (int w = threadIdx.x; w < EB * L::Q; w += blockDim.x) {
    const int el = w / L::Q, q = w % L::Q;
    const int a = q % M, b = (q / M) % M, c = q / (M * M);
    const double wq = tb.W[a] * tb.W[b] * tb.W[c] * g.detJ;
    double* fu = gu[el];
    double* fp = gp[el];
    if (MODE == MODE_MASS) {
      const double sc = args.c_m * g.rho * wq;
#pragma unroll
      for (int i = 0; i < 3; ++i) fp[(i * 4 + 3) * L::Q + q] *= sc;
      continue;
    }
    double H[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int d = 0; d < 3; ++d) H[i][d] = fu[(i * 3 + d) * L::Q + q];
    QpState st;
    qp_state(H, g.mu, g.lam, st);
    if (st.detF <= 0.0 && valid[el]) {
      const unsigned long long key =
          (unsigned long long)eid[el] * L::Q + (unsigned long long)((a * M + b) * M + c);
      atomicMin(args.inv_flag, key);
    }
    if (MODE == MODE_FINT) {
      // P1 = F S ; flux Q[i][d] = wq * s_d * P1[i][d]   (written into gp slots)
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double p1 = st.F[i][0] * st.S[0][d] + st.F[i][1] * st.S[1][d] + st.F[i][2] * st.S[2][d];
          fp[(i * 4 + d) * L::Q + q] = wq * g.s[d] * p1;
        }
    } else {
      double Hp[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int d = 0; d < 3; ++d) Hp[i][d] = fp[(i * 4 + d) * L::Q + q];
      double dP[3][3];
      qp_dP(st, Hp, g.mu, g.lam, dP);
      const double sk = args.c_k * wq;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int d = 0; d < 3; ++d) fp[(i * 4 + d) * L::Q + q] = sk * g.s[d] * dP[i][d];
      if (args.c_m != 0.0) {
        const double sc = args.c_m * g.rho * wq;
#pragma unroll
        for (int i = 0; i < 3; ++i) fp[(i * 4 + 3) * L::Q + q] *= sc;
      }
    }
  }
  __syncthreads();

#pragma unroll 1
  for (int comp = 0; comp < 3; ++comp) {
    double* fl[EB];
#pragma unroll
    for (int e = 0; e < EB; ++e) fl[e] = gp[e] + comp * 4 * L::Q;
    if (MODE == MODE_FINT)
      backward_field<N, M, true, false, EB>(tb, g, smem, fl, args.y + comp * g.Ns, comp, base, valid);
    else if (MODE == MODE_MASS)
      backward_field<N, M, false, true, EB>(tb, g, smem, fl, args.y + comp * g.Ns, comp, base, valid);
    else if (args.c_m != 0.0)
      backward_field<N, M, true, true, EB>(tb, g, smem, fl, args.y + comp * g.Ns, comp, base, valid);
    else
      backward_field<N, M, true, false, EB>(tb, g, smem, fl, args.y + comp * g.Ns, comp, base, valid);
  }
}

// ---------------------------------------------------------------------------
// K4: diagonal of c_k K_T(u) + c_m M (closed form):
//   diag[f,c] = sum_q w sum_{d,e} g_fd g_fe (A^c_de + S_de) + c_m rho sum_q w N_f^2
//   A^c_de = sum_{i,k} F_ci F_ck DD_idke,
//   DD_ijkl = lam Ci_ij Ci_kl + (mu - lam lnJ)(Ci_ik Ci_jl + Ci_il Ci_jk).
// For axis-aligned elements g_fd g_fe factorises into products of the 1D
// tables B^2, B D, D^2, so each of the 6 symmetric (d,e) pairs plus the mass
// term is one backward contraction with "squared" tables.
template <int N, int M, int EB>
__global__ void __launch_bounds__(128) element_diag(const __grid_constant__ Tab<N, M> tb,
                                                    const __grid_constant__ Geo g, OpArgs args) {
  using L = Smem<N, M>;
  extern __shared__ double smem[];
  __shared__ int base[EB][3];
  __shared__ bool valid[EB];
  __shared__ long long eid[EB];
  if (threadIdx.x < EB) {
    int ei = 0, ej = 0, ek = 0;
    const long long idx = (long long)blockIdx.x * EB + threadIdx.x;
    const bool ok = colour_element(g, args.colour, idx, ei, ej, ek);
    valid[threadIdx.x] = ok;
    base[threadIdx.x][0] = (N - 1) * ei;
    base[threadIdx.x][1] = (N - 1) * ej;
    base[threadIdx.x][2] = (N - 1) * ek;
    eid[threadIdx.x] = ((long long)ek * g.ny + ej) * g.nx + ei;
  }
  __syncthreads();
  double* gu[EB];
  double* gp[EB];
#pragma unroll
  for (int e = 0; e < EB; ++e) {
    gu[e] = smem + e * L::per_elem + L::kGu;
    gp[e] = smem + e * L::per_elem + L::kGp;
  }
  if (args.c_k != 0.0) {
#pragma unroll 1
    for (int comp = 0; comp < 3; ++comp) {
      double* dst[EB];
#pragma unroll
      for (int e = 0; e < EB; ++e) dst[e] = gu[e] + comp * 3 * L::Q;
      forward_field<N, M, true, false, EB>(tb, g, smem, args.u + comp * g.Ns, base, valid, dst);
    }
  }
  // point coefficients: per comp c, 6 pairs (d<=e) + mass -> gp[c*... ] is 12*Q;
  // we need 3*6 + 1 = 19 Q-arrays: use gu (9Q, reused after reading) + gp (12Q).
  for (int w = threadIdx.x; w < EB * L::Q; w += blockDim.x) {
    const int el = w / L::Q, q = w % L::Q;
    const int a = q % M, b = (q / M) % M, c = q / (M * M);
    const double wq = tb.W[a] * tb.W[b] * tb.W[c] * g.detJ;
    double* fu = gu[el];
    double* fp = gp[el];
    double coef[3][6];
    if (args.c_k != 0.0) {
      double H[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int d = 0; d < 3; ++d) H[i][d] = fu[(i * 3 + d) * L::Q + q];
      QpState st;
      qp_state(H, g.mu, g.lam, st);
      if (st.detF <= 0.0 && valid[el]) {
        const unsigned long long key =
            (unsigned long long)eid[el] * L::Q + (unsigned long long)((a * M + b) * M + c);
        atomicMin(args.inv_flag, key);
      }
      const double cc = g.mu - g.lam * st.lnJ;
      // G_c[i][d] = sum_k F_ck Ci_... : A^c_de = lam (F Ci)_cd (F Ci)_ce + cc[(F Ci F^T)_cc Ci_de + (F Ci)_ce (F Ci)_cd]
      double FC[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int d = 0; d < 3; ++d)
          FC[i][d] = st.F[i][0] * st.Ci[0][d] + st.F[i][1] * st.Ci[1][d] + st.F[i][2] * st.Ci[2][d];
      const int pd[6] = {0, 1, 2, 0, 1, 0};
      const int pe[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double fcf = FC[i][0] * st.F[i][0] + FC[i][1] * st.F[i][1] + FC[i][2] * st.F[i][2];
#pragma unroll
        for (int t = 0; t < 6; ++t) {
          const int d = pd[t], e = pe[t];
          const double A = g.lam * FC[i][d] * FC[i][e] + cc * (fcf * st.Ci[d][e] + FC[i][e] * FC[i][d]);
          const double mult = (d == e) ? 1.0 : 2.0;
          coef[i][t] = args.c_k * mult * wq * g.s[d] * g.s[e] * (A + st.S[d][e]);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int t = 0; t < 6; ++t) coef[i][t] = 0.0;
    }
    // layout: slots 0..17 = coef[i][t] -> slot i*6+t ; slot 18 = mass
    // slots 0..8 in gu (9Q), 9..18 in gp (10 of 12Q)
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int t = 0; t < 6; ++t) {
        const int sl = i * 6 + t;
        double* dstp = sl < 9 ? fu + sl * L::Q : fp + (sl - 9) * L::Q;
        dstp[q] = coef[i][t];
      }
    fp[9 * L::Q + q] = args.c_m * g.rho * wq;
  }
  __syncthreads();
  // NOTE: the point loop above reads fu[q] for all 9 gradient entries before
  // any thread overwrites them only at the same q, so in-place reuse is safe.

  // backward with squared tables: out[k][j][i] = sum Tz[c][k] Ty[b][j] Tx[a][i] Q
  // table id: 0 = B^2, 1 = B D, 2 = D^2.
  const int pd[6] = {0, 1, 2, 0, 1, 0};
  const int pe[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll 1
  for (int comp = 0; comp < 3; ++comp) {
    // 7 terms per component (6 symmetric (d,e) pairs + mass); each is one
    // backward contraction chain, summed in smem (sX1) before the scatter.
#pragma unroll 1
    for (int term = 0; term < 7; ++term) {
      // tables per axis: number of derivative factors along that axis
      int tx = 0, ty = 0, tz = 0;
      if (term < 6) {
        const int d = pd[term], e = pe[term];
        tx = (d == 0) + (e == 0);
        ty = (d == 1) + (e == 1);
        tz = (d == 2) + (e == 2);
      }
      // Stage Z': (b,a) pencils over c -> sY0[k][b][a]
      for (int w = threadIdx.x; w < EB * M * M; w += blockDim.x) {
        const int el = w / (M * M), it = w % (M * M);
        double* s = smem + el * L::per_elem;
        const int sl = term < 6 ? comp * 6 + term : 18;
        const double* f = sl < 9 ? gu[el] + sl * L::Q : gp[el] + (sl - 9) * L::Q;
        double qv[M];
#pragma unroll
        for (int c = 0; c < M; ++c) qv[c] = f[c * M * M + it];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double h = 0.0;
#pragma unroll
          for (int c = 0; c < M; ++c) {
            const double t = tz == 0 ? tb.B[c][k] * tb.B[c][k]
                           : (tz == 1 ? tb.B[c][k] * tb.D[c][k] : tb.D[c][k] * tb.D[c][k]);
            h = fma(t, qv[c], h);
          }
          s[L::kY0 + k * M * M + it] = h;
        }
      }
      __syncthreads();
      // Stage Y': (k,a) pencils over b -> sX0[k][j][a]
      for (int w = threadIdx.x; w < EB * N * M; w += blockDim.x) {
        const int el = w / (N * M), it = w % (N * M);
        const int k = it / M, a = it % M;
        double* s = smem + el * L::per_elem;
        double hv[M];
#pragma unroll
        for (int b = 0; b < M; ++b) hv[b] = s[L::kY0 + (k * M + b) * M + a];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double acc = 0.0;
#pragma unroll
          for (int b = 0; b < M; ++b) {
            const double t = ty == 0 ? tb.B[b][j] * tb.B[b][j]
                           : (ty == 1 ? tb.B[b][j] * tb.D[b][j] : tb.D[b][j] * tb.D[b][j]);
            acc = fma(t, hv[b], acc);
          }
          s[L::kX0 + (k * N + j) * M + a] = acc;
        }
      }
      __syncthreads();
      // Stage X': (k,j) pencils over a -> accumulate into sX1[k][j][i] (n^3 <= n*n*m)
      for (int w = threadIdx.x; w < EB * N * N; w += blockDim.x) {
        const int el = w / (N * N), it = w % (N * N);
        double* s = smem + el * L::per_elem;
        double jv[M];
#pragma unroll
        for (int a = 0; a < M; ++a) jv[a] = s[L::kX0 + it * M + a];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int a = 0; a < M; ++a) {
            const double t = tx == 0 ? tb.B[a][i] * tb.B[a][i]
                           : (tx == 1 ? tb.B[a][i] * tb.D[a][i] : tb.D[a][i] * tb.D[a][i]);
            acc = fma(t, jv[a], acc);
          }
          double* accp = s + L::kX1 + it * N + i;
          *accp = (term == 0 ? 0.0 : *accp) + acc;
        }
      }
      __syncthreads();
    }
    // scatter this component
    for (int w = threadIdx.x; w < EB * N * N; w += blockDim.x) {
      const int el = w / (N * N), it = w % (N * N);
      if (!valid[el]) continue;
      const int k = it / N, j = it % N;
      double* s = smem + el * L::per_elem;
      const int Z = base[el][2] + k, Y = base[el][1] + j;
      if (args.ev) {
        double* er = args.ev + (eid[el] * 3 + comp) * (N * N * N) + it * N;
#pragma unroll
        for (int i = 0; i < N; ++i) er[i] = s[L::kX1 + it * N + i];
        continue;
      }
      double* row = args.y + comp * g.Ns + ((long long)Z * g.Ly + Y) * g.Lx + base[el][0];
#pragma unroll
      for (int i = 0; i < N; ++i)
        if (!constrained(g, comp, base[el][0] + i, Y, Z)) row[i] += s[L::kX1 + it * N + i];
    }
    __syncthreads();
  }
}

// E-vector mode: y += sum of the element boxes covering each lattice point.
// Along each axis a point lies in one element (interior offset) or two (a
// shared plane: offset P in the left element, 0 in the right one); the up to
// 8 contributions are summed in a fixed (z, y, x, ascending element) order,
// so results are bit-reproducible.  Constrained points are left untouched.
__device__ __forceinline__ int ev_cands(int X, int P, int n, int (&e)[2], int (&o)[2]) {
  const int q = X / P, r = X - q * P;
  if (r != 0) { e[0] = q; o[0] = r; return 1; }
  if (q == 0) { e[0] = 0; o[0] = 0; return 1; }
  if (q == n) { e[0] = n - 1; o[0] = P; return 1; }
  e[0] = q - 1; o[0] = P; e[1] = q; o[1] = 0;
  return 2;
}

// gathered value of lattice entry idx (comp-major); false on constrained points
// (E-vector mode only: meshes of <= kEvMaxElements elements, so 32-bit index math)
template <int N>
__device__ __forceinline__ bool ev_point(const double* __restrict__ ev, const Geo& g, long long idx_, double& s) {
  constexpr int P = N - 1, B = N * N * N;
  const int idx = (int)idx_, ns = (int)g.Ns;
  const int comp = idx / ns;
  const int r = idx - comp * ns;
  const int rxy = r / g.Lx, X = r - rxy * g.Lx;
  const int Z = rxy / g.Ly, Y = rxy - Z * g.Ly;
  if (constrained(g, comp, X, Y, Z)) return false;
  int ex[2], ox[2], ey[2], oy[2], ez[2], oz[2];
  const int nx = ev_cands(X, P, g.nx, ex, ox), ny = ev_cands(Y, P, g.ny, ey, oy),
            nz = ev_cands(Z, P, g.nz, ez, oz);
  // all (up to 8) loads issued before the fixed-order sum
  double v[8];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const bool ok = a < nz && b < ny && c < nx;
        const int e = (ez[a & (nz - 1)] * g.ny + ey[b & (ny - 1)]) * g.nx + ex[c & (nx - 1)];
        v[(a * 2 + b) * 2 + c] =
            ok ? ev[(long long)(e * 3 + comp) * B + (oz[a & (nz - 1)] * N + oy[b & (ny - 1)]) * N +
                    ox[c & (nx - 1)]]
               : 0.0;
      }
  s = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += v[t];
  return true;
}

template <int N>
__global__ void __launch_bounds__(256) k_ev_gather(double* __restrict__ y, const double* __restrict__ ev,
                                                   const __grid_constant__ Geo g, const int* skip) {
  if (skip && *(volatile const int*)skip) return;
  const long long total = 3 * g.Ns;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    double s;
    if (ev_point<N>(ev, g, idx, s)) y[idx] += s;
  }
}

}  // namespace sdme
