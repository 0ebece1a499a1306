// Element kernels v3 (hot path): f_int, (c_k K + c_m M) p, c_m M p.
//
// Schedule: a group of WPE warps owns one element (named-barrier / __syncwarp
// sync, no block-wide barriers), persistent over the elements of one colour
// pass; grad u at the thread's own points stays in registers between the u and
// p forward passes; results leave with fire-and-forget RED.ADD -- within a
// colour pass every lattice point gets at most one contribution and passes
// are ordered launches, so sums are bit-reproducible.  The contraction stages
// run NC displacement components at a time (NC = 3: more pencils per stage;
// NC = 1: 3x smaller stage buffers, so more elements fit per SM).
//
// Changes over the first (v1/v2) schedules, from their ncu profiles
// (profiles/ncu_apply_r01_v*.txt):
//  1. constitutive point work in the F^{-T} form (fewer FP64 instructions):
//       K = F^{-T} = cof(F)/det F,  lnJ = ln det F,
//       P  = mu F + (lam lnJ - mu) K                       (f_int, = F S)
//       dP = mu Hp + lam (K:Hp) K + (mu - lam lnJ) K Hp^T K  (= Hp S + F dS)
//     identical to material.py:65-105 / femcore.py:99-146 in exact arithmetic;
//  2. the 1D weights, det J and dxi/dX are folded into per-axis tables, so
//     points carry raw physical gradients and fluxes (no scaling multiplies);
//  3. padded shared strides and per-stage lane orders chosen with
//     tools/bank_model.py (half-warp 64-bit bank model, matches ncu counts).
// Next element's input rows are prefetched into L2 while the current one runs.
#pragma once
#include "tma.cuh"
#include "element_kernels.cuh"

namespace sdme {

template <int N, int M>
struct Tab3 {
  double B[M][N];                          // forward values
  double Dx[M][N], Dy[M][N], Dz[M][N];     // forward physical derivatives (D * 2/h)
  double bBx[M][N], bDx[M][N];             // backward x: B w, D w 2/hx
  double bBy[M][N], bDy[M][N];             // backward y
  double bBz[M][N], bDz[M][N];             // backward z (also carries det J)
};

// shared layout parameters (tools/bank_model.py search); xo: 0 natural,
// 1 j-first; yo: 0 natural, 1 ck-first, 2 k-first
template <int N, int M, int NC>
struct Lay {
  static constexpr int xo = 0, yo = 0, sx = N * M, sy = M * M;
  static constexpr int sq = M * M * M + (((M * M - M * M * M) % 16) + 16) % 16;
};
#define SDME_LAY(NN, MM, NCC, XO, YO, SX, SY, SQ) \
  template <> struct Lay<NN, MM, NCC> { static constexpr int xo = XO, yo = YO, sx = SX, sy = SY, sq = SQ; };
SDME_LAY(2, 2, 3, 0, 0, 5, 6, 20)
SDME_LAY(2, 3, 3, 0, 0, 6, 9, 41)
SDME_LAY(3, 3, 3, 0, 1, 9, 9, 41)
SDME_LAY(3, 4, 3, 0, 1, 25, 19, 64)
SDME_LAY(4, 4, 3, 0, 0, 19, 20, 64)
SDME_LAY(4, 5, 3, 0, 2, 20, 28, 137)
SDME_LAY(5, 5, 3, 1, 0, 27, 37, 137)
SDME_LAY(5, 6, 3, 0, 2, 45, 45, 228)
SDME_LAY(6, 6, 3, 1, 0, 43, 42, 228)
SDME_LAY(6, 7, 3, 1, 0, 55, 55, 353)
SDME_LAY(7, 7, 3, 1, 0, 59, 55, 353)
SDME_LAY(7, 8, 3, 1, 2, 71, 71, 512)
SDME_LAY(8, 8, 3, 1, 0, 67, 68, 512)
SDME_LAY(8, 9, 3, 1, 0, 73, 89, 737)
SDME_LAY(9, 9, 3, 1, 0, 89, 89, 737)
SDME_LAY(9, 10, 3, 0, 2, 105, 105, 1012)
SDME_LAY(5, 5, 1, 0, 0, 25, 37, 137)
#undef SDME_LAY
// stride of one (comp, s) slab of the Y layout when it is not N * sy: P = 2
// (y-stage writes over lanes (comp, k, a), z-stage reads over lanes (comp, b, a);
// bank model 63 -> 45 wavefronts per field pass, 36 ideal)
template <int N, int M, int NC>
struct LayYS {
  static constexpr int v = N * Lay<N, M, NC>::sy;
};
template <>
struct LayYS<3, 3, 3> {
  static constexpr int v = 41;
};

template <int N, int M, int WPE, int NC, bool VALS = true>
struct V3 {
  using Ly = Lay<N, M, NC>;
  static constexpr int Q = M * M * M;
  static constexpr int XS = NC * N * Ly::sx;     // one X-layout array ([comp][k] rows of sx)
  static constexpr int XO = 2 * XS;
  static constexpr int YS = LayYS<N, M, NC>::v;  // one (comp, s) slab of the Y layout
  static constexpr int YO = 3 * NC * YS;
  static constexpr int GO = (VALS ? 12 : 9) * Ly::sq;  // point slots [d][comp] of sq
  // NC = 3: the x-stage scratch reuses A (free before the points are written);
  // NC < 3: A keeps earlier groups' points, so the x scratch sits after YO in B.
  static constexpr int SA = (NC == 3 && XO > GO) ? XO : GO;
  static constexpr int SB = YO + (NC == 3 ? 0 : XO);
  static constexpr int PER = SA + SB;
  static constexpr int T = 32 * WPE;
  static constexpr int QPT = (Q + T - 1) / T;
  // X layout: [s][comp][k] rows of stride sx, row = j*M + a   (comp local to the group)
  __device__ static int xi(int s, int ck, int j, int a) { return s * XS + ck * Ly::sx + j * M + a; }
  // Y layout: [comp][s][k] rows of stride sy, row = b*M + a
  __device__ static int yi(int comp, int s, int k, int ba) { return (comp * 3 + s) * YS + k * Ly::sy + ba; }
  // point slots: [d][comp][q], d = 3 is the value slot (comp global)
  __device__ static int qi(int d, int comp, int q) { return (d * 3 + comp) * Ly::sq + q; }
  __device__ static void item_x(int w, int& ck, int& j) {
    if (Ly::xo == 0) { ck = w / N; j = w % N; }
    else { j = w / (NC * N); ck = w % (NC * N); }
  }
  __device__ static void item_y(int w, int& ck, int& a) {
    if (Ly::yo == 0) { ck = w / M; a = w % M; }
    else if (Ly::yo == 1) { a = w / (NC * N); ck = w % (NC * N); }
    else { const int c = w / (N * M), r = w % (N * M); a = r / N; ck = c * N + r % N; }
  }
};

template <int WPE>
__device__ __forceinline__ void group_sync(int gid) {
  if (WPE == 1) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(gid + 1), "r"(WPE * 32) : "memory");
  }
}

__device__ __forceinline__ void red_add(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory"); }

// Asynchronous staging of one component's (P+1)^2 rows of an element box into
// shared memory, rows [k][j] of N doubles (cp.async, no registers held).
template <int N, int T>
__device__ __forceinline__ void v3_stage_rows(const Geo& g, const double* __restrict__ field, int comp, int X0,
                                              int Y0, int Z0, double* rows, int t) {
  for (int w = t; w < N * N * N; w += T) {
    const int kj = w / N, i = w % N;
    const int k = kj / N, j = kj % N;
    SDME_CHECK(comp >= 0 && comp < 3 && Z0 + k < g.Lz && Y0 + j < g.Ly && X0 + i < g.Lx && X0 >= 0);
    cp_async8(rows + w, field + comp * g.Ns + ((long long)(Z0 + k) * g.Ly + (Y0 + j)) * g.Px + X0 + i);
  }
  cp_async_commit();
}

// What to stage after the last component of a forward pass.
struct NextRows {
  const double* field;  // nullptr: nothing to stage
  int X0, Y0, Z0;
};

// TMA element boxes of the NC = 3 kernels (element_v3 TMB): the x stage reads
// rows from a shared box [comp][k][j][BW] (rows start at `shift`, the box's x
// start is the even lattice x at or below X0), the x' stage writes the output
// box that one lane then adds back with bulk tensor reduce-adds (tma.cuh).
template <int N>
struct BoxW {
  static constexpr int BW = (N + 2) & ~1;  // even box width covering [X0, X0 + N) from an even start
  static constexpr int CB = (N * N * BW + 15) / 16 * 16;  // one component's box (TMA: 128-B aligned)
};
struct BoxIO {
  const double* in = nullptr;   // forward: shared input box
  double* out = nullptr;        // backward: shared output box
  int shift = 0;                // X0 - (box x start)
  const void* ymap = nullptr;   // backward: tensor map of the output vector
  int xs = 0, Y0 = 0, Z0 = 0;   // box start
};

template <int N, int T>
__device__ __forceinline__ void v3_prefetch(const Geo& g, const double* __restrict__ src, int X0, int Y0, int Z0,
                                            int t) {
  for (int w = t; w < 3 * N * N; w += T) {
    const int comp = w / (N * N), kj = w % (N * N);
    const double* row = src + comp * g.Ns + ((long long)(Z0 + kj / N) * g.Ly + (Y0 + kj % N)) * g.Px + X0;
    prefetch_l2(row);
    prefetch_l2(row + N - 1);
  }
}

// Forward pass of the three components of one field.  STAGED (NC == 1): the
// element rows come from the cp.async double buffer R (component c0 already
// staged into R + buf*N^3 by the caller / previous pass); the next
// component's rows -- or `next` after the last one -- are staged while this
// component computes, so global latency is off the critical path.
template <int N, int M, int WPE, int NC, bool GRAD, bool VAL, bool STAGED = false>
__device__ __forceinline__ void v3_forward(const Tab3<N, M>& tb0, int zv, const Geo& g, const double* __restrict__ src,
                                           int X0, int Y0, int Z0, double* A, double* B, int t, int gid,
                                           double* R = nullptr, int* buf = nullptr, NextRows next = {},
                                           BoxIO = {}) {
  using C = V3<N, M, WPE, NC>;
  static_assert(!STAGED || NC == 1, "row staging is per component");
  constexpr int NX = NC * N * N, NY = NC * N * M, NZ = NC * M * M;
  double* const P = A;  // points buffer (all components)
#pragma unroll 1
  for (int c0 = 0; c0 < 3; c0 += NC) {
    // tables re-read from the constant bank per element / component group (OpArgs::zero)
    const auto& tb = reload_tab(tb0, N >= SDME_V3_RELOAD_MIN_N ? zv * (c0 + 1) : 0);
    double* const X = (NC == 3) ? A : B + C::YO;  // x-stage scratch (see V3::SB)
    if (STAGED) {
      double* nb = R + (*buf ^ 1) * N * N * N;
      if (c0 + 1 < 3) {
        v3_stage_rows<N, C::T>(g, src, c0 + 1, X0, Y0, Z0, nb, t);
        cp_async_wait<1>();
      } else if (next.field) {
        v3_stage_rows<N, C::T>(g, next.field, 0, next.X0, next.Y0, next.Z0, nb, t);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      group_sync<WPE>(gid);
    }
#pragma unroll
    for (int r = 0; r < (NX + C::T - 1) / C::T; ++r) {
      const int w = t + r * C::T;
      if (w < NX) {
        int ck, j;
        C::item_x(w, ck, j);
        const int comp = c0 + ck / N, k = ck % N;
        double v[N];
        if (STAGED) {
          const double* row = R + *buf * N * N * N + (k * N + j) * N;
#pragma unroll
          for (int i = 0; i < N; ++i) v[i] = row[i];
        } else {
          const double* row = src + comp * g.Ns + ((long long)(Z0 + k) * g.Ly + (Y0 + j)) * g.Px + X0;
#pragma unroll
          for (int i = 0; i < N; ++i) v[i] = __ldg(row + i);
        }
#pragma unroll
        for (int a = 0; a < M; ++a) {
          double b0 = 0.0, b1 = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) {
            b0 = fma(tb.B[a][i], v[i], b0);
            if (GRAD) b1 = fma(tb.Dx[a][i], v[i], b1);
          }
          X[C::xi(0, ck, j, a)] = b0;
          if (GRAD) X[C::xi(1, ck, j, a)] = b1;
        }
      }
    }
    group_sync<WPE>(gid);
#pragma unroll
    for (int r = 0; r < (NY + C::T - 1) / C::T; ++r) {
      const int w = t + r * C::T;
      if (w < NY) {
        int ck, a;
        C::item_y(w, ck, a);
        double x0[N], x1[N];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          x0[j] = X[C::xi(0, ck, j, a)];
          if (GRAD) x1[j] = X[C::xi(1, ck, j, a)];
        }
        const int cl = ck / N, k = ck % N;
#pragma unroll
        for (int b = 0; b < M; ++b) {
          double bb = 0.0, db = 0.0, bd = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            bb = fma(tb.B[b][j], x0[j], bb);
            if (GRAD) {
              db = fma(tb.Dy[b][j], x0[j], db);
              bd = fma(tb.B[b][j], x1[j], bd);
            }
          }
          B[C::yi(cl, 0, k, b * M + a)] = bb;  // B_y B_x
          if (GRAD) {
            B[C::yi(cl, 1, k, b * M + a)] = db;  // D_y B_x
            B[C::yi(cl, 2, k, b * M + a)] = bd;  // B_y D_x
          }
        }
      }
    }
    group_sync<WPE>(gid);
#pragma unroll
    for (int r = 0; r < (NZ + C::T - 1) / C::T; ++r) {
      const int w = t + r * C::T;
      if (w < NZ) {
        const int cl = w / (M * M), ba = w % (M * M);
        const int comp = c0 + cl;
        double y0[N], y1[N], y2[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          y0[k] = B[C::yi(cl, 0, k, ba)];
          if (GRAD) {
            y1[k] = B[C::yi(cl, 1, k, ba)];
            y2[k] = B[C::yi(cl, 2, k, ba)];
          }
        }
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double gx = 0.0, gy = 0.0, gz = 0.0, vv = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) {
            if (GRAD) {
              gx = fma(tb.B[c][k], y2[k], gx);
              gy = fma(tb.B[c][k], y1[k], gy);
              gz = fma(tb.Dz[c][k], y0[k], gz);
            }
            if (VAL) vv = fma(tb.B[c][k], y0[k], vv);
          }
          const int q = c * M * M + ba;
          if (GRAD) {
            P[C::qi(0, comp, q)] = gx;
            P[C::qi(1, comp, q)] = gy;
            P[C::qi(2, comp, q)] = gz;
          }
          if (VAL) P[C::qi(3, comp, q)] = vv;
        }
      }
    }
    if (STAGED) *buf ^= 1;
    group_sync<WPE>(gid);
  }
}

// evb != nullptr (E-vector mode): the element's box goes to evb[comp][k][j][i]
// instead of being scattered with RED into the lattice.
template <int N, int M, int WPE, int NC, bool GRAD, bool VAL>
__device__ __forceinline__ void v3_backward(const Tab3<N, M>& tb0, int zv, const Geo& g, double* __restrict__ dst,
                                            int X0, int Y0, int Z0, double* A, double* B, int t, int gid,
                                            double* evb = nullptr, BoxIO = {}) {
  using C = V3<N, M, WPE, NC>;
  constexpr int NX = NC * N * N, NY = NC * N * M, NZ = NC * M * M;
#pragma unroll 1
  for (int c0 = 0; c0 < 3; c0 += NC) {
    // tables re-read from the constant bank per element / component group (OpArgs::zero)
    const auto& tb = reload_tab(tb0, N >= SDME_V3_RELOAD_MIN_N ? zv * (c0 + 1) : 0);
    double* const X = (NC == 3) ? A : B + C::YO;
#pragma unroll
    for (int r = 0; r < (NZ + C::T - 1) / C::T; ++r) {
      const int w = t + r * C::T;
      if (w < NZ) {
        const int cl = w / (M * M), ba = w % (M * M);
        const int comp = c0 + cl;
        double qx[M], qy[M], qz[M], qv[M];
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const int q = c * M * M + ba;
          if (GRAD) {
            qx[c] = A[C::qi(0, comp, q)];
            qy[c] = A[C::qi(1, comp, q)];
            qz[c] = A[C::qi(2, comp, q)];
          }
          if (VAL) qv[c] = A[C::qi(3, comp, q)];
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          double hx = 0.0, hy = 0.0, hz = 0.0;
#pragma unroll
          for (int c = 0; c < M; ++c) {
            if (GRAD) {
              hx = fma(tb.bBz[c][k], qx[c], hx);
              hy = fma(tb.bBz[c][k], qy[c], hy);
              hz = fma(tb.bDz[c][k], qz[c], hz);
            }
            if (VAL) hz = fma(tb.bBz[c][k], qv[c], hz);
          }
          if (GRAD) {
            B[C::yi(cl, 0, k, ba)] = hx;
            B[C::yi(cl, 1, k, ba)] = hy;
          }
          B[C::yi(cl, 2, k, ba)] = hz;
        }
      }
    }
    group_sync<WPE>(gid);
#pragma unroll
    for (int r = 0; r < (NY + C::T - 1) / C::T; ++r) {
      const int w = t + r * C::T;
      if (w < NY) {
        int ck, a;
        C::item_y(w, ck, a);
        const int cl = ck / N, k = ck % N;
        double hx[M], hy[M], hz[M];
#pragma unroll
        for (int b = 0; b < M; ++b) {
          if (GRAD) {
            hx[b] = B[C::yi(cl, 0, k, b * M + a)];
            hy[b] = B[C::yi(cl, 1, k, b * M + a)];
          }
          hz[b] = B[C::yi(cl, 2, k, b * M + a)];
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double jx = 0.0, jyz = 0.0;
#pragma unroll
          for (int b = 0; b < M; ++b) {
            if (GRAD) {
              jx = fma(tb.bBy[b][j], hx[b], jx);
              jyz = fma(tb.bDy[b][j], hy[b], jyz);
            }
            jyz = fma(tb.bBy[b][j], hz[b], jyz);
          }
          if (GRAD) X[C::xi(0, ck, j, a)] = jx;
          X[C::xi(1, ck, j, a)] = jyz;
        }
      }
    }
    group_sync<WPE>(gid);
#pragma unroll
    for (int r = 0; r < (NX + C::T - 1) / C::T; ++r) {
      const int w = t + r * C::T;
      if (w < NX) {
        int ck, j;
        C::item_x(w, ck, j);
        const int comp = c0 + ck / N, k = ck % N;
        double jx[M], jyz[M];
#pragma unroll
        for (int a = 0; a < M; ++a) {
          if (GRAD) jx[a] = X[C::xi(0, ck, j, a)];
          jyz[a] = X[C::xi(1, ck, j, a)];
        }
        const int Z = Z0 + k, Y = Y0 + j;
        const bool chk = touches_dirichlet(g, comp, X0, Y0, Z0, N);
        double* row = dst + comp * g.Ns + ((long long)Z * g.Ly + Y) * g.Px + X0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double acc = 0.0;
#pragma unroll
          for (int a = 0; a < M; ++a) {
            if (GRAD) acc = fma(tb.bDx[a][i], jx[a], acc);
            acc = fma(tb.bBx[a][i], jyz[a], acc);
          }
          if (evb) evb[((comp * N + k) * N + j) * N + i] = acc;
          else if (!chk || !constrained(g, comp, X0 + i, Y, Z)) red_add(row + i, acc);
        }
      }
    }
    group_sync<WPE>(gid);
  }
}

// K = F^{-T}, det F, ln det F from H = grad u
struct QpK {
  double F[3][3];
  double K[3][3];
  double det, lnJ;
};

__device__ __forceinline__ void qp_k(const double (&H)[9], QpK& s) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) s.F[i][j] = H[i * 3 + j] + (i == j ? 1.0 : 0.0);
  const double(&F)[3][3] = s.F;
  const double c00 = F[1][1] * F[2][2] - F[1][2] * F[2][1];
  const double c01 = F[1][2] * F[2][0] - F[1][0] * F[2][2];
  const double c02 = F[1][0] * F[2][1] - F[1][1] * F[2][0];
  const double c10 = F[0][2] * F[2][1] - F[0][1] * F[2][2];
  const double c11 = F[0][0] * F[2][2] - F[0][2] * F[2][0];
  const double c12 = F[0][1] * F[2][0] - F[0][0] * F[2][1];
  const double c20 = F[0][1] * F[1][2] - F[0][2] * F[1][1];
  const double c21 = F[0][2] * F[1][0] - F[0][0] * F[1][2];
  const double c22 = F[0][0] * F[1][1] - F[0][1] * F[1][0];
  s.det = F[0][0] * c00 + F[0][1] * c01 + F[0][2] * c02;
  const double inv = 1.0 / s.det;
  s.K[0][0] = c00 * inv; s.K[0][1] = c01 * inv; s.K[0][2] = c02 * inv;
  s.K[1][0] = c10 * inv; s.K[1][1] = c11 * inv; s.K[1][2] = c12 * inv;
  s.K[2][0] = c20 * inv; s.K[2][1] = c21 * inv; s.K[2][2] = c22 * inv;
  s.lnJ = log(s.det);
}

// STG: cp.async double-buffered row staging (NC == 1); needs 2*N^3 extra
// doubles of shared memory per element (see V3 launch in sdme_abi.cu).
// TB: Tab3 (plain contractions) or TabEO (even-odd, element_eo.cuh).
// TMB: TMA element boxes (NC == 3, WPE == 1, even-odd tables): per element two
// staging boxes of all three components (u / p / next element, mbarrier
// completion) and an output box added back with bulk tensor reduce-adds.
template <int N, int M, int WPE, int NC, bool VALS, bool STG, bool TMB>
struct V3Smem {
  using C = V3<N, M, WPE, NC, VALS>;
  static constexpr int BW = BoxW<N>::BW;
  static constexpr int BOX = 3 * BoxW<N>::CB;  // one box: three 128-B aligned component boxes
  static constexpr int BOXO = (C::PER + 15) / 16 * 16;
  static constexpr int PERS =
      TMB ? (BOXO + 3 * BOX + 2 + 15) / 16 * 16 : C::PER + (STG ? 2 * N * N * N : 0);
};

template <int N, int M, int WPE, int NC, int EPB, int MINB, int MODE, bool VAL, bool STG = false,
          class TB = Tab3<N, M>, bool TMB = false>
__global__ void __launch_bounds__(EPB * WPE * 32, MINB) element_v3(const __grid_constant__ TB tb,
                                                                     const __grid_constant__ Geo g, OpArgs args) {
  using C = V3<N, M, WPE, NC, VAL || MODE == MODE_MASS>;
  using SM = V3Smem<N, M, WPE, NC, VAL || MODE == MODE_MASS, STG, TMB>;
  static_assert(!TMB || (NC == 3 && WPE == 1 && !STG), "TMA boxes: all-component shape");
  constexpr int PERS = SM::PERS;
  constexpr int BW = SM::BW;
  extern __shared__ __align__(128) double smem[];
  const int gid = threadIdx.x / C::T;
  const int t = threadIdx.x % C::T;
  double* A = smem + gid * PERS;
  SDME_CHECK(smem_ok(A, PERS * 8, 8));
  double* Bf = A + C::SA;
  double* Rb = A + C::PER;  // staged rows [2][N^3] (STG)
  int buf = 0;
  if (args.skip && *(volatile const int*)args.skip) return;
  const long long cnt = colour_count(g, args.colour);
  constexpr bool GRADP = (MODE == MODE_APPLY || MODE == MODE_PA);
  constexpr bool UPASS = (MODE == MODE_APPLY || MODE == MODE_FINT || MODE == MODE_SETUP || MODE == MODE_ENERGY);
  constexpr bool PPASS = (MODE == MODE_APPLY || MODE == MODE_MASS || MODE == MODE_PA);
  const long long stride = (long long)gridDim.x * EPB;
  // dP constants with c_k folded in
  const double mu_k = args.c_k * g.mu, lam_k = args.c_k * g.lam;
  const double cmr = args.c_m * g.rho;
  const double* first_field = UPASS ? args.u : args.p;
  // TMB: boxes [buf 0][buf 1][out], then two mbarriers (one per staging box)
  double* Rbox = A + SM::BOXO;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(Rbox + 3 * SM::BOX);
  const CUtensorMap* umap = static_cast<const CUtensorMap*>(args.tu);
  const CUtensorMap* pmap = static_cast<const CUtensorMap*>(args.tp);
  unsigned ph = 0;
  auto issue = [&](const CUtensorMap* map, int X0, int Y0, int Z0, int b) {
    // one lane: the three component boxes of an element into staging box b
    mbar_expect_tx(bars + b, 3 * N * N * BW * 8);
#pragma unroll
    for (int c = 0; c < 3; ++c) tma_load_box(Rbox + b * SM::BOX + c * BoxW<N>::CB, map, X0 & ~1, Y0, Z0, c, bars + b);
  };
  if (TMB) {
    if (t == 0) {
      mbar_init(bars, 1);
      mbar_init(bars + 1, 1);
      mbar_fence_init();
    }
    group_sync<WPE>(gid);
    if (t == 0 && (long long)blockIdx.x * EPB + gid < cnt) {
      int ei, ej, ek;
      colour_element(g, args.colour, (long long)blockIdx.x * EPB + gid, ei, ej, ek);
      issue(UPASS ? umap : pmap, (N - 1) * ei, (N - 1) * ej, (N - 1) * ek, 0);
    }
  }
  if (STG && (long long)blockIdx.x * EPB + gid < cnt) {
    int ei, ej, ek;
    colour_element(g, args.colour, (long long)blockIdx.x * EPB + gid, ei, ej, ek);
    v3_stage_rows<N, C::T>(g, first_field, 0, (N - 1) * ei, (N - 1) * ej, (N - 1) * ek, Rb, t);
  }
  int zit = 0;  // loop-variant multiplier of args.zero (table re-reads, OpArgs::zero)
  for (long long idx = (long long)blockIdx.x * EPB + gid; idx < cnt; idx += stride) {
    const int zv = args.zero * (++zit);
    int ei, ej, ek;
    colour_element(g, args.colour, idx, ei, ej, ek);
    const int X0 = (N - 1) * ei, Y0 = (N - 1) * ej, Z0 = (N - 1) * ek;
    NextRows nxt{nullptr, 0, 0, 0};
    if (STG && idx + stride < cnt) {
      int ni, nj, nk;
      colour_element(g, args.colour, idx + stride, ni, nj, nk);
      nxt = NextRows{first_field, (N - 1) * ni, (N - 1) * nj, (N - 1) * nk};
    }
    int nX0 = -1, nY0 = 0, nZ0 = 0;  // TMB: next element of this warp
    if (TMB && idx + stride < cnt) {
      int ni, nj, nk;
      colour_element(g, args.colour, idx + stride, ni, nj, nk);
      nX0 = (N - 1) * ni, nY0 = (N - 1) * nj, nZ0 = (N - 1) * nk;
    }
    if (!STG && !TMB && idx + stride < cnt) {  // warm L2 with the next element's rows
      int ni, nj, nk;
      colour_element(g, args.colour, idx + stride, ni, nj, nk);
      if (UPASS) v3_prefetch<N, C::T>(g, args.u, (N - 1) * ni, (N - 1) * nj, (N - 1) * nk, t);
      if (PPASS) v3_prefetch<N, C::T>(g, args.p, (N - 1) * ni, (N - 1) * nj, (N - 1) * nk, t);
    }
    BoxIO bx{};
    bx.shift = X0 & 1;
    auto box_next = [&](bool to_p) {
      // TMB: issue the next box into the other buffer, wait for the current one
      if (!TMB) return;
      if (t == 0) {
        if (to_p) issue(pmap, X0, Y0, Z0, buf ^ 1);
        else if (nX0 >= 0) issue(UPASS ? umap : pmap, nX0, nY0, nZ0, buf ^ 1);
      }
      mbar_wait(bars + buf, (ph >> buf) & 1u);
      ph ^= 1u << buf;
      bx.in = Rbox + buf * SM::BOX;
    };
    double Hu[C::QPT][9];
    if (UPASS) {
      const NextRows after_u = MODE == MODE_APPLY ? NextRows{args.p, X0, Y0, Z0} : nxt;
      box_next(MODE == MODE_APPLY);
      v3_forward<N, M, WPE, NC, true, false, STG>(tb, zv, g, args.u, X0, Y0, Z0, A, Bf, t, gid, Rb, &buf, after_u, bx);
      if (TMB) buf ^= 1;
#pragma unroll
      for (int r = 0; r < C::QPT; ++r) {
        const int q = t + r * C::T;
        if (q < C::Q) {
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int d = 0; d < 3; ++d) Hu[r][i * 3 + d] = A[C::qi(d, i, q)];
        }
      }
      group_sync<WPE>(gid);
    }
    if (PPASS) {
      box_next(false);
      v3_forward<N, M, WPE, NC, GRADP, VAL, STG>(tb, zv, g, args.p, X0, Y0, Z0, A, Bf, t, gid, Rb, &buf, nxt, bx);
      if (TMB) buf ^= 1;
    }
#pragma unroll
    for (int r = 0; r < C::QPT; ++r) {
      const int q = t + r * C::T;
      if (q >= C::Q) continue;
      if (MODE == MODE_MASS) {
#pragma unroll
        for (int i = 0; i < 3; ++i) A[C::qi(3, i, q)] *= cmr;
        continue;
      }
      const long long eid = ((long long)ek * g.ny + ej) * g.nx + ei;
      QpK s;
      if (MODE == MODE_PA) {
        const double* qd = args.qpd + eid * (kQpSlots * C::Q) + q;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) s.K[i][d] = __ldg(qd + (i * 3 + d) * C::Q);
        s.lnJ = __ldg(qd + 9 * C::Q);
      } else {
        qp_k(Hu[r], s);
        if (!(s.det > 0.0)) {
          const int a = q % M, b = (q / M) % M, c = q / (M * M);
          atomicMin(args.inv_flag, (unsigned long long)eid * C::Q + (unsigned long long)((a * M + b) * M + c));
        }
      }
      if (MODE == MODE_ENERGY) {
        // psi = mu/2 (tr C - 3) - mu ln J + lam/2 ln J^2 (material.py:80), weighted
        double trc = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) trc = fma(s.F[i][d], s.F[i][d], trc);
        const double psi = 0.5 * g.mu * (trc - 3.0) - g.mu * s.lnJ + 0.5 * g.lam * s.lnJ * s.lnJ;
        const int a = q % M, b = (q / M) % M, c = q / (M * M);
        A[C::qi(0, 0, q)] = __ldg(args.p + a) * __ldg(args.p + b) * __ldg(args.p + c) * g.detJ * psi;
        continue;
      }
      if (MODE == MODE_SETUP) {
        double* qd = args.qpd + eid * (kQpSlots * C::Q) + q;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) qd[(i * 3 + d) * C::Q] = s.K[i][d];
        qd[9 * C::Q] = s.lnJ;
        continue;
      }
      if (MODE == MODE_FINT) {
        const double cK = g.lam * s.lnJ - g.mu;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) A[C::qi(d, i, q)] = fma(g.mu, s.F[i][d], cK * s.K[i][d]);
      } else {
        double Hp[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) Hp[i][d] = A[C::qi(d, i, q)];
        double tr = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) tr = fma(s.K[i][d], Hp[i][d], tr);
        // M1 = K Hp^T
        double M1[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j)
            M1[i][j] = fma(s.K[i][0], Hp[j][0], fma(s.K[i][1], Hp[j][1], s.K[i][2] * Hp[j][2]));
        const double cc = mu_k - lam_k * s.lnJ;
        const double lt = lam_k * tr;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const double m2 = fma(M1[i][0], s.K[0][d], fma(M1[i][1], s.K[1][d], M1[i][2] * s.K[2][d]));
            A[C::qi(d, i, q)] = fma(cc, m2, fma(lt, s.K[i][d], mu_k * Hp[i][d]));
          }
        if (VAL) {
#pragma unroll
          for (int i = 0; i < 3; ++i) A[C::qi(3, i, q)] *= cmr;
        }
      }
    }
    group_sync<WPE>(gid);
    if (MODE == MODE_SETUP) continue;
    if (MODE == MODE_ENERGY) {
      // fixed-order element sum (one thread), then the next element may reuse A
      if (t == 0) {
        double e = 0.0;
        for (int q = 0; q < C::Q; ++q) e += A[C::qi(0, 0, q)];
        args.qpd[((long long)ek * g.ny + ej) * g.nx + ei] = e;
      }
      group_sync<WPE>(gid);
      continue;
    }
    double* evb = args.ev ? args.ev + (((long long)ek * g.ny + ej) * g.nx + ei) * 3 * (N * N * N) : nullptr;
    if (TMB) {
      bx.out = Rbox + 2 * SM::BOX;
      bx.ymap = args.ty;
      bx.xs = X0 & ~1, bx.Y0 = Y0, bx.Z0 = Z0;
    }
    if (MODE == MODE_MASS)
      v3_backward<N, M, WPE, NC, false, true>(tb, zv, g, args.y, X0, Y0, Z0, A, Bf, t, gid, evb, bx);
    else if (MODE == MODE_FINT)
      v3_backward<N, M, WPE, NC, true, false>(tb, zv, g, args.y, X0, Y0, Z0, A, Bf, t, gid, evb, bx);
    else
      v3_backward<N, M, WPE, NC, true, VAL>(tb, zv, g, args.y, X0, Y0, Z0, A, Bf, t, gid, evb, bx);
  }
  if (TMB && t == 0) bulk_wait_all();
}

}  // namespace sdme
