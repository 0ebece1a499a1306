// Element kernels v2: a group of WPE warps per element, persistent over the
// elements of one colour pass, no block-wide barriers.
//
// Same mathematics as element_kernels.cuh (f_int, (c_k K + c_m M) p, c_m M p;
// femcore.py:87-156), re-scheduled for latency tolerance on sm_100a:
//  * each element is owned by WPE warps that synchronise with a named barrier
//    (WPE = 1: __syncwarp) -- no __syncthreads across unrelated elements;
//  * all three displacement components go through each contraction stage
//    together (3x the independent pencils per stage);
//  * grad u at the thread's own points lives in registers between the u and p
//    forward passes, so only two shared buffers per element are needed;
//  * results leave with fire-and-forget RED.ADD: within a colour pass every
//    lattice point receives at most one contribution and passes are ordered
//    kernel launches, so the sum at each point is bit-reproducible.
#pragma once
#include "element_kernels.cuh"

namespace sdme {

template <int N, int M, int WPE>
struct V2 {
  static constexpr int Q = M * M * M;
  static constexpr int XO = 3 * 2 * N * N * M;  // x stage: [comp][B|D][k][j][a]
  static constexpr int YO = 3 * 3 * N * M * M;  // y stage: [comp][3][k][b][a]
  static constexpr int GO = 12 * Q;             // points:  [comp][4][c][b][a]
  static constexpr int SA = XO > GO ? XO : GO;
  static constexpr int SB = YO;
  static constexpr int PER = SA + SB;           // doubles of shared memory per element
  static constexpr int T = 32 * WPE;
  static constexpr int QPT = (Q + T - 1) / T;   // points per thread
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

// forward pass of the three components of one field: global lattice -> A (points)
template <int N, int M, int WPE, bool GRAD, bool VAL>
__device__ __forceinline__ void v2_forward(const Tab<N, M>& tb, const Geo& g, const double* __restrict__ src,
                                           int X0, int Y0, int Z0, double* A, double* B, int t, int gid) {
  using C = V2<N, M, WPE>;
  constexpr int NX = 3 * N * N;
  // stage X: items (comp, k, j), pencil along x straight from global memory
#pragma unroll
  for (int r = 0; r < (NX + C::T - 1) / C::T; ++r) {
    const int w = t + r * C::T;
    if (w < NX) {
      const int comp = w / (N * N), kj = w % (N * N);
      const int k = kj / N, j = kj % N;
      const double* row = src + comp * g.Ns + ((long long)(Z0 + k) * g.Ly + (Y0 + j)) * g.Lx + X0;
      double v[N];
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = __ldg(row + i);
#pragma unroll
      for (int a = 0; a < M; ++a) {
        double b0 = 0.0, b1 = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) {
          b0 = fma(tb.B[a][i], v[i], b0);
          if (GRAD) b1 = fma(tb.D[a][i], v[i], b1);
        }
        A[w * M + a] = b0;
        if (GRAD) A[NX * M + w * M + a] = b1;
      }
    }
  }
  group_sync<WPE>(gid);
  // stage Y: items (comp, k, a)
  constexpr int NY = 3 * N * M;
#pragma unroll
  for (int r = 0; r < (NY + C::T - 1) / C::T; ++r) {
    const int w = t + r * C::T;
    if (w < NY) {
      const int ck = w / M, a = w % M;  // ck = comp*N + k
      double x0[N], x1[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        x0[j] = A[(ck * N + j) * M + a];
        if (GRAD) x1[j] = A[NX * M + (ck * N + j) * M + a];
      }
      const int comp = ck / N, k = ck % N;
#pragma unroll
      for (int b = 0; b < M; ++b) {
        double bb = 0.0, db = 0.0, bd = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          bb = fma(tb.B[b][j], x0[j], bb);
          if (GRAD) {
            db = fma(tb.D[b][j], x0[j], db);
            bd = fma(tb.B[b][j], x1[j], bd);
          }
        }
        const int o = ((comp * 3) * N + k) * M * M + b * M + a;
        B[o] = bb;
        if (GRAD) {
          B[o + N * M * M] = db;
          B[o + 2 * N * M * M] = bd;
        }
      }
    }
  }
  group_sync<WPE>(gid);
  // stage Z: items (comp, b, a) -> points [comp][d][c][b][a]
  constexpr int NZ = 3 * M * M;
#pragma unroll
  for (int r = 0; r < (NZ + C::T - 1) / C::T; ++r) {
    const int w = t + r * C::T;
    if (w < NZ) {
      const int comp = w / (M * M), ba = w % (M * M);
      double y0[N], y1[N], y2[N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const int o = ((comp * 3) * N + k) * M * M + ba;
        y0[k] = B[o];
        if (GRAD) {
          y1[k] = B[o + N * M * M];
          y2[k] = B[o + 2 * N * M * M];
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
            gz = fma(tb.D[c][k], y0[k], gz);
          }
          if (VAL) vv = fma(tb.B[c][k], y0[k], vv);
        }
        const int q = c * M * M + ba;
        if (GRAD) {
          A[(comp * 4 + 0) * C::Q + q] = gx * g.s[0];
          A[(comp * 4 + 1) * C::Q + q] = gy * g.s[1];
          A[(comp * 4 + 2) * C::Q + q] = gz * g.s[2];
        }
        if (VAL) A[(comp * 4 + 3) * C::Q + q] = vv;
      }
    }
  }
  group_sync<WPE>(gid);
}

// backward pass: fluxes in A ([comp][4][q]) -> element vector -> RED into y
template <int N, int M, int WPE, bool GRAD, bool VAL>
__device__ __forceinline__ void v2_backward(const Tab<N, M>& tb, const Geo& g, double* __restrict__ dst,
                                            int X0, int Y0, int Z0, double* A, double* B, int t, int gid) {
  using C = V2<N, M, WPE>;
  constexpr int NZ = 3 * M * M;
  // stage Z': items (comp, b, a), contract over c -> B [comp][3][k][b][a]
#pragma unroll
  for (int r = 0; r < (NZ + C::T - 1) / C::T; ++r) {
    const int w = t + r * C::T;
    if (w < NZ) {
      const int comp = w / (M * M), ba = w % (M * M);
      double qx[M], qy[M], qz[M], qv[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        const int q = c * M * M + ba;
        if (GRAD) {
          qx[c] = A[(comp * 4 + 0) * C::Q + q];
          qy[c] = A[(comp * 4 + 1) * C::Q + q];
          qz[c] = A[(comp * 4 + 2) * C::Q + q];
        }
        if (VAL) qv[c] = A[(comp * 4 + 3) * C::Q + q];
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        double hx = 0.0, hy = 0.0, hz = 0.0;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          if (GRAD) {
            hx = fma(tb.B[c][k], qx[c], hx);
            hy = fma(tb.B[c][k], qy[c], hy);
            hz = fma(tb.D[c][k], qz[c], hz);
          }
          if (VAL) hz = fma(tb.B[c][k], qv[c], hz);
        }
        const int o = ((comp * 3) * N + k) * M * M + ba;
        if (GRAD) {
          B[o] = hx;
          B[o + N * M * M] = hy;
        }
        B[o + 2 * N * M * M] = hz;
      }
    }
  }
  group_sync<WPE>(gid);
  // stage Y': items (comp, k, a), contract over b -> A [comp][2][k][j][a]
  constexpr int NY = 3 * N * M;
#pragma unroll
  for (int r = 0; r < (NY + C::T - 1) / C::T; ++r) {
    const int w = t + r * C::T;
    if (w < NY) {
      const int ck = w / M, a = w % M;
      const int comp = ck / N, k = ck % N;
      double hx[M], hy[M], hz[M];
#pragma unroll
      for (int b = 0; b < M; ++b) {
        const int o = ((comp * 3) * N + k) * M * M + b * M + a;
        if (GRAD) {
          hx[b] = B[o];
          hy[b] = B[o + N * M * M];
        }
        hz[b] = B[o + 2 * N * M * M];
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double jx = 0.0, jyz = 0.0;
#pragma unroll
        for (int b = 0; b < M; ++b) {
          if (GRAD) {
            jx = fma(tb.B[b][j], hx[b], jx);
            jyz = fma(tb.D[b][j], hy[b], jyz);
          }
          jyz = fma(tb.B[b][j], hz[b], jyz);
        }
        const int o = (ck * N + j) * M + a;
        if (GRAD) A[o] = jx;
        A[3 * N * N * M + o] = jyz;
      }
    }
  }
  group_sync<WPE>(gid);
  // stage X': items (comp, k, j), contract over a, RED into the lattice
  constexpr int NX = 3 * N * N;
#pragma unroll
  for (int r = 0; r < (NX + C::T - 1) / C::T; ++r) {
    const int w = t + r * C::T;
    if (w < NX) {
      const int comp = w / (N * N), kj = w % (N * N);
      const int k = kj / N, j = kj % N;
      double jx[M], jyz[M];
#pragma unroll
      for (int a = 0; a < M; ++a) {
        if (GRAD) jx[a] = A[w * M + a];
        jyz[a] = A[3 * N * N * M + w * M + a];
      }
      const int Z = Z0 + k, Y = Y0 + j;
      double* row = dst + comp * g.Ns + ((long long)Z * g.Ly + Y) * g.Lx + X0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < M; ++a) {
          if (GRAD) acc = fma(tb.D[a][i], jx[a], acc);
          acc = fma(tb.B[a][i], jyz[a], acc);
        }
        if (!constrained(g, comp, X0 + i, Y, Z)) red_add(row + i, acc);
      }
    }
  }
  group_sync<WPE>(gid);
}

// One colour pass.  Block = EPB elements x WPE warps; persistent grid-stride
// over the elements of the colour.
template <int N, int M, int WPE, int EPB, int MODE, bool VAL>
__global__ void __launch_bounds__(EPB * WPE * 32) element_v2(const __grid_constant__ Tab<N, M> tb,
                                                               const __grid_constant__ Geo g, OpArgs args) {
  using C = V2<N, M, WPE>;
  extern __shared__ double smem[];
  const int gid = threadIdx.x / C::T;      // element slot in the block
  const int t = threadIdx.x % C::T;        // thread within the element group
  double* A = smem + gid * C::PER;
  double* Bf = A + C::SA;
  const long long cnt = colour_count(g, args.colour);
  constexpr bool GRADP = (MODE == MODE_APPLY);
  for (long long idx = (long long)blockIdx.x * EPB + gid; idx < cnt; idx += (long long)gridDim.x * EPB) {
    int ei, ej, ek;
    colour_element(g, args.colour, idx, ei, ej, ek);
    const int X0 = (N - 1) * ei, Y0 = (N - 1) * ej, Z0 = (N - 1) * ek;
    double Hu[C::QPT][9];
    if (MODE != MODE_MASS) {
      v2_forward<N, M, WPE, true, false>(tb, g, args.u, X0, Y0, Z0, A, Bf, t, gid);
#pragma unroll
      for (int r = 0; r < C::QPT; ++r) {
        const int q = t + r * C::T;
        if (q < C::Q) {
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int d = 0; d < 3; ++d) Hu[r][i * 3 + d] = A[(i * 4 + d) * C::Q + q];
        }
      }
      group_sync<WPE>(gid);
    }
    if (MODE != MODE_FINT)
      v2_forward<N, M, WPE, GRADP, VAL>(tb, g, args.p, X0, Y0, Z0, A, Bf, t, gid);
    // point work: flux written in place into A
#pragma unroll
    for (int r = 0; r < C::QPT; ++r) {
      const int q = t + r * C::T;
      if (q >= C::Q) continue;
      const int a = q % M, b = (q / M) % M, c = q / (M * M);
      const double wq = tb.W[a] * tb.W[b] * tb.W[c] * g.detJ;
      if (MODE == MODE_MASS) {
        const double sc = args.c_m * g.rho * wq;
#pragma unroll
        for (int i = 0; i < 3; ++i) A[(i * 4 + 3) * C::Q + q] *= sc;
        continue;
      }
      double H[3][3];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int d = 0; d < 3; ++d) H[i][d] = Hu[r][i * 3 + d];
      QpState st;
      qp_state(H, g.mu, g.lam, st);
      if (st.detF <= 0.0) {
        const long long e = ((long long)ek * g.ny + ej) * g.nx + ei;
        atomicMin(args.inv_flag, (unsigned long long)e * C::Q + (unsigned long long)((a * M + b) * M + c));
      }
      if (MODE == MODE_FINT) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const double p1 = st.F[i][0] * st.S[0][d] + st.F[i][1] * st.S[1][d] + st.F[i][2] * st.S[2][d];
            A[(i * 4 + d) * C::Q + q] = wq * g.s[d] * p1;
          }
      } else {
        double Hp[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) Hp[i][d] = A[(i * 4 + d) * C::Q + q];
        double dP[3][3];
        qp_dP(st, Hp, g.mu, g.lam, dP);
        const double sk = args.c_k * wq;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) A[(i * 4 + d) * C::Q + q] = sk * g.s[d] * dP[i][d];
        if (VAL) {
          const double sc = args.c_m * g.rho * wq;
#pragma unroll
          for (int i = 0; i < 3; ++i) A[(i * 4 + 3) * C::Q + q] *= sc;
        }
      }
    }
    group_sync<WPE>(gid);
    if (MODE == MODE_MASS)
      v2_backward<N, M, WPE, false, true>(tb, g, args.y, X0, Y0, Z0, A, Bf, t, gid);
    else if (MODE == MODE_FINT)
      v2_backward<N, M, WPE, true, false>(tb, g, args.y, X0, Y0, Z0, A, Bf, t, gid);
    else
      v2_backward<N, M, WPE, true, VAL>(tb, g, args.y, X0, Y0, Z0, A, Bf, t, gid);
  }
}

}  // namespace sdme
