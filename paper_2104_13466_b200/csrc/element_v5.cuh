// element_v5: K(u).p with the p field's z stage, the point work and the
// backward z' stage fused per (b, a) quadrature column, in registers.
//
// v3 (component-serial, even-odd) moves, per element and per component, the
// p gradient at the points through shared memory (z stage writes 3 x M^3,
// point stage reads 9 x M^3 and writes the 9 x M^3 flux, z' stage reads it
// back).  Here the thread that owns column (b, a) keeps grad p of its M points
// for all three components in registers (hp[comp][dir][c]), computes the
// linearised stress at those points (grad u is read from shared memory, where
// the u pass left it) and accumulates the flux straight into the even / odd
// partial sums of the z' contraction.  Shared-memory traffic of those three
// steps disappears; the arithmetic and its order are v3's, so results are
// bit-identical to the v3 even-odd kernel.
//
// Requires the even-odd tables (eo.cuh) and one warp per element with
// M * M <= 32 (P <= 4 at m = P + 1).
#pragma once
#include "element_eo.cuh"

namespace sdme {

// p forward (component-serial, staged rows) with the z-stage output kept in
// registers: hp[comp][d][c] = d/dx_d p_comp at point (c, b, a) of column t,
// vv[comp][c] = p_comp (VAL).
template <int N, int M, bool VAL, int MIR>
__device__ __forceinline__ void v5_forward_p(const TabEO<N, M, MIR>& tb, const Geo& g, const double* __restrict__ src,
                                             int X0, int Y0, int Z0, double* B, int t, double* R, int* buf,
                                             NextRows next, double (&hp)[3][3][M], double (&vv)[3][M]) {
  using C = V3<N, M, 1, 1, false>;
  using Mr = Mir<N, MIR>;
  constexpr int NE = Mr::NE > 0 ? Mr::NE : 1, NO = Mr::NO > 0 ? Mr::NO : 1;
  double* const X = B + C::YO;
#pragma unroll
  for (int c0 = 0; c0 < 3; ++c0) {
    {
      double* nb = R + (*buf ^ 1) * N * N * N;
      if (c0 + 1 < 3) {
        v3_stage_rows<N, 32>(g, src, c0 + 1, X0, Y0, Z0, nb, t);
        cp_async_wait<1>();
      } else if (next.field) {
        v3_stage_rows<N, 32>(g, next.field, 0, next.X0, next.Y0, next.Z0, nb, t);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
    }
    // x stage: item (k, j)
    for (int w = t; w < N * N; w += 32) {
      int ck, j;
      C::item_x(w, ck, j);
      const int k = ck;
      const double* row = R + *buf * N * N * N + (k * N + j) * N;
      double v[N];
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = row[i];
      double E[NE], O[NO], o0[M], o1[M];
      eo_split<N, MIR>(v, E, O);
      eo_fwd<M, Mr::NE, Mr::NO>(tb.B, E, O, o0);
      eo_fwd<M, Mr::NO, Mr::NE>(tb.Dx, O, E, o1);
#pragma unroll
      for (int a = 0; a < M; ++a) {
        X[C::xi(0, ck, j, a)] = o0[a];
        X[C::xi(1, ck, j, a)] = o1[a];
      }
    }
    __syncwarp();
    // y stage: item (k, a)
    for (int w = t; w < N * M; w += 32) {
      int ck, a;
      C::item_y(w, ck, a);
      const int k = ck;
      double x0[N], x1[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        x0[j] = X[C::xi(0, ck, j, a)];
        x1[j] = X[C::xi(1, ck, j, a)];
      }
      double E0[NE], O0[NO], E1[NE], O1[NO], bb[M], db[M], bd[M];
      eo_split<N, MIR>(x0, E0, O0);
      eo_split<N, MIR>(x1, E1, O1);
      eo_fwd<M, Mr::NE, Mr::NO>(tb.B, E0, O0, bb);
      eo_fwd<M, Mr::NO, Mr::NE>(tb.Dy, O0, E0, db);
      eo_fwd<M, Mr::NE, Mr::NO>(tb.B, E1, O1, bd);
#pragma unroll
      for (int b = 0; b < M; ++b) {
        B[C::yi(0, 0, k, b * M + a)] = bb[b];
        B[C::yi(0, 1, k, b * M + a)] = db[b];
        B[C::yi(0, 2, k, b * M + a)] = bd[b];
      }
    }
    __syncwarp();
    // z stage: column (b, a) = t, into registers
    if (t < M * M) {
      double y0[N], y1[N], y2[N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        y0[k] = B[C::yi(0, 0, k, t)];
        y1[k] = B[C::yi(0, 1, k, t)];
        y2[k] = B[C::yi(0, 2, k, t)];
      }
      double E0[NE], O0[NO], E1[NE], O1[NO], E2[NE], O2[NO];
      eo_split<N, MIR>(y0, E0, O0);
      eo_split<N, MIR>(y1, E1, O1);
      eo_split<N, MIR>(y2, E2, O2);
      eo_fwd<M, Mr::NE, Mr::NO>(tb.B, E2, O2, hp[c0][0]);
      eo_fwd<M, Mr::NE, Mr::NO>(tb.B, E1, O1, hp[c0][1]);
      eo_fwd<M, Mr::NO, Mr::NE>(tb.Dz, O0, E0, hp[c0][2]);
      if (VAL) eo_fwd<M, Mr::NE, Mr::NO>(tb.B, E0, O0, vv[c0]);
    }
    *buf ^= 1;
    __syncwarp();
  }
}

// Point work + z' contraction of column t.  grad u at the points is read from
// A (slots qi(d, i, q)); the z' results of all three components are written
// to Y3 = A in the component-major Y layout (yi(comp, s, k, ba)).
template <int N, int M, bool VAL, int MIR>
__device__ __forceinline__ void v5_points(const TabEO<N, M, MIR>& tb, const Geo& g, double* A, int t,
                                          const double (&hp)[3][3][M], const double (&vv)[3][M], double mu_k,
                                          double lam_k, double cmr, long long eid, unsigned long long* inv_flag) {
  using C = V3<N, M, 1, 1, false>;
  using Mr = Mir<N, MIR>;
  constexpr int NE = Mr::NE, NO = Mr::NO;
  constexpr int H = Half<M>::H, HP = Half<M>::HP;
  constexpr int W = NE > NO ? NE : NO;
  constexpr int Q = M * M * M;
  double YE[3][3][W], YO[3][3][W], VE[3][W], VO[3][W];
  if (t < M * M) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int e = 0; e < W; ++e) {
#pragma unroll
        for (int d = 0; d < 3; ++d) YE[i][d][e] = YO[i][d][e] = 0.0;
        VE[i][e] = VO[i][e] = 0.0;
      }
#pragma unroll
    for (int a = 0; a < HP; ++a) {
      const bool pair = a < H;
      double f[2][3][3];
#pragma unroll
      for (int side = 0; side < 2; ++side) {
        if (side == 1 && !pair) continue;
        const int c = side == 0 ? a : M - 1 - a;
        const int q = c * M * M + t;
        double Hu[9];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) Hu[i * 3 + d] = A[C::qi(d, i, q)];
        QpK s;
        qp_k(Hu, s);
        if (!(s.det > 0.0)) {
          const int aa = t % M, bb = t / M;
          atomicMin(inv_flag, (unsigned long long)eid * Q + (unsigned long long)((aa * M + bb) * M + c));
        }
        double tr = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) tr = fma(s.K[i][d], hp[i][d][c], tr);
        double M1[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j)
            M1[i][j] = fma(s.K[i][0], hp[j][0][c], fma(s.K[i][1], hp[j][1][c], s.K[i][2] * hp[j][2][c]));
        const double cc = mu_k - lam_k * s.lnJ;
        const double lt = lam_k * tr;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const double m2 = fma(M1[i][0], s.K[0][d], fma(M1[i][1], s.K[1][d], M1[i][2] * s.K[2][d]));
            f[side][i][d] = fma(cc, m2, fma(lt, s.K[i][d], mu_k * hp[i][d][c]));
          }
      }
      // even / odd point-side combinations, accumulated into the z' sums
#pragma unroll
      for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double qe = pair ? f[0][i][d] + f[1][i][d] : f[0][i][d];
          const double qo = pair ? f[0][i][d] - f[1][i][d] : 0.0;
          if (d < 2) {
#pragma unroll
            for (int e = 0; e < NE; ++e) YE[i][d][e] = fma(tb.bBz.E[e][a], qe, YE[i][d][e]);
            if (pair) {
#pragma unroll
              for (int o = 0; o < NO; ++o) YO[i][d][o] = fma(tb.bBz.O[o][a], qo, YO[i][d][o]);
            }
          } else {
#pragma unroll
            for (int e = 0; e < NO; ++e) YE[i][d][e] = fma(tb.bDz.E[e][a], qe, YE[i][d][e]);
            if (pair) {
#pragma unroll
              for (int o = 0; o < NE; ++o) YO[i][d][o] = fma(tb.bDz.O[o][a], qo, YO[i][d][o]);
            }
          }
        }
        if (VAL) {
          const int c0 = a, c1 = M - 1 - a;
          const double v0 = cmr * vv[i][c0];
          const double v1 = pair ? cmr * vv[i][c1] : 0.0;
          const double qe = pair ? v0 + v1 : v0;
          const double qo = v0 - v1;
#pragma unroll
          for (int e = 0; e < NE; ++e) VE[i][e] = fma(tb.bBz.E[e][a], qe, VE[i][e]);
          if (pair) {
#pragma unroll
            for (int o = 0; o < NO; ++o) VO[i][o] = fma(tb.bBz.O[o][a], qo, VO[i][o]);
          }
        }
      }
    }
  }
  __syncwarp();  // every lane is done reading grad u before Y3 overwrites A
  if (t < M * M) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double hx[N], hy[N], hz[N];
      eo_recon<N, MIR, 1, NE, NO, false>(YE[i][0], YO[i][0], hx);
      eo_recon<N, MIR, 1, NE, NO, false>(YE[i][1], YO[i][1], hy);
      eo_recon<N, MIR, -1, NO, NE, false>(YE[i][2], YO[i][2], hz);
      if (VAL) eo_recon<N, MIR, 1, NE, NO, true>(VE[i], VO[i], hz);
#pragma unroll
      for (int k = 0; k < N; ++k) {
        A[C::yi(i, 0, k, t)] = hx[k];
        A[C::yi(i, 1, k, t)] = hy[k];
        A[C::yi(i, 2, k, t)] = hz[k];
      }
    }
  }
  __syncwarp();
}

// y' and x' stages of the three components from the Y3 layout in A; RED into
// the lattice (or the E-vector box evb).
template <int N, int M, int MIR>
__device__ __forceinline__ void v5_backward_yx(const TabEO<N, M, MIR>& tb, const Geo& g, double* __restrict__ dst,
                                               int X0, int Y0, int Z0, const double* Y3, double* X, int t,
                                               double* evb) {
  using C = V3<N, M, 1, 1, false>;
  using Mr = Mir<N, MIR>;
  constexpr int HP = Half<M>::HP, H = Half<M>::H > 0 ? Half<M>::H : 1;
#pragma unroll 1
  for (int comp = 0; comp < 3; ++comp) {
    // y' stage: item (k, a), contract over b
    for (int w = t; w < N * M; w += 32) {
      int ck, a;
      C::item_y(w, ck, a);
      const int k = ck;
      double jx[N], jyz[N];
      double q[M], qe[HP], qo[H];
#pragma unroll
      for (int b = 0; b < M; ++b) q[b] = Y3[C::yi(comp, 0, k, b * M + a)];
      eo_qsplit<M>(q, qe, qo);
      eo_bwd<N, M, MIR, 1, Mr::NE, Mr::NO, false>(tb.bBy, qe, qo, jx);
#pragma unroll
      for (int b = 0; b < M; ++b) q[b] = Y3[C::yi(comp, 1, k, b * M + a)];
      eo_qsplit<M>(q, qe, qo);
      eo_bwd<N, M, MIR, -1, Mr::NO, Mr::NE, false>(tb.bDy, qe, qo, jyz);
#pragma unroll
      for (int b = 0; b < M; ++b) q[b] = Y3[C::yi(comp, 2, k, b * M + a)];
      eo_qsplit<M>(q, qe, qo);
      eo_bwd<N, M, MIR, 1, Mr::NE, Mr::NO, true>(tb.bBy, qe, qo, jyz);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        X[C::xi(0, ck, j, a)] = jx[j];
        X[C::xi(1, ck, j, a)] = jyz[j];
      }
    }
    __syncwarp();
    // x' stage: item (k, j), contract over a, RED into the lattice
    for (int w = t; w < N * N; w += 32) {
      int ck, j;
      C::item_x(w, ck, j);
      const int k = ck;
      double acc[N];
      double q[M], qe[HP], qo[H];
#pragma unroll
      for (int a = 0; a < M; ++a) q[a] = X[C::xi(0, ck, j, a)];
      eo_qsplit<M>(q, qe, qo);
      eo_bwd<N, M, MIR, -1, Mr::NO, Mr::NE, false>(tb.bDx, qe, qo, acc);
#pragma unroll
      for (int a = 0; a < M; ++a) q[a] = X[C::xi(1, ck, j, a)];
      eo_qsplit<M>(q, qe, qo);
      eo_bwd<N, M, MIR, 1, Mr::NE, Mr::NO, true>(tb.bBx, qe, qo, acc);
      if (evb) {
        double* er = evb + ((comp * N + k) * N + j) * N;
#pragma unroll
        for (int i = 0; i < N; ++i) er[i] = acc[i];
        continue;
      }
      const int Z = Z0 + k, Y = Y0 + j;
      const bool chk = touches_dirichlet(g, comp, X0, Y0, Z0, N);
      double* row = dst + comp * g.Ns + ((long long)Z * g.Ly + Y) * g.Px + X0;
#pragma unroll
      for (int i = 0; i < N; ++i)
        if (!chk || !constrained(g, comp, X0 + i, Y, Z)) red_add(row + i, acc[i]);
    }
    __syncwarp();
  }
}

// K(u).p (+ c_m M p when VAL): one warp per element, persistent over the
// elements of a colour pass (or all elements in E-vector mode).
template <int N, int M, int MINB, bool VAL, int MIR>
__global__ void __launch_bounds__(32, MINB) element_v5(const __grid_constant__ TabEO<N, M, MIR> tb,
                                                       const __grid_constant__ Geo g, OpArgs args) {
  using C = V3<N, M, 1, 1, false>;
  static_assert(M * M <= 32, "one column per lane");
  static_assert(9 * C::YS <= C::SA + C::YO, "Y3 must fit below the x-stage scratch");
  constexpr int PERS = C::PER + 2 * N * N * N;
  extern __shared__ double smem[];
  const int t = threadIdx.x;
  double* A = smem;
  double* Bf = A + C::SA;
  double* Rb = A + C::PER;
  int buf = 0;
  (void)PERS;
  if (args.skip && *(volatile const int*)args.skip) return;
  const long long cnt = colour_count(g, args.colour);
  const long long stride = gridDim.x;
  const double mu_k = args.c_k * g.mu, lam_k = args.c_k * g.lam;
  const double cmr = args.c_m * g.rho;
  if ((long long)blockIdx.x < cnt) {
    int ei, ej, ek;
    colour_element(g, args.colour, blockIdx.x, ei, ej, ek);
    v3_stage_rows<N, 32>(g, args.u, 0, (N - 1) * ei, (N - 1) * ej, (N - 1) * ek, Rb, t);
  }
  for (long long idx = blockIdx.x; idx < cnt; idx += stride) {
    int ei, ej, ek;
    colour_element(g, args.colour, idx, ei, ej, ek);
    const int X0 = (N - 1) * ei, Y0 = (N - 1) * ej, Z0 = (N - 1) * ek;
    NextRows nxt{nullptr, 0, 0, 0};
    if (idx + stride < cnt) {
      int ni, nj, nk;
      colour_element(g, args.colour, idx + stride, ni, nj, nk);
      nxt = NextRows{args.u, (N - 1) * ni, (N - 1) * nj, (N - 1) * nk};
    }
    // grad u -> A (points), p rows staged meanwhile
    v3_forward<N, M, 1, 1, true, false, true>(tb, g, args.u, X0, Y0, Z0, A, Bf, t, 0, Rb, &buf,
                                              NextRows{args.p, X0, Y0, Z0});
    double hp[3][3][M], vv[3][M];
    v5_forward_p<N, M, VAL, MIR>(tb, g, args.p, X0, Y0, Z0, Bf, t, Rb, &buf, nxt, hp, vv);
    const long long eid = ((long long)ek * g.ny + ej) * g.nx + ei;
    v5_points<N, M, VAL, MIR>(tb, g, A, t, hp, vv, mu_k, lam_k, cmr, eid, args.inv_flag);
    double* evb = args.ev ? args.ev + eid * 3 * (N * N * N) : nullptr;
    v5_backward_yx<N, M, MIR>(tb, g, args.y, X0, Y0, Z0, A, Bf + C::YO, t, evb);
  }
}

}  // namespace sdme
