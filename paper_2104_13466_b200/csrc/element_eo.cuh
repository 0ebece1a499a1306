// Even-odd (eo.cuh) overloads of the v3 contraction stages.  Selected by
// passing a TabEO table to element_v3; the schedule, shared layouts, staging
// and point work are the v3 ones -- only the 1D contractions change (about
// half the multiply-adds).  NC = 1 (component-serial, optionally with staged
// rows) or NC = 3 (all components per stage, small P).
#pragma once
#include "element_v3.cuh"
#include "eo.cuh"

namespace sdme {

template <int N, int M, int WPE, int NC, bool GRAD, bool VAL, bool STAGED = false, int MIR>
__device__ __forceinline__ void v3_forward(const TabEO<N, M, MIR>& tb0, int zv, const Geo& g, const double* __restrict__ src,
                                           int X0, int Y0, int Z0, double* A, double* B, int t, int gid,
                                           double* R = nullptr, int* buf = nullptr, NextRows next = {},
                                           BoxIO bx = {}) {
  static_assert(!STAGED || NC == 1, "row staging is per component");
  using C = V3<N, M, WPE, NC>;
  using Mr = Mir<N, MIR>;
  constexpr int NE = Mr::NE > 0 ? Mr::NE : 1, NO = Mr::NO > 0 ? Mr::NO : 1;
  double* const P = A;
#pragma unroll 1
  for (int c0 = 0; c0 < 3; c0 += NC) {
    // tables re-read from the constant bank per element / component group (OpArgs::zero)
    const auto& tb = reload_tab(tb0, N >= SDME_V3_RELOAD_MIN_N ? zv * (c0 + 1) : 0);
    double* const X = (NC == 3) ? A : B + C::YO;
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
    // x stage: item (comp, k, j)
    for (int w = t; w < NC * N * N; w += C::T) {
      int ck, j;
      C::item_x(w, ck, j);
      const int comp = c0 + ck / N, k = ck % N;
      double v[N];
      if (STAGED) {
        const double* row = R + *buf * N * N * N + (k * N + j) * N;
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = row[i];
      } else if (bx.in && N == 3 && BoxW<N>::BW == 4) {
        // P = 2 (shift 0): 32-byte box rows, one 16-byte and one 8-byte load
        const double* row = bx.in + comp * BoxW<N>::CB + (k * N + j) * 4;
        SDME_CHECK(smem_ok(row, 24, 16));
        const double2 d = *reinterpret_cast<const double2*>(row);
        v[0] = d.x;
        v[1 % N] = d.y;
        v[2 % N] = row[2];
      } else if (bx.in) {
        const double* row = bx.in + comp * BoxW<N>::CB + (k * N + j) * BoxW<N>::BW + bx.shift;
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = row[i];
      } else {
        const double* row = src + comp * g.Ns + ((long long)(Z0 + k) * g.Ly + (Y0 + j)) * g.Px + X0;
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = __ldg(row + i);
      }
      double E[NE], O[NO], o0[M], o1[M];
      eo_split<N, MIR>(v, E, O);
      eo_fwd<M, Mr::NE, Mr::NO>(tb.B, E, O, o0);
      if (GRAD) eo_fwd<M, Mr::NO, Mr::NE>(tb.Dx, O, E, o1);
#pragma unroll
      for (int a = 0; a < M; ++a) {
        X[C::xi(0, ck, j, a)] = o0[a];
        if (GRAD) X[C::xi(1, ck, j, a)] = o1[a];
      }
    }
    group_sync<WPE>(gid);
    // y stage: item (comp, k, a)
    for (int w = t; w < NC * N * M; w += C::T) {
      int ck, a;
      C::item_y(w, ck, a);
      const int cl = ck / N, k = ck % N;
      double x0[N], x1[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        x0[j] = X[C::xi(0, ck, j, a)];
        if (GRAD) x1[j] = X[C::xi(1, ck, j, a)];
      }
      double E0[NE], O0[NO], bb[M], db[M], bd[M];
      eo_split<N, MIR>(x0, E0, O0);
      eo_fwd<M, Mr::NE, Mr::NO>(tb.B, E0, O0, bb);
      if (GRAD) {
        double E1[NE], O1[NO];
        eo_split<N, MIR>(x1, E1, O1);
        eo_fwd<M, Mr::NO, Mr::NE>(tb.Dy, O0, E0, db);
        eo_fwd<M, Mr::NE, Mr::NO>(tb.B, E1, O1, bd);
      }
#pragma unroll
      for (int b = 0; b < M; ++b) {
        B[C::yi(cl, 0, k, b * M + a)] = bb[b];
        if (GRAD) {
          B[C::yi(cl, 1, k, b * M + a)] = db[b];
          B[C::yi(cl, 2, k, b * M + a)] = bd[b];
        }
      }
    }
    group_sync<WPE>(gid);
    // z stage: item (comp, b, a) -> points
    for (int w = t; w < NC * M * M; w += C::T) {
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
      double E0[NE], O0[NO];
      eo_split<N, MIR>(y0, E0, O0);
      if (GRAD) {
        double E1[NE], O1[NO], E2[NE], O2[NO], gx[M], gy[M], gz[M];
        eo_split<N, MIR>(y1, E1, O1);
        eo_split<N, MIR>(y2, E2, O2);
        eo_fwd<M, Mr::NE, Mr::NO>(tb.B, E2, O2, gx);
        eo_fwd<M, Mr::NE, Mr::NO>(tb.B, E1, O1, gy);
        eo_fwd<M, Mr::NO, Mr::NE>(tb.Dz, O0, E0, gz);
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const int q = c * M * M + ba;
          P[C::qi(0, comp, q)] = gx[c];
          P[C::qi(1, comp, q)] = gy[c];
          P[C::qi(2, comp, q)] = gz[c];
        }
      }
      if (VAL) {
        double vv[M];
        eo_fwd<M, Mr::NE, Mr::NO>(tb.B, E0, O0, vv);
#pragma unroll
        for (int c = 0; c < M; ++c) P[C::qi(3, comp, c * M * M + ba)] = vv[c];
      }
    }
    if (STAGED) *buf ^= 1;
    group_sync<WPE>(gid);
  }
}

template <int N, int M, int WPE, int NC, bool GRAD, bool VAL, int MIR>
__device__ __forceinline__ void v3_backward(const TabEO<N, M, MIR>& tb0, int zv, const Geo& g, double* __restrict__ dst,
                                            int X0, int Y0, int Z0, double* A, double* B, int t, int gid,
                                            double* evb = nullptr, BoxIO bx = {}) {
  using C = V3<N, M, WPE, NC>;
  using Mr = Mir<N, MIR>;
  constexpr int HP = Half<M>::HP, H = Half<M>::H > 0 ? Half<M>::H : 1;
  constexpr int BW = BoxW<N>::BW;
#pragma unroll 1
  for (int c0 = 0; c0 < 3; c0 += NC) {
    // tables re-read from the constant bank per element / component group (OpArgs::zero)
    const auto& tb = reload_tab(tb0, N >= SDME_V3_RELOAD_MIN_N ? zv * (c0 + 1) : 0);
    double* const X = (NC == 3) ? A : B + C::YO;
    // z' stage: item (comp, b, a), contract over c
    for (int w = t; w < NC * M * M; w += C::T) {
      const int cl = w / (M * M), ba = w % (M * M);
      const int comp = c0 + cl;
      double hx[N], hy[N], hz[N];
      if (GRAD) {
        double q[M], qe[HP], qo[H];
#pragma unroll
        for (int c = 0; c < M; ++c) q[c] = A[C::qi(0, comp, c * M * M + ba)];
        eo_qsplit<M>(q, qe, qo);
        eo_bwd<N, M, MIR, 1, Mr::NE, Mr::NO, false>(tb.bBz, qe, qo, hx);
#pragma unroll
        for (int c = 0; c < M; ++c) q[c] = A[C::qi(1, comp, c * M * M + ba)];
        eo_qsplit<M>(q, qe, qo);
        eo_bwd<N, M, MIR, 1, Mr::NE, Mr::NO, false>(tb.bBz, qe, qo, hy);
#pragma unroll
        for (int c = 0; c < M; ++c) q[c] = A[C::qi(2, comp, c * M * M + ba)];
        eo_qsplit<M>(q, qe, qo);
        eo_bwd<N, M, MIR, -1, Mr::NO, Mr::NE, false>(tb.bDz, qe, qo, hz);
      }
      if (VAL) {
        double q[M], qe[HP], qo[H];
#pragma unroll
        for (int c = 0; c < M; ++c) q[c] = A[C::qi(3, comp, c * M * M + ba)];
        eo_qsplit<M>(q, qe, qo);
        if (GRAD)
          eo_bwd<N, M, MIR, 1, Mr::NE, Mr::NO, true>(tb.bBz, qe, qo, hz);
        else
          eo_bwd<N, M, MIR, 1, Mr::NE, Mr::NO, false>(tb.bBz, qe, qo, hz);
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        if (GRAD) {
          B[C::yi(cl, 0, k, ba)] = hx[k];
          B[C::yi(cl, 1, k, ba)] = hy[k];
        }
        B[C::yi(cl, 2, k, ba)] = hz[k];
      }
    }
    group_sync<WPE>(gid);
    // y' stage: item (comp, k, a), contract over b
    for (int w = t; w < NC * N * M; w += C::T) {
      int ck, a;
      C::item_y(w, ck, a);
      const int cl = ck / N, k = ck % N;
      double jx[N], jyz[N];
      double q[M], qe[HP], qo[H];
      if (GRAD) {
#pragma unroll
        for (int b = 0; b < M; ++b) q[b] = B[C::yi(cl, 0, k, b * M + a)];
        eo_qsplit<M>(q, qe, qo);
        eo_bwd<N, M, MIR, 1, Mr::NE, Mr::NO, false>(tb.bBy, qe, qo, jx);
#pragma unroll
        for (int b = 0; b < M; ++b) q[b] = B[C::yi(cl, 1, k, b * M + a)];
        eo_qsplit<M>(q, qe, qo);
        eo_bwd<N, M, MIR, -1, Mr::NO, Mr::NE, false>(tb.bDy, qe, qo, jyz);
      }
#pragma unroll
      for (int b = 0; b < M; ++b) q[b] = B[C::yi(cl, 2, k, b * M + a)];
      eo_qsplit<M>(q, qe, qo);
      if (GRAD)
        eo_bwd<N, M, MIR, 1, Mr::NE, Mr::NO, true>(tb.bBy, qe, qo, jyz);
      else
        eo_bwd<N, M, MIR, 1, Mr::NE, Mr::NO, false>(tb.bBy, qe, qo, jyz);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        if (GRAD) X[C::xi(0, ck, j, a)] = jx[j];
        X[C::xi(1, ck, j, a)] = jyz[j];
      }
    }
    group_sync<WPE>(gid);
    // x' stage: item (comp, k, j), contract over a, RED into the lattice
    // (or into the output box of the TMA reduce-add)
    if (bx.out) {
      if (t == 0) bulk_wait_read();  // the previous element's reduce-adds have read the box
      group_sync<WPE>(gid);
    }
    for (int w = t; w < NC * N * N; w += C::T) {
      int ck, j;
      C::item_x(w, ck, j);
      const int comp = c0 + ck / N, k = ck % N;
      double acc[N];
      double q[M], qe[HP], qo[H];
      if (GRAD) {
#pragma unroll
        for (int a = 0; a < M; ++a) q[a] = X[C::xi(0, ck, j, a)];
        eo_qsplit<M>(q, qe, qo);
        eo_bwd<N, M, MIR, -1, Mr::NO, Mr::NE, false>(tb.bDx, qe, qo, acc);
      }
#pragma unroll
      for (int a = 0; a < M; ++a) q[a] = X[C::xi(1, ck, j, a)];
      eo_qsplit<M>(q, qe, qo);
      if (GRAD)
        eo_bwd<N, M, MIR, 1, Mr::NE, Mr::NO, true>(tb.bBx, qe, qo, acc);
      else
        eo_bwd<N, M, MIR, 1, Mr::NE, Mr::NO, false>(tb.bBx, qe, qo, acc);
      if (evb) {
        double* er = evb + ((comp * N + k) * N + j) * N;
#pragma unroll
        for (int i = 0; i < N; ++i) er[i] = acc[i];
        continue;
      }
      const int Z = Z0 + k, Y = Y0 + j;
      const bool chk = touches_dirichlet(g, comp, X0, Y0, Z0, N);
      if (bx.out) {
        // output box row: the element's N values at `shift`, zeros elsewhere
        // (slots outside the element belong to elements of other colours)
        double* orow = bx.out + comp * BoxW<N>::CB + (k * N + j) * BW;
        if constexpr (N == 3 && BW == 4) {
          // P = 2 (shift 0): the row as two 16-byte stores, pad slot 0
          double o[N];
#pragma unroll
          for (int i = 0; i < N; ++i) o[i] = (chk && constrained(g, comp, X0 + i, Y, Z)) ? 0.0 : acc[i];
          SDME_CHECK(smem_ok(orow, 32, 16));
          reinterpret_cast<double2*>(orow)[0] = make_double2(o[0], o[1]);
          reinterpret_cast<double2*>(orow)[1] = make_double2(o[2], 0.0);
          continue;
        }
#pragma unroll
        for (int i = 0; i < N; ++i) orow[bx.shift + i] = (chk && constrained(g, comp, X0 + i, Y, Z)) ? 0.0 : acc[i];
        if (BW - N == 1) {
          orow[N] = 0.0;
        } else {
          orow[N + 1] = 0.0;
          orow[bx.shift ? 0 : N] = 0.0;
        }
        continue;
      }
      SDME_CHECK(comp >= 0 && comp < 3 && Z >= 0 && Z < g.Lz && Y >= 0 && Y < g.Ly && X0 >= 0 && X0 + N <= g.Lx);
      double* row = dst + comp * g.Ns + ((long long)Z * g.Ly + Y) * g.Px + X0;
#pragma unroll
      for (int i = 0; i < N; ++i)
        if (!chk || !constrained(g, comp, X0 + i, Y, Z)) red_add(row + i, acc[i]);
    }
    if (bx.out) {
      fence_proxy_async_smem();
      group_sync<WPE>(gid);
      if (t == 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
          tma_reduce_add_box(static_cast<const CUtensorMap*>(bx.ymap), bx.out + c * BoxW<N>::CB, bx.xs, bx.Y0,
                             bx.Z0, c);
      }
    }
    group_sync<WPE>(gid);
  }
}

}  // namespace sdme
