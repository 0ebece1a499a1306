// Jacobi diagonal diag(c_k K_T(u) + c_m M) (solver.py:105-110 on the
// assembled operator), v3-style: one warp (or WPE warps) per element.
//
// For component i and local function f = (l, j, k) (lattice-local 1D indices)
//   D_i(f) = sum_q sum_{d,e} c_k (A^i_de + S_de)(q) dphi_f/dx_d dphi_f/dx_e
//            + c_m rho sum_q phi_f^2,
// A^i_de = lam (F C^-1)_id (F C^-1)_ie + (mu - lam ln J)
//          [(F C^-1 F^T)_ii C^-1_de + (F C^-1)_ie (F C^-1)_id]
// (the i-th diagonal block of the material + geometric tangent, material.py:84-105).
// Each symmetric pair (d, e) is one backward contraction with "squared" 1D
// tables per axis -- B^2, B D (x 2/h) or D^2 (x (2/h)^2), weights and det J
// folded in -- so the element's diagonal costs 6 chains per component
// (the mass term shares the (z, z) chain after its z' stage) instead of the
// dense element matrix.  grad u comes from the v3 forward pass.
#pragma once
#include "element_v3.cuh"

#ifndef SDME_DIAG_RELOAD
#define SDME_DIAG_RELOAD 1
#endif

namespace sdme {

template <int N, int M>
struct TabD {
  double x[3][M][N], y[3][M][N], z[3][M][N];  // [#derivatives along the axis][a][l]
};

// symmetric pairs (d, e): 0 (x,x) 1 (y,y) 2 (z,z) 3 (x,y) 4 (y,z) 5 (x,z)
__host__ __device__ constexpr int pair_d(int tt) { return tt < 3 ? tt : (tt == 4 ? 1 : 0); }
__host__ __device__ constexpr int pair_e(int tt) { return tt < 3 ? tt : (tt == 3 ? 1 : 2); }

// shared layout: 19 point slots (6 pair coefficients x 3 components + mass;
// grad u of the forward pass sits in the first 9 until the point stage
// overwrites it in place), then the v3 z'/y' scratch
template <int N, int M, int WPE>
struct DiagLay {
  using C = V3<N, M, WPE, 1, true>;
  static constexpr int SQ = C::Ly::sq;
  static constexpr int SA = 19 * SQ;
  static constexpr int PER = SA + C::SB;
};

template <int N, int M, int WPE, int EPB, int MINB>
__global__ void __launch_bounds__(EPB * WPE * 32, MINB) element_diag3(const __grid_constant__ Tab3<N, M> tb,
                                                                        const __grid_constant__ TabD<N, M> td0,
                                                                        const __grid_constant__ Geo g, OpArgs args) {
  using C = V3<N, M, WPE, 1, true>;
  using L = DiagLay<N, M, WPE>;
  constexpr int SQ = L::SQ;
  constexpr int NR = (N * N + C::T - 1) / C::T;  // x' rows per thread
  extern __shared__ double smem[];
  const int gid = threadIdx.x / C::T;
  const int t = threadIdx.x % C::T;
  double* A = smem + gid * L::PER;
  double* Bf = A + L::SA;  // z' output slab
  double* X = Bf + C::YO;  // y' output
  const long long cnt = colour_count(g, args.colour);
  const long long stride = (long long)gridDim.x * EPB;
  const bool stiff = args.c_k != 0.0;
  const double cmr = args.c_m * g.rho;
  int zit = 0;  // table re-reads (OpArgs::zero)
  for (long long idx = (long long)blockIdx.x * EPB + gid; idx < cnt; idx += stride) {
    const int zv = args.zero * (++zit);
    int ei, ej, ek;
    colour_element(g, args.colour, idx, ei, ej, ek);
    const int X0 = (N - 1) * ei, Y0 = (N - 1) * ej, Z0 = (N - 1) * ek;
    const long long eid = ((long long)ek * g.ny + ej) * g.nx + ei;
    if (stiff) v3_forward<N, M, WPE, 1, true, false>(tb, zv, g, args.u, X0, Y0, Z0, A, Bf, t, gid);
    // point coefficients: slot comp * 6 + pair, slot 18 mass
    for (int q = t; q < C::Q; q += C::T) {
      double coef[3][6];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int tt = 0; tt < 6; ++tt) coef[i][tt] = 0.0;
      if (stiff) {
        double H[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) H[i][d] = A[C::qi(d, i, q)];
        QpState st;
        qp_state(H, g.mu, g.lam, st);
        if (!(st.detF > 0.0)) {
          const int a = q % M, b = (q / M) % M, c = q / (M * M);
          atomicMin(args.inv_flag, (unsigned long long)eid * C::Q + (unsigned long long)((a * M + b) * M + c));
        }
        const double cc = g.mu - g.lam * st.lnJ;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          double FC[3];
#pragma unroll
          for (int d = 0; d < 3; ++d)
            FC[d] = st.F[i][0] * st.Ci[0][d] + st.F[i][1] * st.Ci[1][d] + st.F[i][2] * st.Ci[2][d];
          const double fcf = FC[0] * st.F[i][0] + FC[1] * st.F[i][1] + FC[2] * st.F[i][2];
#pragma unroll
          for (int tt = 0; tt < 6; ++tt) {
            const int d = pair_d(tt), e = pair_e(tt);
            const double Ade = g.lam * FC[d] * FC[e] + cc * (fcf * st.Ci[d][e] + FC[e] * FC[d]);
            coef[i][tt] = args.c_k * (d == e ? 1.0 : 2.0) * (Ade + st.S[d][e]);
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int tt = 0; tt < 6; ++tt) A[(i * 6 + tt) * SQ + q] = coef[i][tt];
      A[18 * SQ + q] = cmr;
    }
    group_sync<WPE>(gid);
#pragma unroll 1
    for (int comp = 0; comp < 3; ++comp) {
      double acc[NR][N];
#pragma unroll
      for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int i = 0; i < N; ++i) acc[r][i] = 0.0;
      // the six chains unrolled: their table choice (tx, ty, tz) is then a
      // compile-time offset (rolled, every multiply-add took an indexed LDC.64
      // for its table entry: 100 of the kernel's 452 DFMA sites)
      const TabD<N, M>& td = reload_tab(td0, SDME_DIAG_RELOAD ? zv * (comp + 1) : 0);
#pragma unroll
      for (int tt = 0; tt < 6; ++tt) {
        if (!stiff && tt != 2) continue;  // mass only: the (z, z) chain carries it
        const int d = pair_d(tt), e = pair_e(tt);
        const int tx = (d == 0) + (e == 0), ty = (d == 1) + (e == 1), tz = (d == 2) + (e == 2);
        const double* cf = A + (comp * 6 + tt) * SQ;
        const double* cm = A + 18 * SQ;
        // z' stage: column (b, a), contract over c (the mass term joins the (z, z) chain)
        for (int w = t; w < M * M; w += C::T) {
#pragma unroll
          for (int k = 0; k < N; ++k) {
            double h = 0.0;
#pragma unroll
            for (int c = 0; c < M; ++c) {
              h = fma(td.z[tz][c][k], cf[c * M * M + w], h);
              if (tt == 2) h = fma(td.z[0][c][k], cm[c * M * M + w], h);
            }
            Bf[C::yi(0, 0, k, w)] = h;
          }
        }
        group_sync<WPE>(gid);
        // y' stage: item (k, a), contract over b
        for (int w = t; w < N * M; w += C::T) {
          int ck, a;
          C::item_y(w, ck, a);
          double hv[M];
#pragma unroll
          for (int b = 0; b < M; ++b) hv[b] = Bf[C::yi(0, 0, ck, b * M + a)];
#pragma unroll
          for (int j = 0; j < N; ++j) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < M; ++b) s = fma(td.y[ty][b][j], hv[b], s);
            X[C::xi(0, ck, j, a)] = s;
          }
        }
        group_sync<WPE>(gid);
        // x' stage: item (k, j), contract over a, the chains accumulate in registers
#pragma unroll
        for (int r = 0; r < NR; ++r) {
          const int w = t + r * C::T;
          if (w >= N * N) continue;
          int ck, j;
          C::item_x(w, ck, j);
          double jv[M];
#pragma unroll
          for (int a = 0; a < M; ++a) jv[a] = X[C::xi(0, ck, j, a)];
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double s = acc[r][i];
#pragma unroll
            for (int a = 0; a < M; ++a) s = fma(td.x[tx][a][i], jv[a], s);
            acc[r][i] = s;
          }
        }
        group_sync<WPE>(gid);
      }
      // scatter this component's diagonal box
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int w = t + r * C::T;
        if (w >= N * N) continue;
        int ck, j;
        C::item_x(w, ck, j);
        const int k = ck;
        if (args.ev) {
          double* er = args.ev + (eid * 3 + comp) * (N * N * N) + (k * N + j) * N;
#pragma unroll
          for (int i = 0; i < N; ++i) er[i] = acc[r][i];
          continue;
        }
        const int Z = Z0 + k, Y = Y0 + j;
        SDME_CHECK(Z >= 0 && Z < g.Lz && Y >= 0 && Y < g.Ly && X0 >= 0 && X0 + N <= g.Lx);
        double* row = args.y + comp * g.Ns + ((long long)Z * g.Ly + Y) * g.Px + X0;
#pragma unroll
        for (int i = 0; i < N; ++i)
          if (!constrained(g, comp, X0 + i, Y, Z)) red_add(row + i, acc[r][i]);
      }
    }
  }
}

}  // namespace sdme
