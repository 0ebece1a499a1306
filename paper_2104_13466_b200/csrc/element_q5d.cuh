// Jacobi diagonal at P = 4 (n = m = 5) on the quintet schedule of element_q5.cuh:
// diag(c_k K_T(u) + c_m M), five elements per 4-warp CTA, TMA boxes in, bulk
// tensor reduce-add out (solver.py:105-110 of the reference builds the same
// diagonal from the assembled matrix).
//
//   diag[comp][k, j, i] = sum_pairs (d, e) sum_points (c, b, a)
//        coef[comp][(d, e)](c, b, a)  Tz^{tz}[c][k]  Ty^{ty}[b][j]  Tx^{tx}[a][i]
//
// with the squared tables T^0 = w B.B, T^1 = w B.D, T^2 = w D.D of TabD
// (element_diag.cuh; t. = how many of d, e lie along the axis).  The point
// coefficient is the (i d, i e) entry of the tangent moduli; with K = F^-T,
//   coef[i][(d, e)] = c_k m_de (mu delta_de + (lam + mu - lam ln J) K_id K_ie),
// m_de = 1 (d = e) or 2: element_diag3's expression (lam FC_d FC_e + cc (fcf
// C^-1_de + FC_e FC_d) + S_de, FC = F C^-1, fcf = FC . F_i) reduces to it since
// F C^-1 = F^-T, fcf = 1 and the C^-1 terms of cc and S cancel (dP of
// material.py:84-105 applied to the one-row gradient e_i (x) g).  So a point
// stores K (9 values, over grad u) and kappa = c_k (lam + mu - lam ln J).
// Schedule per quintet:
//   * grad u at the points by q5_forward (collocated, element_q5.cuh) into
//     point slots 0..8;
//   * point stage: the thread's points t + 128 r -> K in place, kappa;
//   * per component i: the column threads load K_i. and kappa of their five
//     points once, then six z' stages (one per pair, coefficients formed in
//     registers) ping-pong two stage arrays, the y' stage of each pair
//     accumulates its output into three register groups by x table (tx = 0:
//     (y,y), (z,z), (y,z); 1: (x,y), (x,z); 2: (x,x)), then one x' stage
//     contracts the three groups into the rows of the output box: 6 + 6 + 1
//     stage passes instead of 18.
// Shared memory: 9 slots x 625 doubles + three stage arrays + the output boxes
// + kappa = 73 KB, three CTAs per SM.  The two TMA staging buffers of the
// forward pass are the output boxes and the kappa array (idle until the point
// stage), so the first box of a quintet is fetched at its start, after the
// previous quintet's reduce-adds have read the output boxes.
// Lane orders and array layouts are those of element_q5.cuh (conflict-free).
#pragma once
#include "element_diag.cuh"
#include "element_q5.cuh"

namespace sdme {

struct Q5DLay {
  static constexpr int N = 5, E = 5, Q = 125, EQ = E * Q;
  static constexpr int NSLOT = 9;
  static constexpr int X = NSLOT * EQ, Y = X + EQ, U = Y + EQ;
  static constexpr int RP = BoxW<N>::BW, RB = BoxW<N>::CB;
  static constexpr int O = (U + EQ + 15) / 16 * 16;  // output boxes [e][RB] = staging buffer 0
  static constexpr int KP = O + E * RB;              // kappa [e][q] (+ pad) = staging buffer 1
  static constexpr int R = O;                        // staging [2][e][RB]
  static constexpr int BAR = R + 2 * E * RB;
  static constexpr int COORD = BAR + 2;              // int [e][4]: X0, Y0, Z0, ghost
  static constexpr int PER = COORD + (E * 4 + 1) / 2;
  static constexpr unsigned BOXBYTES = N * N * RP * 8;
  static_assert(EQ <= E * RB, "kappa must fit the second staging buffer");
  __device__ static int slot(int d, int comp) { return (d * 3 + comp) * EQ; }  // grad u, then K[comp][d]
  __device__ static int vslot(int) { return 0; }                               // (no value slots)
};

template <int MINB, int MIR, bool ISO>
__global__ void __launch_bounds__(128, MINB) element_q5_diag(const __grid_constant__ TabC<5, MIR> tb,
                                                             const __grid_constant__ TabD<5, 5> td0,
                                                             const __grid_constant__ Geo g, OpArgs args) {
  constexpr int N = 5, Q = 125, T = 128;
  using L = Q5DLay;
  constexpr int QPT = (L::EQ + T - 1) / T;
  extern __shared__ __align__(128) double S[];
  const int t = threadIdx.x;
  const int zoff = args.zero;
  SDME_CHECK(smem_ok(S, L::PER * 8, 128));
  const bool act = t < L::EQ / N;
  const int tt0 = act ? t : 0;
  const int o5 = 5 * tt0;
  const int o_row = (tt0 / 25) * L::RB + (tt0 % 25) * L::RP;
  const int o_y = 125 * ((tt0 / 5) % 5) + 25 * (tt0 % 5) + tt0 / 25;
  const int o_z = 125 * (tt0 % 5) + 5 * (tt0 / 25) + (tt0 / 5) % 5;
  const long long cnt = colour_count(g, args.colour);
  const long long nq = (cnt + L::E - 1) / L::E;
  const double cmr = args.c_m * g.rho;
  const CUtensorMap* umap = static_cast<const CUtensorMap*>(args.tu);
  const CUtensorMap* ymap = static_cast<const CUtensorMap*>(args.ty);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(S + L::BAR);
  int* coord = reinterpret_cast<int*>(S + L::COORD);
  unsigned ph = 0;
  int buf = 0;
  if (t == 0) {
    mbar_init(bars, L::E);
    mbar_init(bars + 1, L::E);
    mbar_fence_init();
  }
  __syncthreads();
  for (long long qd = blockIdx.x; qd < nq; qd += gridDim.x) {
    // this quintet's elements and their first boxes (the staging buffers were
    // the output boxes and kappa of the previous quintet: its reduce-adds have
    // read the boxes, generic writes precede the async-proxy box loads)
    fence_proxy_async_smem();
    __syncthreads();
    if (t < L::E) {
      bulk_wait_read();
      const long long idx = qd * L::E + t;
      int ei, ej, ek;
      colour_element(g, args.colour, idx < cnt ? idx : cnt - 1, ei, ej, ek);
      int* cc = coord + t * 4;
      cc[0] = (N - 1) * ei, cc[1] = (N - 1) * ej, cc[2] = (N - 1) * ek, cc[3] = idx >= cnt;
      mbar_expect_tx(bars + buf, L::BOXBYTES);
      tma_load_box(S + L::R + (buf * L::E + t) * L::RB, umap, cc[0], cc[1], cc[2], 0, bars + buf);
    }
    __syncthreads();  // coord visible
    q5_forward<L, MIR, false, ISO>(tb, zoff, S, t, act, o_row, o5, o_y, o_z, &buf, &ph, umap, 0, Q5Next{nullptr, 0},
                                   true, false);
    // point stage: grad u -> K = F^-T in place, kappa = c_k (lam + mu - lam ln J)
    const double lm = args.c_k * (g.lam + g.mu), cl = args.c_k * g.lam, cmu = args.c_k * g.mu;
#pragma unroll 1
    for (int r = 0; r < QPT; ++r) {
      const int pid = t + r * T;
      if (pid >= L::EQ) continue;
      double H[9];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int d = 0; d < 3; ++d) H[i * 3 + d] = S[L::slot(d, i) + pid];
      QpK st;
      qp_k(H, st);
      if (!(st.det > 0.0)) {
        const int e = pid / Q, q = pid - e * Q;
        const int* cc = coord + e * 4;
        const long long eid = ((long long)(cc[2] / (N - 1)) * g.ny + cc[1] / (N - 1)) * g.nx + cc[0] / (N - 1);
        const int a = q % N, b = (q / N) % N, c = q / (N * N);
        atomicMin(args.inv_flag, (unsigned long long)eid * Q + (unsigned long long)((a * N + b) * N + c));
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int d = 0; d < 3; ++d) S[L::slot(d, i) + pid] = st.K[i][d];
      S[L::KP + pid] = fma(-cl, st.lnJ, lm);
    }
    __syncthreads();
#pragma unroll 1
    for (int comp = 0; comp < 3; ++comp) {
      const TabD<5, 5>& td = reload_tab(td0, zoff * (comp + 1));
      // K[comp][.] and kappa at the column thread's five points
      double Kc[3][N], kp[N];
#pragma unroll
      for (int c = 0; c < N; ++c) {
#pragma unroll
        for (int d = 0; d < 3; ++d) Kc[d][c] = S[L::slot(d, comp) + o_z + 25 * c];
        kp[c] = S[L::KP + o_z + 25 * c];
      }
      double XG[3][N];  // y' outputs of this thread's item (e; k, a), grouped by x table
#pragma unroll
      for (int gq = 0; gq < 3; ++gq)
#pragma unroll
        for (int j = 0; j < N; ++j) XG[gq][j] = 0.0;
#pragma unroll
      for (int tt = 0; tt < 6; ++tt) {
        const int d = pair_d(tt), e2 = pair_e(tt);
        const int tx = (d == 0) + (e2 == 0), ty = (d == 1) + (e2 == 1), tz = (d == 2) + (e2 == 2);
        double* Yb = S + ((tt & 1) ? L::U : L::Y);
        // z' stage: column (e; b, a), contract over the points c (the mass
        // term joins the (z, z) chain: its tables are T^0 on every axis)
        if (act) {
          double cf[N];
#pragma unroll
          for (int c = 0; c < N; ++c)
            cf[c] = d == e2 ? fma(kp[c] * Kc[d][c], Kc[e2][c], cmu) : 2.0 * (kp[c] * Kc[d][c] * Kc[e2][c]);
#pragma unroll
          for (int k = 0; k < N; ++k) {
            double h = 0.0;
#pragma unroll
            for (int c = 0; c < N; ++c) {
              h = fma(td.z[tz][c][k], cf[c], h);
              if (tt == 2) h = fma(td.z[0][c][k], cmr, h);
            }
            Yb[o_z + 25 * k] = h;
          }
        }
        __syncthreads();
        // y' stage: item (e; k, a), contract over b into the thread's group
        if (act) {
          double hv[N];
#pragma unroll
          for (int b = 0; b < N; ++b) hv[b] = Yb[o_y + 5 * b];
#pragma unroll
          for (int j = 0; j < N; ++j) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < N; ++b) s = fma(td.y[ty][b][j], hv[b], s);
            XG[tx][j] += s;
          }
        }
      }
      __syncthreads();  // the last y' stages have read Y and U
      if (act) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          S[L::X + o_y + 5 * j] = XG[0][j];
          S[L::Y + o_y + 5 * j] = XG[1][j];
          S[L::U + o_y + 5 * j] = XG[2][j];
        }
      }
      // the previous component's reduce-adds have read the output boxes
      if (t < L::E) bulk_wait_read();
      __syncthreads();
      // x' stage: item (e; k, j), contract over a -> row of the output box;
      // constrained points and the pitch slot get 0 (as element_q5)
      if (act) {
        double acc[N];
#pragma unroll
        for (int i = 0; i < N; ++i) acc[i] = 0.0;
#pragma unroll
        for (int gq = 0; gq < 3; ++gq) {
          double jv[N];
          const int base = gq == 0 ? L::X : (gq == 1 ? L::Y : L::U);
#pragma unroll
          for (int a = 0; a < N; ++a) jv[a] = S[base + o5 + a];
#pragma unroll
          for (int i = 0; i < N; ++i)
#pragma unroll
            for (int a = 0; a < N; ++a) acc[i] = fma(td.x[gq][a][i], jv[a], acc[i]);
        }
        if (g.dmask[comp]) {
          const int e = t / 25, w = t - 25 * e;
          const int* cc = coord + e * 4;
          const int X0 = cc[0], Y0 = cc[1], Z0 = cc[2];
          if (touches_dirichlet(g, comp, X0, Y0, Z0, N)) {
            const int Z = Z0 + w / N, Yc = Y0 + w % N;
#pragma unroll
            for (int i = 0; i < N; ++i)
              if (constrained(g, comp, X0 + i, Yc, Z)) acc[i] = 0.0;
          }
        }
        double2* orow = reinterpret_cast<double2*>(S + L::O + o_row);
        SDME_CHECK(smem_ok(orow, L::RP * 8, 16));
#pragma unroll
        for (int i = 0; i < L::RP / 2; ++i) orow[i] = make_double2(acc[2 * i], 2 * i + 1 < N ? acc[2 * i + 1] : 0.0);
      }
      fence_proxy_async_smem();
      __syncthreads();
      if (t < L::E && ymap) {
        const int* cc = coord + t * 4;
        if (!cc[3]) tma_reduce_add_box(ymap, S + L::O + t * L::RB, cc[0], cc[1], cc[2], comp);
      }
    }
  }
  if (t < L::E) bulk_wait_all();
}

}  // namespace sdme
