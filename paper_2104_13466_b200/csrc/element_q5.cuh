// P = 4 (n = m = 5) collocated element kernel, five elements per 4-warp CTA.
//
// The warp-per-element kernel (element_col.cuh) runs every 1D stage of an
// element on 25 of a warp's 32 lanes: each 64-bit shared access then costs two
// wavefronts for 25 words (78% of the data pipe's width) and 22% of every
// FP64 issue slot is idle.  Here a CTA of 128 threads owns a *quintet* of
// elements: a stage has 5 x 25 = 125 pencils on 128 lanes (98%).
//
// Shared layout.  Every stage array of the quintet is the dense 5^4 array
// [e][.][.][.] (element-major, the natural per-element [k][j][a] order, no
// padding).  Its four strides 1, 5, 25, 125 are 5^0..5^3 = 1, 5, 9, 13 mod 16.
// A pencil access fixes one coordinate (the loop index) and spreads the
// other three over the lanes; whichever three strides remain, they are
// alpha * {1, 5, 25} mod 16 for alpha = the stride that follows the missing
// one in the cycle 1 -> 5 -> 9 -> 13 -> 1.  With the lanes ordered
// t = 25 x + 5 y + z, (z, y, x) the coordinates of strides (alpha, 5 alpha,
// 25 alpha), the address is alpha * t + const (mod 16), and alpha is odd: any 16
// consecutive lanes hit 16 distinct 8-byte banks.  So every stage is free of
// bank conflicts in all three pencil directions -- which no layout of a single
// 5^3 element achieves ("structural" conflicts) -- at 8 wavefronts
// per 125-lane access.  The lane orders that follow:
//   x stage, x pencils of the points:  t = 25 e + 5 k + j   (natural)
//   y stage, y pencils of the points:  t = 25 a + 5 e + k
//   z stage:                           t = 25 b + 5 a + e
// The point work runs on pid = t + 128 r over the 625 points in array order.
//
// Boxes come and go by TMA as in element_col (one box per element and
// component, loads by lanes 0..4 on one mbarrier per staging buffer, results
// by bulk tensor reduce-add); the output boxes reuse the staging buffer that
// is idle during the backward pass.  Arithmetic per pencil and per point is
// that of element_col, so results are bit-identical to it.
#pragma once
#include "element_col.cuh"

namespace sdme {

template <int MODE, bool VAL>
struct Q5Lay {
  static constexpr int N = 5, E = 5, Q = 125, EQ = E * Q;
  static constexpr bool GRAD = MODE != MODE_MASS;
  static constexpr int VB = GRAD ? 9 : 0;                    // first value slot
  static constexpr int NSLOT = VB + (VAL ? 3 : 0);           // point slots [slot][e][q]
  static constexpr int X = NSLOT * EQ;                       // [e][k][j][a]
  static constexpr int Y = X + EQ;                           // [e][k][b][a]
  static constexpr int U = Y + EQ;                           // [e][c][b][a]
  static constexpr int W = U + EQ;                           // w_a w_b w_c det J, [q]
  static constexpr int RP = BoxW<N>::BW;                     // box row pitch (6)
  static constexpr int RB = BoxW<N>::CB;                     // one element's box, 128-B multiple (160)
  static constexpr int R = (W + Q + 15) / 16 * 16;           // staging buffers [2][e][RB]
  static constexpr int BAR = R + 2 * E * RB;                 // two mbarriers
  static constexpr int COORD = BAR + 2;                      // int [2][e][4]: X0, Y0, Z0, ghost
  static constexpr int PER = COORD + (2 * E * 4 + 1) / 2;
  static constexpr unsigned BOXBYTES = N * N * RP * 8;
  __device__ static int slot(int d, int comp) { return (d * 3 + comp) * EQ; }
  __device__ static int vslot(int comp) { return (VB + comp) * EQ; }
};

// which element coordinates a lane 0..4 stages next (coordinate set of the
// quintet table) and from which tensor map; map == nullptr: nothing
struct Q5Next {
  const CUtensorMap* map;
  int set;
};

// forward pass of one field: per component x, y, z value stages (B), the z
// derivative fused into the z stage, then the x and y derivatives at the
// points.  Three CTA barriers per component (the derivative stage needs none
// after it: the next component does not touch U before its own two barriers).
template <class L, int MIR, bool WITHVAL, bool ISO>
__device__ __forceinline__ void q5_forward(const TabC<5, MIR>& tb0, int zoff, double* S, int t, bool act, int o_row, int o5,
                                           int o_y, int o_z, int* buf, unsigned* ph, const CUtensorMap* smap,
                                           int cset, Q5Next nxt, bool grad, bool first) {
  constexpr int N = 5;
  using Mr = Mir<N, MIR>;
  using Mp = Mir<N, 0>;
  constexpr int NE = Mr::NE > 0 ? Mr::NE : 1, NO = Mr::NO > 0 ? Mr::NO : 1;
  constexpr int PE = Mp::NE, PO = Mp::NO > 0 ? Mp::NO : 1;
  double* R = S + L::R;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(S + L::BAR);
  const int* coord = reinterpret_cast<const int*>(S + L::COORD);
#pragma unroll 1
  for (int comp = 0; comp < 3; ++comp) {
    const TabC<5, MIR>& tb = reload_tab(tb0, ISO ? 0 : zoff * (comp + 1));
    const auto& tDy = ISO ? tb.Dx : tb.Dy;
    const auto& tDz = ISO ? tb.Dx : tb.Dz;
    const int nbi = *buf ^ 1;
    if (t < L::E) {
      // lane e stages element e's next box (this field's next component, or
      // the next field / quintet); all lanes then wait for the current boxes
      if (comp + 1 < 3) {
        const int* cc = coord + (cset * L::E + t) * 4;
        // first component of a quintet: buffer nbi held this lane's output
        // boxes of the previous quintet -- their reduce-adds have read them
        if (first && comp == 0) bulk_wait_read();
        mbar_expect_tx(bars + nbi, L::BOXBYTES);
        tma_load_box(R + (nbi * L::E + t) * L::RB, smap, cc[0], cc[1], cc[2], comp + 1, bars + nbi);
      } else if (nxt.map) {
        const int* cc = coord + (nxt.set * L::E + t) * 4;
        mbar_expect_tx(bars + nbi, L::BOXBYTES);
        tma_load_box(R + (nbi * L::E + t) * L::RB, nxt.map, cc[0], cc[1], cc[2], 0, bars + nbi);
      }
    }
    mbar_wait(bars + *buf, (*ph >> *buf) & 1u);
    *ph ^= 1u << *buf;
    // x stage: row (e; k, j) of the box -> values at a
    if (act) {
      double v[N], E[NE], O[NO], o[N];
      const double2* row = reinterpret_cast<const double2*>(R + *buf * L::E * L::RB + o_row);
      SDME_CHECK(smem_ok(row, L::RP * 8, 16));
#pragma unroll
      for (int i = 0; i < L::RP / 2; ++i) {
        const double2 d = row[i];
        v[2 * i] = d.x;
        if (2 * i + 1 < N) v[2 * i + 1] = d.y;
      }
      eo_split<N, MIR>(v, E, O);
      eo_fwd<N, Mr::NE, Mr::NO>(tb.B, E, O, o);
#pragma unroll
      for (int a = 0; a < N; ++a) S[L::X + o5 + a] = o[a];
    }
    __syncthreads();
    // y stage: (e; k, a) -> values at b
    if (act) {
      double v[N], E[NE], O[NO], o[N];
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = S[L::X + o_y + 5 * j];
      eo_split<N, MIR>(v, E, O);
      eo_fwd<N, Mr::NE, Mr::NO>(tb.B, E, O, o);
#pragma unroll
      for (int b = 0; b < N; ++b) S[L::Y + o_y + 5 * b] = o[b];
    }
    __syncthreads();
    // z stage: column (e; b, a) -> point values at c and d/dz at the points
    if (act) {
      double v[N], E[NE], O[NO], u[N];
#pragma unroll
      for (int k = 0; k < N; ++k) v[k] = S[L::Y + o_z + 25 * k];
      eo_split<N, MIR>(v, E, O);
      eo_fwd<N, Mr::NE, Mr::NO>(tb.B, E, O, u);
      if (grad) {
#pragma unroll
        for (int c = 0; c < N; ++c) S[L::U + o_z + 25 * c] = u[c];
      }
      if (WITHVAL) {
#pragma unroll
        for (int c = 0; c < N; ++c) S[L::vslot(comp) + o_z + 25 * c] = u[c];
      }
      if (grad) {
        double pe[PE], po[PO], gz[N];
        eo_split<N, 0>(u, pe, po);
        eo_fwd<N, Mp::NO, Mp::NE>(tDz, po, pe, gz);
#pragma unroll
        for (int c = 0; c < N; ++c) S[L::slot(2, comp) + o_z + 25 * c] = gz[c];
      }
    }
    __syncthreads();
    if (grad && act) {
      double v[N], pe[PE], po[PO], gd[N];
      // x pencils (e; c, b) of the point values
#pragma unroll
      for (int a = 0; a < N; ++a) v[a] = S[L::U + o5 + a];
      eo_split<N, 0>(v, pe, po);
      eo_fwd<N, Mp::NO, Mp::NE>(tb.Dx, po, pe, gd);
#pragma unroll
      for (int a = 0; a < N; ++a) S[L::slot(0, comp) + o5 + a] = gd[a];
      // y pencils (e; c, a)
#pragma unroll
      for (int b = 0; b < N; ++b) v[b] = S[L::U + o_y + 5 * b];
      eo_split<N, 0>(v, pe, po);
      eo_fwd<N, Mp::NO, Mp::NE>(tDy, po, pe, gd);
#pragma unroll
      for (int b = 0; b < N; ++b) S[L::slot(1, comp) + o_y + 5 * b] = gd[b];
    }
    *buf ^= 1;
  }
  __syncthreads();
}

// backward pass: per component the weighted flux slots (and the weighted value
// slot) -> B^T (x) B^T (x) B^T (sum_d D^_d^T F_d [+ V]) as an output box per
// element, added to y by lanes 0..4 (bulk tensor reduce-add)
template <int MODE, int MIR, bool VAL, bool VALS, bool ISO>
__device__ __forceinline__ void q5_backward(const TabC<5, MIR>& tb0, int zoff, const Geo& g, double* S, int t, bool act,
                                            int o_row, int o5, int o_y, int o_z, int obuf, int cset, bool grad,
                                            const CUtensorMap* ymap, bool* waited) {
  constexpr int N = 5;
  using L = Q5Lay<MODE, VALS>;
  using Mr = Mir<N, MIR>;
  using Mp = Mir<N, 0>;
  constexpr int HP = Half<N>::HP, H = Half<N>::H;
  const int* coord = reinterpret_cast<const int*>(S + L::COORD);
  double* O = S + L::R + obuf * L::E * L::RB;
#pragma unroll 1
  for (int comp = 0; comp < 3; ++comp) {
    const TabC<5, MIR>& tb = reload_tab(tb0, ISO ? 0 : zoff * (comp + 1));
    const auto& tDy = ISO ? tb.Dx : tb.Dy;
    const auto& tDz = ISO ? tb.Dx : tb.Dz;
    if (grad) {
      // x' pencils (e; c, b): U = D^_x^T F_x
      if (act) {
        double q[N], qe[HP], qo[H], y[N];
#pragma unroll
        for (int a = 0; a < N; ++a) q[a] = S[L::slot(0, comp) + o5 + a];
        eo_qsplit<N>(q, qe, qo);
        eo_bwd_t<N, N, 0, -1, Mp::NO, Mp::NE, false>(tb.Dx, qe, qo, y);
#pragma unroll
        for (int a = 0; a < N; ++a) S[L::U + o5 + a] = y[a];
      }
      __syncthreads();
      // y' pencils (e; c, a): U += D^_y^T F_y
      if (act) {
        double q[N], qe[HP], qo[H], y[N];
#pragma unroll
        for (int b = 0; b < N; ++b) {
          q[b] = S[L::slot(1, comp) + o_y + 5 * b];
          y[b] = S[L::U + o_y + 5 * b];
        }
        eo_qsplit<N>(q, qe, qo);
        eo_bwd_t<N, N, 0, -1, Mp::NO, Mp::NE, true>(tDy, qe, qo, y);
#pragma unroll
        for (int b = 0; b < N; ++b) S[L::U + o_y + 5 * b] = y[b];
      }
      __syncthreads();
    }
    // z' columns (e; b, a): V = U + D^_z^T F_z (+ value term), then B^T along z
    if (act) {
      double v[N], q[N], qe[HP], qo[H], h[N];
#pragma unroll
      for (int c = 0; c < N; ++c) v[c] = grad ? S[L::U + o_z + 25 * c] : 0.0;
      if (grad) {
#pragma unroll
        for (int c = 0; c < N; ++c) q[c] = S[L::slot(2, comp) + o_z + 25 * c];
        eo_qsplit<N>(q, qe, qo);
        eo_bwd_t<N, N, 0, -1, Mp::NO, Mp::NE, true>(tDz, qe, qo, v);
      }
      if (VAL) {
#pragma unroll
        for (int c = 0; c < N; ++c) v[c] += S[L::vslot(comp) + o_z + 25 * c];
      }
      eo_qsplit<N>(v, qe, qo);
      eo_bwd_t<N, N, MIR, 1, Mr::NE, Mr::NO, false>(tb.B, qe, qo, h);
#pragma unroll
      for (int k = 0; k < N; ++k) S[L::Y + o_z + 25 * k] = h[k];
    }
    __syncthreads();
    // y' items (e; k, a): B^T along y
    if (act) {
      double v[N], qe[HP], qo[H], h[N];
#pragma unroll
      for (int b = 0; b < N; ++b) v[b] = S[L::Y + o_y + 5 * b];
      eo_qsplit<N>(v, qe, qo);
      eo_bwd_t<N, N, MIR, 1, Mr::NE, Mr::NO, false>(tb.B, qe, qo, h);
#pragma unroll
      for (int j = 0; j < N; ++j) S[L::X + o_y + 5 * j] = h[j];
    }
    // the previous component's reduce-adds have read their output boxes
    if (t < L::E) bulk_wait_read();
    __syncthreads();
    // x' items (e; k, j): B^T along x -> row of the element's output box;
    // constrained points and the pitch slot get 0 (as element_col)
    if (act) {
      double v[N], qe[HP], qo[H], acc[N];
#pragma unroll
      for (int a = 0; a < N; ++a) v[a] = S[L::X + o5 + a];
      eo_qsplit<N>(v, qe, qo);
      eo_bwd_t<N, N, MIR, 1, Mr::NE, Mr::NO, false>(tb.B, qe, qo, acc);
      if (g.dmask[comp]) {
        const int e = t / 25, w = t - 25 * e;
        const int* cc = coord + (cset * L::E + e) * 4;
        const int X0 = cc[0], Y0 = cc[1], Z0 = cc[2];
        if (touches_dirichlet(g, comp, X0, Y0, Z0, N)) {
          const int Z = Z0 + w / N, Y = Y0 + w % N;
#pragma unroll
          for (int i = 0; i < N; ++i)
            if (constrained(g, comp, X0 + i, Y, Z)) acc[i] = 0.0;
        }
      }
      double2* orow = reinterpret_cast<double2*>(O + o_row);
      SDME_CHECK(smem_ok(orow, L::RP * 8, 16));
#pragma unroll
      for (int i = 0; i < L::RP / 2; ++i) orow[i] = make_double2(acc[2 * i], 2 * i + 1 < N ? acc[2 * i + 1] : 0.0);
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (t < L::E && ymap) {
      const int* cc = coord + (cset * L::E + t) * 4;
      if (!cc[3]) {
        // first write to y by this lane: the previous launch on the stream (a
        // colour pass, or the zeroing of y) has completed (PDL, tma.cuh)
        if (!*waited) {
          pdl_wait();
          *waited = true;
        }
        tma_reduce_add_box(ymap, O + t * L::RB, cc[0], cc[1], cc[2], comp);
      }
    }
  }
}

// Stored-data operator (MODE_PA): the point data K, ln J (10 doubles per point,
// [elem][slot][q]) is on its way while the forward pass of p runs, not fetched
// at the point stage where its HBM latency would sit between two CTA barriers.
// SDME_PA_PREF (measured at config 2, K.p / K.p + c_m M in ms; 0: 1.52 / 1.96):
//   1  loads into registers before the forward pass           1.63 / 1.51
//   2  L2 prefetch of the quintet's lines before the pass     1.48 / 1.85
//   3  1 + L2 prefetch of the next quintet a round ahead      1.35 / 1.49  (default)
//   4  3 with the register loads at the point stage           1.38 / 1.56
// SDME_Q5_BOX_PREF: L2 prefetch (cp.async.bulk.prefetch.tensor) of the next
// quintet's u / p boxes.  Measured slower (K.p 1.606 -> 1.639 ms, f_int 1.105 ->
// 1.128: the double-buffered box loads already hide their latency and the 30
// extra bulk operations per quintet cost more than they save): off.
#ifndef SDME_Q5_BOX_PREF
#define SDME_Q5_BOX_PREF 0
#endif
#ifndef SDME_PA_PREF
#define SDME_PA_PREF 3
#endif

template <int MINB, int MODE, bool VAL, int MIR, bool ISO>
__global__ void __launch_bounds__(128, MINB) element_q5(const __grid_constant__ TabC<5, MIR> tb,
                                                        const __grid_constant__ Geo g, OpArgs args) {
  constexpr int N = 5, Q = 125, T = 128;
  using L = Q5Lay<MODE, VAL>;
  constexpr int QPT = (L::EQ + T - 1) / T;  // 5 point rounds
  constexpr bool UPASS = (MODE == MODE_APPLY || MODE == MODE_FINT || MODE == MODE_SETUP);
  constexpr bool PPASS = (MODE == MODE_APPLY || MODE == MODE_PA || MODE == MODE_MASS);
  constexpr bool PGRAD = MODE != MODE_MASS;
  extern __shared__ __align__(128) double S[];
  const int t = threadIdx.x;
  const int zoff = args.zero;
  if (args.skip && *(volatile const int*)args.skip) return;
  pdl_launch_dependents();
  SDME_CHECK(smem_ok(S, L::PER * 8, 128));
  const bool act = t < L::EQ / N;  // 125 pencils per stage
  const int tt = act ? t : 0;
  // lane orders (header): natural, (a; e; k), (b; a; e)
  const int o5 = 5 * tt;
  const int o_row = (tt / 25) * L::RB + (tt % 25) * L::RP;
  const int o_y = 125 * ((tt / 5) % 5) + 25 * (tt % 5) + tt / 25;
  const int o_z = 125 * (tt % 5) + 5 * (tt / 25) + (tt / 5) % 5;
  const long long cnt = colour_count(g, args.colour);
  const long long nq = (cnt + L::E - 1) / L::E;
  const double mu_k = args.c_k * g.mu, lam_k = args.c_k * g.lam;
  const double cmr = args.c_m * g.rho;
  const CUtensorMap* umap = static_cast<const CUtensorMap*>(args.tu);
  const CUtensorMap* pmap = static_cast<const CUtensorMap*>(args.tp);
  const CUtensorMap* ymap = static_cast<const CUtensorMap*>(args.ty);
  const CUtensorMap* first_map = UPASS ? umap : pmap;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(S + L::BAR);
  int* coord = reinterpret_cast<int*>(S + L::COORD);
  unsigned ph = 0;
  int buf = 0;
  bool waited = false;
  for (int q = t; q < Q; q += T) S[L::W + q] = tb.wq[q % N] * tb.wq[(q / N) % N] * tb.wq[q / (N * N)] * tb.detJ;
  if (t == 0) {
    mbar_init(bars, L::E);
    mbar_init(bars + 1, L::E);
    mbar_fence_init();
  }
  __syncthreads();
  if (t < L::E && (long long)blockIdx.x < nq) {
    const long long idx = (long long)blockIdx.x * L::E + t;
    int ei, ej, ek;
    colour_element(g, args.colour, idx < cnt ? idx : cnt - 1, ei, ej, ek);
    int* cc = coord + t * 4;
    cc[0] = (N - 1) * ei, cc[1] = (N - 1) * ej, cc[2] = (N - 1) * ek, cc[3] = idx >= cnt;
    mbar_expect_tx(bars, L::BOXBYTES);
    tma_load_box(S + L::R + t * L::RB, first_map, cc[0], cc[1], cc[2], 0, bars);
  }
  if (MODE == MODE_PA && SDME_PA_PREF) __syncthreads();  // coordinates of the first quintet
  int cur = 0;
  for (long long qd = blockIdx.x; qd < nq; qd += gridDim.x, cur ^= 1) {
    const bool has_next = qd + gridDim.x < nq;
    if (t < L::E && has_next) {
      const long long idx = (qd + gridDim.x) * L::E + t;
      int ei, ej, ek;
      colour_element(g, args.colour, idx < cnt ? idx : cnt - 1, ei, ej, ek);
      int* cc = coord + ((cur ^ 1) * L::E + t) * 4;
      cc[0] = (N - 1) * ei, cc[1] = (N - 1) * ej, cc[2] = (N - 1) * ek, cc[3] = idx >= cnt;
      if (SDME_Q5_BOX_PREF) {
        // the next quintet's input boxes on their way into L2 a round ahead of
        // their TMA loads (which then complete at L2 latency)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (UPASS) tma_prefetch_box(umap, cc[0], cc[1], cc[2], c);
          if (PPASS) tma_prefetch_box(pmap, cc[0], cc[1], cc[2], c);
        }
      }
    }
    const Q5Next after_last{has_next ? first_map : nullptr, cur ^ 1};
    double Hu[QPT][9];
    if (UPASS) {
      const Q5Next after_u = MODE == MODE_APPLY ? Q5Next{pmap, cur} : after_last;
      q5_forward<L, MIR, false, ISO>(tb, zoff, S, t, act, o_row, o5, o_y, o_z, &buf, &ph, umap, cur, after_u, true,
                                              true);
#pragma unroll
      for (int r = 0; r < QPT; ++r) {
        const int pid = t + r * T;
        if (pid < L::EQ) {
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int d = 0; d < 3; ++d) Hu[r][i * 3 + d] = S[L::slot(d, i) + pid];
        }
      }
    }
    constexpr bool KREG = MODE == MODE_PA && (SDME_PA_PREF == 1 || SDME_PA_PREF == 3 || SDME_PA_PREF == 4);
    double Kq[KREG ? QPT : 1][kQpSlots];
    auto load_kq = [&]() {
#pragma unroll
      for (int r = 0; r < QPT; ++r) {
        const int pid = t + r * T;
        if (pid < L::EQ) {
          const int e = pid / Q, q = pid - e * Q;
          const int* cc = coord + (cur * L::E + e) * 4;
          const long long eid = ((long long)(cc[2] / (N - 1)) * g.ny + cc[1] / (N - 1)) * g.nx + cc[0] / (N - 1);
          const double* qp = args.qpd + eid * (kQpSlots * Q) + q;
#pragma unroll
          for (int k = 0; k < kQpSlots; ++k) Kq[KREG ? r : 0][k] = __ldg(qp + k * Q);
        }
      }
    };
    // L2 prefetch of the point data of coordinate set `set` (an element's 10,000
    // bytes start 16-byte aligned: 80 lines cover them)
    auto prefetch_set = [&](int set) {
      constexpr int LPE = (kQpSlots * Q * 8 + 127) / 128 + 1;
      for (int l = t; l < L::E * LPE; l += T) {
        const int e = l / LPE, j = l - e * LPE;
        const int* cc = coord + (set * L::E + e) * 4;
        const long long eid = ((long long)(cc[2] / (N - 1)) * g.ny + cc[1] / (N - 1)) * g.nx + cc[0] / (N - 1);
        const char* base = reinterpret_cast<const char*>(args.qpd + eid * (kQpSlots * Q));
        const int off = j * 128 < kQpSlots * Q * 8 - 8 ? j * 128 : kQpSlots * Q * 8 - 8;
        prefetch_l2(base + off);
      }
    };
    if (MODE == MODE_PA && (SDME_PA_PREF == 1 || SDME_PA_PREF == 3)) load_kq();
    if (MODE == MODE_PA && (SDME_PA_PREF == 2 || (SDME_PA_PREF >= 3 && qd == blockIdx.x))) prefetch_set(cur);
    if (PPASS)
      q5_forward<L, MIR, VAL, ISO>(tb, zoff, S, t, act, o_row, o5, o_y, o_z, &buf, &ph, pmap, cur, after_last,
                                            PGRAD, !UPASS);
    if (MODE == MODE_PA && SDME_PA_PREF >= 3 && has_next) prefetch_set(cur ^ 1);
    if (MODE == MODE_PA && SDME_PA_PREF == 4) load_kq();
#pragma unroll
    for (int r = 0; r < QPT; ++r) {
      const int pid = t + r * T;
      if (pid >= L::EQ) continue;
      const int e = pid / Q, q = pid - e * Q;
      const double wdet = S[L::W + q];
      if (MODE == MODE_MASS) {
#pragma unroll
        for (int i = 0; i < 3; ++i) S[L::vslot(i) + pid] *= cmr * wdet;
        continue;
      }
      long long eid = 0;
      if ((MODE == MODE_PA && !KREG) || MODE == MODE_SETUP) {
        const int* cc = coord + (cur * L::E + e) * 4;
        eid = ((long long)(cc[2] / (N - 1)) * g.ny + cc[1] / (N - 1)) * g.nx + cc[0] / (N - 1);
      }
      QpK s;
      if (KREG) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) s.K[i][d] = Kq[KREG ? r : 0][i * 3 + d];
        s.lnJ = Kq[KREG ? r : 0][9];
      } else if (MODE == MODE_PA) {
        const double* qd = args.qpd + eid * (kQpSlots * Q) + q;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) s.K[i][d] = __ldg(qd + (i * 3 + d) * Q);
        s.lnJ = __ldg(qd + 9 * Q);
      } else {
        qp_k(Hu[r], s);
        if (!(s.det > 0.0)) {
          const int* cc = coord + (cur * L::E + e) * 4;
          const long long ref = ((long long)(cc[2] / (N - 1)) * g.ny + cc[1] / (N - 1)) * g.nx + cc[0] / (N - 1);
          const int a = q % N, b = (q / N) % N, c = q / (N * N);
          atomicMin(args.inv_flag, (unsigned long long)ref * Q + (unsigned long long)((a * N + b) * N + c));
        }
      }
      if (MODE == MODE_SETUP) {
        // ghost elements repeat the last element: identical values, harmless
        double* qd = args.qpd + eid * (kQpSlots * Q) + q;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) qd[(i * 3 + d) * Q] = s.K[i][d];
        qd[9 * Q] = s.lnJ;
        continue;
      }
      if (MODE == MODE_FINT) {
        const double cK = g.lam * s.lnJ - g.mu;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) S[L::slot(d, i) + pid] = wdet * fma(g.mu, s.F[i][d], cK * s.K[i][d]);
      } else {
        double Hp[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) Hp[i][d] = S[L::slot(d, i) + pid];
        double tr = 0.0;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) tr = fma(s.K[i][d], Hp[i][d], tr);
        double M1[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j)
            M1[i][j] = fma(s.K[i][0], Hp[j][0], fma(s.K[i][1], Hp[j][1], s.K[i][2] * Hp[j][2]));
        const double cc2 = mu_k - lam_k * s.lnJ;
        const double lt = lam_k * tr;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const double m2 = fma(M1[i][0], s.K[0][d], fma(M1[i][1], s.K[1][d], M1[i][2] * s.K[2][d]));
            S[L::slot(d, i) + pid] = wdet * fma(cc2, m2, fma(lt, s.K[i][d], mu_k * Hp[i][d]));
          }
        if (VAL) {
#pragma unroll
          for (int i = 0; i < 3; ++i) S[L::vslot(i) + pid] *= cmr * wdet;
        }
      }
    }
    if (MODE == MODE_SETUP) {
      __syncthreads();  // the next quintet's z stage rewrites the slots
      continue;
    }
    __syncthreads();
    q5_backward<MODE, MIR, VAL, VAL, ISO>(tb, zoff, g, S, t, act, o_row, o5, o_y, o_z, buf ^ 1, cur, PGRAD, ymap, &waited);
  }
  // the reduce-adds have completed before the CTA (and its shared memory) retires
  if (t < L::E) bulk_wait_all();
}

}  // namespace sdme
