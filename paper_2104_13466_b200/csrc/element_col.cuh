// Collocated sum factorisation (m = P + 1): f_int and K(u).p with the
// gradient taken at the quadrature points.
//
// With as many Gauss points as basis functions per axis the 1D value table B
// (m x n, n = m) is square and well conditioned (cond <= 34 for every basis
// and P <= 8), so the 1D derivative at the points is the collocation matrix
// D^ = D B^-1 (m x m, the same for every basis).  The forward pass becomes
//   values:    U = (B (x) B (x) B) u          (three 1-array stages)
//   gradient:  d_x U = D^_x U along x, d_y, d_z likewise (point pencils)
// and the backward pass the transpose, with the quadrature weights and det J
// applied to the flux at the points.  Against element_v3 (derivative tables in
// the x / y / z stages, 1 -> 2 -> 3 arrays) this moves ~20% fewer words through
// shared memory and does ~25% fewer multiply-adds per element; all 1D
// operators keep the even-odd split (eo.cuh): the basis mirror for B and the
// reversal mirror of the Gauss points for D^.
//
// Mathematically identical to the v3 kernel; results agree to rounding
// (parity tests at 1e-12 against the reference).
#pragma once
#include "element_eo.cuh"
#include "tma.cuh"

namespace sdme {

template <int N, int MIR>
struct TabC {
  using Mr = Mir<N, MIR>;
  using Mp = Mir<N, 0>;  // Gauss points: reversal mirror
  EoFwd<N, Mr::NE, Mr::NO> B;              // coefficients -> point values
  EoFwd<N, Mp::NO, Mp::NE> Dx, Dy, Dz;     // collocated derivative (x 2/h), points -> points
  EoBwd<N, Mr::NE, Mr::NO> bB;             // B^T: points -> coefficients
  EoBwd<N, Mp::NO, Mp::NE> bDx, bDy, bDz;  // D^^T
  double wq[N];                            // 1D rule weights
  double detJ;
};

// shared layout of one element (component-serial): point slots [d][comp][q]
// (V3 qi), x-stage output [k][j][a], y-stage output [k][b][a], point values /
// backward accumulator U[c][b][a], the weight table W[q] = w_a w_b w_c det J,
// then either (TM = false) the cp.async-staged rows [2][N^3] and the table of
// lattice offsets of the N^3 box entries (a staged copy costs one shared load
// and an add), or (TM = true) three TMA boxes [k][j][RP] (two staging buffers
// and the output box of the bulk reduce-add; RP = row pitch, N rounded up to
// even so that box rows are 16-byte multiples) and their two mbarriers.
template <int N, bool VALS, bool TM = false>
struct ColLay {
  using C = V3<N, N, 1, 1, VALS>;
  static constexpr int SQ = TM ? N * N * N : C::Ly::sq;    // point slot stride (no cross-slot accesses)
  static constexpr int SX = N * N;                          // x output, k stride
  // odd N >= 7 (P = 6, 8): y-stage output and point values in transposed slabs,
  // Y(k, b, a) = k N^2 + b + a N and U(c, b, a) = c N + b + a N^2 (bank model,
  // tools/col_layout_n.py: 882 -> 504 / 1344 -> 1218 wavefronts at N = 7,
  // 1377 -> 972 / 2160 -> 2025 at N = 9; worse for even N)
  static constexpr bool TY = N >= 7 && (N & 1);
  // N = 4 with TMA boxes (P = 3, one element per half-warp): 16 lanes touch a
  // 4x4 slice of a 4x4x4 array with one coordinate fixed; bank (within a
  // 16-double row, row = slowest index s) (4 m + f) ^ 5 s makes every
  // axis-aligned slice hit 16 distinct banks (Y, U and the point slots)
  static constexpr bool SW = TM && N == 4;
  static constexpr int SY = TY ? N * N : (SW ? 16 : C::Ly::sy);  // y output, k stride
  static constexpr int SU = N * N;                          // point values region per c (size)
  static constexpr int YB = TY ? 1 : N, YA = TY ? N : 1;
  static constexpr int UC = TY ? N : SU, UB = TY ? 1 : N, UA = TY ? N * N : 1;
  __device__ static int yo(int k, int b, int a) {
    const int o = SW ? k * 16 + ((b * 4 + a) ^ (5 * k)) : k * SY + b * YB + a * YA;
    SDME_CHECK(k >= 0 && k < N && b >= 0 && b < N && a >= 0 && a < N && o >= 0 && o < N * SY);
    return o;
  }
  __device__ static int uo(int c, int b, int a) {
    const int o = SW ? c * 16 + ((b * 4 + a) ^ (5 * c)) : c * UC + b * UB + a * UA;
    SDME_CHECK(c >= 0 && c < N && b >= 0 && b < N && a >= 0 && a < N && o >= 0 && o < N * SU);
    return o;
  }
  static constexpr int PTS = (VALS ? 12 : 9) * SQ;
  // x-stage output X(k, j, a) = k XK + j XJ + a XA: TM layout (XK, XJ, XA) =
  // (N, 1, N^2 rounded up to 1 mod 16), bank-conflict free for both the x-stage
  // rows (lanes (k, j)) and the y-stage columns (lanes (k, a)) -- tools/col_layout.py;
  // else rows [k][j][a]
  static constexpr int XK = TM ? N : SX, XJ = TM ? 1 : N;
  static constexpr int XA = TM ? (N * N + 14) / 16 * 16 + 1 : 1;
  static constexpr int XSPAN = TM ? (N - 1) * (XK + XJ + XA) + 1 : N * SX;
  __device__ static int xo(int k, int j, int a) {
    SDME_CHECK(k >= 0 && k < N && j >= 0 && j < N && a >= 0 && a < N);
    return k * XK + j * XJ + a * XA;
  }
  static constexpr int X = PTS, Y = X + XSPAN, U = Y + N * SY, W = U + N * SU;
  static constexpr int RP = TM ? BoxW<N>::BW : N;           // staged row pitch (TMA box width)
  static constexpr int RB = TM ? (N * N * RP + 15) / 16 * 16 : N * N * N;  // one staging buffer (128-B multiple)
  static constexpr int R = TM ? (W + N * N * N + 15) / 16 * 16 : W + N * N * N;
  static constexpr int O = R + 2 * RB;                      // TM: output box of the reduce-add
  static constexpr int TAB = R + 2 * RB;                    // !TM: int lattice offsets of the box entries
  static constexpr int BAR = O + RB;                        // TM: two mbarriers
  static constexpr int PER = TM ? BAR + 2 : TAB + (N * N * N + 1) / 2;
  __device__ static int qi(int d, int comp, int q) {
    SDME_CHECK(d >= 0 && d < (VALS ? 4 : 3) && comp >= 0 && comp < 3 && q >= 0 && q < N * N * N);
    return (d * 3 + comp) * SQ + (SW ? q ^ (5 * (q >> 4)) : q);
  }
};

// per-element shared region rounded to 128 B (the SUB = 2 half-warp regions)
template <int N, bool VALS, bool TM = false>
struct ColPer {
  static constexpr int PERP = (ColLay<N, VALS, TM>::PER + 15) / 16 * 16;
};

// tables re-read per component loop (OpArgs::zero)?  N = 5 only with TMA boxes:
// the general-mesh instance of this kernel measured slower with it (48^3 K.p
// 1.54 -> 1.59 ms), the stored-data operator faster (1.51 -> 1.49 ms)
template <int N, bool TM>
__host__ __device__ constexpr bool col_reload() {
  return N >= SDME_COL_RELOAD_MIN_N && (N > 5 || TM);
}

// what to stage after the last component of a forward pass (TMA path)
struct NextBox {
  const CUtensorMap* map;  // nullptr: nothing
  int X0, Y0, Z0;
};

template <int N, int T>
__device__ __forceinline__ void col_stage(const Geo& g, const double* __restrict__ field, int comp, int X0, int Y0,
                                          int Z0, double* rows, int t, const int* tab) {
  const double* base = field + comp * g.Ns + ((long long)Z0 * g.Ly + Y0) * g.Px + X0;
  for (int w = t; w < N * N * N; w += T) cp_async8(rows + w, base + tab[w]);
  cp_async_commit();
}

template <int N, int WPE, int MIR, bool VAL, bool VALS, bool TM = false, int SUB = 1, bool ISO = false>
__device__ __forceinline__ void col_forward(const TabC<N, MIR>& tb0, int zoff, const Geo& g,
                                            const double* __restrict__ src, int X0, int Y0, int Z0, double* S, int t,
                                            int* buf, NextRows next, bool grad, const CUtensorMap* smap = nullptr,
                                            NextBox nbox = {}, unsigned* ph = nullptr) {
  using L = ColLay<N, VALS, TM>;
  using Mr = Mir<N, MIR>;
  using Mp = Mir<N, 0>;
  constexpr int NE = Mr::NE > 0 ? Mr::NE : 1, NO = Mr::NO > 0 ? Mr::NO : 1;
  constexpr int PE = Mp::NE, PO = Mp::NO > 0 ? Mp::NO : 1;
  double* R = S + L::R;
  const int* tab = reinterpret_cast<const int*>(S + L::TAB);
#pragma unroll 1
  for (int comp = 0; comp < 3; ++comp) {
    // tables re-read from the constant bank per component (OpArgs::zero)
    const TabC<N, MIR>& tb = reload_tab(tb0, (col_reload<N, TM>() && !ISO) ? zoff * (comp + 1) : 0);
    // cubic elements (ISO): one derivative table for the three axes
    const auto& tDy = ISO ? tb.Dx : tb.Dy;
    const auto& tDz = ISO ? tb.Dx : tb.Dz;
    if (TM) {
      // one lane issues the next box (this field's next component, or the
      // next field / element), then every lane waits for the current box
      const int nbi = *buf ^ 1;
      unsigned long long* bars = reinterpret_cast<unsigned long long*>(S + L::BAR);
      if (t == 0) {
        if (comp + 1 < 3) {
          mbar_expect_tx(bars + nbi, N * N * L::RP * 8);
          tma_load_box(R + nbi * L::RB, smap, X0 & ~1, Y0, Z0, comp + 1, bars + nbi);
        } else if (nbox.map) {
          mbar_expect_tx(bars + nbi, N * N * L::RP * 8);
          tma_load_box(R + nbi * L::RB, nbox.map, nbox.X0 & ~1, nbox.Y0, nbox.Z0, 0, bars + nbi);
        }
      }
      mbar_wait(bars + *buf, (*ph >> *buf) & 1u);
      *ph ^= 1u << *buf;
    } else {
      double* nb = R + (*buf ^ 1) * N * N * N;
      if (comp + 1 < 3) {
        col_stage<N, 32 * WPE / SUB>(g, src, comp + 1, X0, Y0, Z0, nb, t, tab);
        cp_async_wait<1>();
      } else if (next.field) {
        col_stage<N, 32 * WPE / SUB>(g, next.field, 0, next.X0, next.Y0, next.Z0, nb, t, tab);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      group_sync<WPE>(0);
    }
    // x stage: item (k, j) -> values at a
    for (int w = t; w < N * N; w += 32 * WPE / SUB) {
      double v[N], E[NE], O[NO], o[N];
      if (TM && (N & 1)) {
        // even P: boxes start at the element; 16-byte loads of the pitched
        // box row (conflict-free for RP = 6)
        const double2* row = reinterpret_cast<const double2*>(R + *buf * L::RB + w * L::RP);
        SDME_CHECK(smem_ok(row, L::RP * 8, 16));
#pragma unroll
        for (int i = 0; i < L::RP / 2; ++i) {
          const double2 d = row[i];
          v[2 * i] = d.x;
          if (2 * i + 1 < N) v[2 * i + 1] = d.y;
        }
      } else if (TM) {
        // odd P: the box starts at the even x at or below the element (shift X0 & 1)
        const double* row = R + *buf * L::RB + w * L::RP + (X0 & 1);
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = row[i];
      } else {
        const double* row = R + *buf * N * N * N + w * N;
#pragma unroll
        for (int i = 0; i < N; ++i) v[i] = row[i];
      }
      eo_split<N, MIR>(v, E, O);
      eo_fwd<N, Mr::NE, Mr::NO>(tb.B, E, O, o);
#pragma unroll
      for (int a = 0; a < N; ++a) S[L::X + L::xo(w / N, w % N, a)] = o[a];
    }
    group_sync<WPE>(0);
    // y stage: item (k, a) -> values at b
    for (int w = t; w < N * N; w += 32 * WPE / SUB) {
      const int k = w / N, a = w % N;
      double v[N], E[NE], O[NO], o[N];
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = S[L::X + L::xo(k, j, a)];
      eo_split<N, MIR>(v, E, O);
      eo_fwd<N, Mr::NE, Mr::NO>(tb.B, E, O, o);
#pragma unroll
      for (int b = 0; b < N; ++b) S[L::Y + L::yo(k, b, a)] = o[b];
    }
    group_sync<WPE>(0);
    // z stage: column (b, a) -> values U at c, and d/dz at the points
    for (int w = t; w < N * N; w += 32 * WPE / SUB) {
      double v[N], E[NE], O[NO], u[N];
#pragma unroll
      for (int k = 0; k < N; ++k) v[k] = S[L::Y + L::yo(k, w / N, w % N)];
      eo_split<N, MIR>(v, E, O);
      eo_fwd<N, Mr::NE, Mr::NO>(tb.B, E, O, u);
#pragma unroll
      for (int c = 0; c < N; ++c) S[L::U + L::uo(c, w / N, w % N)] = u[c];
      if (VAL) {
#pragma unroll
        for (int c = 0; c < N; ++c) S[L::qi(3, comp, c * N * N + w)] = u[c];
      }
      if (grad) {
        double pe[PE], po[PO], gz[N];
        eo_split<N, 0>(u, pe, po);
        eo_fwd<N, Mp::NO, Mp::NE>(tDz, po, pe, gz);
#pragma unroll
        for (int c = 0; c < N; ++c) S[L::qi(2, comp, c * N * N + w)] = gz[c];
      }
    }
    group_sync<WPE>(0);
    if (grad) {
      // x pencils (c, b) and y pencils (c, a) of the point values
      for (int w = t; w < N * N; w += 32 * WPE / SUB) {
        const int c = w / N, r = w % N;
        double v[N], pe[PE], po[PO], gx[N], gy[N];
#pragma unroll
        for (int a = 0; a < N; ++a) v[a] = S[L::U + L::uo(c, r, a)];
        eo_split<N, 0>(v, pe, po);
        eo_fwd<N, Mp::NO, Mp::NE>(tb.Dx, po, pe, gx);
#pragma unroll
        for (int a = 0; a < N; ++a) S[L::qi(0, comp, c * N * N + r * N + a)] = gx[a];
#pragma unroll
        for (int b = 0; b < N; ++b) v[b] = S[L::U + L::uo(c, b, r)];
        eo_split<N, 0>(v, pe, po);
        eo_fwd<N, Mp::NO, Mp::NE>(tDy, po, pe, gy);
#pragma unroll
        for (int b = 0; b < N; ++b) S[L::qi(1, comp, c * N * N + b * N + r)] = gy[b];
      }
      group_sync<WPE>(0);
    }
    *buf ^= 1;
  }
}

// backward: per component, the weighted flux slots 0..2 (and the weighted
// value slot 3 when VAL) -> y += B^T (x) B^T (x) B^T (sum_d D^_d^T F_d [+ V])
template <int N, int WPE, int MIR, bool VAL, bool VALS, bool TM = false, int SUB = 1, bool ISO = false>
__device__ __forceinline__ void col_backward(const TabC<N, MIR>& tb0, int zoff, const Geo& g,
                                             double* __restrict__ dst, int X0, int Y0, int Z0, double* S, int t,
                                             double* evb, bool grad, const CUtensorMap* ymap = nullptr,
                                             bool* waited = nullptr) {
  using L = ColLay<N, VALS, TM>;
  using Mr = Mir<N, MIR>;
  using Mp = Mir<N, 0>;
  constexpr int HP = Half<N>::HP, H = Half<N>::H > 0 ? Half<N>::H : 1;
  // N <= 5: the forward tables serve the backward pass (make_tabc stores the
  // backward ones as their exact transposes there): half the table constants
  constexpr bool FT = N <= 5;
#pragma unroll 1
  for (int comp = 0; comp < 3; ++comp) {
    const TabC<N, MIR>& tb = reload_tab(tb0, (col_reload<N, TM>() && !ISO) ? zoff * (comp + 1) : 0);
    const auto& tDy = ISO ? tb.Dx : tb.Dy;
    const auto& tDz = ISO ? tb.Dx : tb.Dz;
    if (grad) {
      // x' pencils (c, b): U = D^_x^T F_x
      for (int w = t; w < N * N; w += 32 * WPE / SUB) {
        const int c = w / N, b = w % N;
        double q[N], qe[HP], qo[H], y[N];
#pragma unroll
        for (int a = 0; a < N; ++a) q[a] = S[L::qi(0, comp, c * N * N + b * N + a)];
        eo_qsplit<N>(q, qe, qo);
        if (FT) eo_bwd_t<N, N, 0, -1, Mp::NO, Mp::NE, false>(tb.Dx, qe, qo, y);
        else eo_bwd<N, N, 0, -1, Mp::NO, Mp::NE, false>(tb.bDx, qe, qo, y);
#pragma unroll
        for (int a = 0; a < N; ++a) S[L::U + L::uo(c, b, a)] = y[a];
      }
      group_sync<WPE>(0);
      // y' pencils (c, a): U += D^_y^T F_y
      for (int w = t; w < N * N; w += 32 * WPE / SUB) {
        const int c = w / N, a = w % N;
        double q[N], qe[HP], qo[H], y[N];
#pragma unroll
        for (int b = 0; b < N; ++b) {
          q[b] = S[L::qi(1, comp, c * N * N + b * N + a)];
          y[b] = S[L::U + L::uo(c, b, a)];
        }
        eo_qsplit<N>(q, qe, qo);
        if (FT) eo_bwd_t<N, N, 0, -1, Mp::NO, Mp::NE, true>(tDy, qe, qo, y);
        else eo_bwd<N, N, 0, -1, Mp::NO, Mp::NE, true>(tb.bDy, qe, qo, y);
#pragma unroll
        for (int b = 0; b < N; ++b) S[L::U + L::uo(c, b, a)] = y[b];
      }
      group_sync<WPE>(0);
    }
    // z' columns (b, a): V = U + D^_z^T F_z (+ value term), then B^T along z
    for (int w = t; w < N * N; w += 32 * WPE / SUB) {
      double v[N], q[N], qe[HP], qo[H], h[N];
#pragma unroll
      for (int c = 0; c < N; ++c) v[c] = grad ? S[L::U + L::uo(c, w / N, w % N)] : 0.0;
      if (grad) {
#pragma unroll
        for (int c = 0; c < N; ++c) q[c] = S[L::qi(2, comp, c * N * N + w)];
        eo_qsplit<N>(q, qe, qo);
        if (FT) eo_bwd_t<N, N, 0, -1, Mp::NO, Mp::NE, true>(tDz, qe, qo, v);
        else eo_bwd<N, N, 0, -1, Mp::NO, Mp::NE, true>(tb.bDz, qe, qo, v);
      }
      if (VAL) {
#pragma unroll
        for (int c = 0; c < N; ++c) v[c] += S[L::qi(3, comp, c * N * N + w)];
      }
      eo_qsplit<N>(v, qe, qo);
      if (FT) eo_bwd_t<N, N, MIR, 1, Mr::NE, Mr::NO, false>(tb.B, qe, qo, h);
      else eo_bwd<N, N, MIR, 1, Mr::NE, Mr::NO, false>(tb.bB, qe, qo, h);
#pragma unroll
      for (int k = 0; k < N; ++k) S[L::Y + L::yo(k, w / N, w % N)] = h[k];
    }
    group_sync<WPE>(0);
    // y' items (k, a): B^T along y
    for (int w = t; w < N * N; w += 32 * WPE / SUB) {
      const int k = w / N, a = w % N;
      double v[N], qe[HP], qo[H], h[N];
#pragma unroll
      for (int b = 0; b < N; ++b) v[b] = S[L::Y + L::yo(k, b, a)];
      eo_qsplit<N>(v, qe, qo);
      if (FT) eo_bwd_t<N, N, MIR, 1, Mr::NE, Mr::NO, false>(tb.B, qe, qo, h);
      else eo_bwd<N, N, MIR, 1, Mr::NE, Mr::NO, false>(tb.bB, qe, qo, h);
#pragma unroll
      for (int j = 0; j < N; ++j) S[L::X + L::xo(k, j, a)] = h[j];
    }
    group_sync<WPE>(0);
    // x' items (k, j): B^T along x, scatter
    if (TM) {
      // the output box of the previous component's reduce-add has been read
      if (t == 0) bulk_wait_read();
      group_sync<WPE>(0);
    }
    for (int w = t; w < N * N; w += 32 * WPE / SUB) {
      const int k = w / N, j = w % N;
      double v[N], qe[HP], qo[H], acc[N];
#pragma unroll
      for (int a = 0; a < N; ++a) v[a] = S[L::X + L::xo(k, j, a)];
      eo_qsplit<N>(v, qe, qo);
      if (FT) eo_bwd_t<N, N, MIR, 1, Mr::NE, Mr::NO, false>(tb.B, qe, qo, acc);
      else eo_bwd<N, N, MIR, 1, Mr::NE, Mr::NO, false>(tb.bB, qe, qo, acc);
      if (TM) {
        // row of the output box; constrained points and the pitch slot get 0
        // (the reduce-add of +0.0 outside the element touches only points no
        // other element of this colour pass owns, or is dropped at the edge)
        const int Z = Z0 + k, Y = Y0 + j;
        if (touches_dirichlet(g, comp, X0, Y0, Z0, N)) {
#pragma unroll
          for (int i = 0; i < N; ++i)
            if (constrained(g, comp, X0 + i, Y, Z)) acc[i] = 0.0;
        }
        if constexpr (N & 1) {
          double2* orow = reinterpret_cast<double2*>(S + L::O + w * L::RP);
          SDME_CHECK(smem_ok(orow, L::RP * 8, 16));
#pragma unroll
          for (int i = 0; i < L::RP / 2; ++i)
            orow[i] = make_double2(acc[2 * i], 2 * i + 1 < N ? acc[2 * i + 1] : 0.0);
        } else {
          // odd P: values at the shift, zeros in the two slots outside the element
          double* orow = S + L::O + w * L::RP;
          const int sh = X0 & 1;
#pragma unroll
          for (int i = 0; i < N; ++i) orow[sh + i] = acc[i];
          orow[N + 1] = 0.0;
          orow[sh ? 0 : N] = 0.0;
        }
        continue;
      }
      if (evb) {
        double* er = evb + ((comp * N + k) * N + j) * N;
#pragma unroll
        for (int i = 0; i < N; ++i) er[i] = acc[i];
        continue;
      }
      const int Z = Z0 + k, Y = Y0 + j;
      const bool chk = touches_dirichlet(g, comp, X0, Y0, Z0, N);
      SDME_CHECK(comp >= 0 && comp < 3 && Z >= 0 && Z < g.Lz && Y >= 0 && Y < g.Ly && X0 >= 0 && X0 + N <= g.Lx);
      double* row = dst + comp * g.Ns + ((long long)Z * g.Ly + Y) * g.Px + X0;
#pragma unroll
      for (int i = 0; i < N; ++i)
        if (!chk || !constrained(g, comp, X0 + i, Y, Z)) red_add(row + i, acc[i]);
    }
    if (TM) fence_proxy_async_smem();
    group_sync<WPE>(0);
    if (TM && t == 0 && ymap) {
      // first write to y of this CTA: the previous launch on the stream (a
      // colour pass, or the zeroing of y) has completed (PDL, tma.cuh)
      if (waited && !*waited) {
        pdl_wait();
        *waited = true;
      }
      tma_reduce_add_box(ymap, S + L::O, X0 & ~1, Y0, Z0, comp);
    }
  }
}

// f_int (MODE_FINT), K.p (+ c_m M p with VAL) from u (MODE_APPLY) or from the
// stored quadrature data (MODE_PA), and that data (MODE_SETUP, from the same
// collocated grad u, so MODE_PA is bit-identical to MODE_APPLY); one warp per
// element, persistent.
// general meshes (GEN): 1D tables without 2/h or det J (reference-coordinate
// gradients), per-point J^-1 and w det J from args.geo, element boxes read
// from / written to E-vector buffers (element_gen.cuh gathers and assembles)
template <int N>
__device__ __forceinline__ void gen_jinv(const double* __restrict__ geo, long long eid, int q, double J[3][3]) {
  constexpr int Q = N * N * N;
  const double* gp = geo + eid * (10 * Q) + q;
#pragma unroll
  for (int d = 0; d < 3; ++d)
#pragma unroll
    for (int c = 0; c < 3; ++c) J[d][c] = __ldg(gp + (d * 3 + c) * Q);
}

// H[i][c] <- sum_d H[i][d] J^-1[d][c]  (reference -> material gradient)
__device__ __forceinline__ void gen_to_phys(double* H, const double J[3][3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double h0 = H[i * 3], h1 = H[i * 3 + 1], h2 = H[i * 3 + 2];
#pragma unroll
    for (int c = 0; c < 3; ++c) H[i * 3 + c] = fma(h0, J[0][c], fma(h1, J[1][c], h2 * J[2][c]));
  }
}

// SUB = 2 (TMA boxes, small N): two elements per warp, one per half-warp,
// each with its own shared region and barriers; the halves run the same
// number of iterations (a half past the end of the colour repeats the last
// element without scattering it) so the warp-wide syncs stay uniform
// SDME_COL_BOX_PREF: L2 prefetch (cp.async.bulk.prefetch.tensor) of the next
// element's u / p boxes (TMA path).  Measured slower (P = 3 K.p 1.937 -> 1.997 ms,
// P = 6 1.949 -> 1.964): off.
#ifndef SDME_COL_BOX_PREF
#define SDME_COL_BOX_PREF 0
#endif
// SDME_GEN_GEO_PREF: L2 prefetch of a general-mesh element's J^-1 table
#ifndef SDME_GEN_GEO_PREF
#define SDME_GEN_GEO_PREF 1
#endif
// SDME_COL_PA_PREF: L2 prefetch of the stored point data (MODE_PA) per element
#ifndef SDME_COL_PA_PREF
#define SDME_COL_PA_PREF 1
#endif

template <int N, int WPE, int MINB, int MODE, bool VAL, int MIR, bool TM = false, bool GEN = false, int SUB = 1,
          bool ISO = false>
__global__ void __launch_bounds__(32 * WPE, MINB) element_col(const __grid_constant__ TabC<N, MIR> tb,
                                                        const __grid_constant__ Geo g, OpArgs args) {
  static_assert(SUB == 1 || (SUB == 2 && WPE == 1 && TM && !GEN), "half-warp elements: TMA path only");
  constexpr bool VALS = VAL;
  using L = ColLay<N, VALS, TM>;
  constexpr int T = 32 * WPE / SUB;
  constexpr int Q = N * N * N, QPT = (Q + T - 1) / T;
  extern __shared__ __align__(128) double smem[];
  const int t = threadIdx.x % T;
  double* S = smem + (threadIdx.x / T) * ColPer<N, VALS, TM>::PERP;
  SDME_CHECK(smem_ok(S, L::PER * 8, 128));
  const long long half = threadIdx.x / T;
  int buf = 0;
  if (args.skip && *(volatile const int*)args.skip) return;
  bool waited = false;  // TM colour passes: griddepcontrol.wait done (thread 0)
  // TM: the next colour pass; E-vector mode: the cluster tail of a small-mesh
  // PCG iteration (pcg_small.cuh); a no-op without a programmatic dependent
  pdl_launch_dependents();
  constexpr bool UPASS = (MODE == MODE_APPLY || MODE == MODE_FINT || MODE == MODE_SETUP);
  constexpr bool PPASS = (MODE == MODE_APPLY || MODE == MODE_PA || MODE == MODE_MASS);
  constexpr bool PGRAD = MODE != MODE_MASS;  // c_m M p alone: values only (B stages), no gradient
  const long long cnt = colour_count(g, args.colour);
  const long long stride = (long long)gridDim.x * SUB;
  const double mu_k = args.c_k * g.mu, lam_k = args.c_k * g.lam;
  const double cmr = args.c_m * g.rho;
  const double* first_field = UPASS ? args.u : args.p;
  const CUtensorMap* umap = static_cast<const CUtensorMap*>(args.tu);
  const CUtensorMap* pmap = static_cast<const CUtensorMap*>(args.tp);
  const CUtensorMap* first_map = UPASS ? umap : pmap;
  unsigned ph = 0;  // TM: mbarrier phase bit per staging buffer
  // weight table W[q] = w_a w_b w_c det J and the box-offset table
  int* tab = reinterpret_cast<int*>(S + L::TAB);
  for (int q = t; q < Q; q += T) {
    S[L::W + q] = tb.wq[q % N] * tb.wq[(q / N) % N] * tb.wq[q / (N * N)] * tb.detJ;
    if (!TM) tab[q] = ((q / (N * N)) * g.Ly + (q / N) % N) * g.Px + q % N;
  }
  if (TM && t == 0) {
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(S + L::BAR);
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
    mbar_fence_init();
  }
  group_sync<WPE>(0);
  if (GEN && (long long)blockIdx.x < cnt) {
    col_stage<N, 32 * WPE>(g, first_field + (long long)blockIdx.x * 3 * Q, 0, 0, 0, 0, S + L::R, t, tab);
  } else if ((long long)blockIdx.x * SUB < cnt) {
    int ei, ej, ek;
    colour_element(g, args.colour, SUB == 1 ? (long long)blockIdx.x : min((long long)blockIdx.x * SUB + half, cnt - 1),
                   ei, ej, ek);
    if (TM) {
      if (t == 0) {
        unsigned long long* bars = reinterpret_cast<unsigned long long*>(S + L::BAR);
        mbar_expect_tx(bars, N * N * L::RP * 8);
        tma_load_box(S + L::R, first_map, ((N - 1) * ei) & ~1, (N - 1) * ej, (N - 1) * ek, 0, bars);
      }
    } else {
      col_stage<N, 32 * WPE>(g, first_field, 0, (N - 1) * ei, (N - 1) * ej, (N - 1) * ek, S + L::R, t, tab);
    }
  }
  for (long long base = (long long)blockIdx.x * SUB; base < cnt; base += stride) {
    const long long idx = SUB == 1 ? base : min(base + half, cnt - 1);
    const bool ghost = SUB > 1 && base + half >= cnt;  // repeats idx, scatters nothing
    int X0 = 0, Y0 = 0, Z0 = 0;
    long long eid = idx, eoff = 0;  // GEN: E-vector box offset of this element
    if (GEN) {
      eoff = idx * 3 * Q;
    } else {
      int ei, ej, ek;
      colour_element(g, args.colour, idx, ei, ej, ek);
      X0 = (N - 1) * ei, Y0 = (N - 1) * ej, Z0 = (N - 1) * ek;
      eid = ((long long)ek * g.ny + ej) * g.nx + ei;
    }
    NextRows nxt{nullptr, 0, 0, 0};
    NextBox nxb{nullptr, 0, 0, 0};
    long long next_eid = -1;
    if (base + stride < cnt) {
      if (GEN) {
        nxt = NextRows{first_field + (idx + stride) * 3 * Q, 0, 0, 0};
        next_eid = idx + stride;
      } else {
        int ni, nj, nk;
        colour_element(g, args.colour, SUB == 1 ? idx + stride : min(base + stride + half, cnt - 1), ni, nj, nk);
        next_eid = ((long long)nk * g.ny + nj) * g.nx + ni;
        if (TM) {
          nxb = NextBox{first_map, (N - 1) * ni, (N - 1) * nj, (N - 1) * nk};
          if (SDME_COL_BOX_PREF && t == 0) {
            // the next element's input boxes on their way into L2 an element
            // ahead of their TMA loads
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              if (UPASS) tma_prefetch_box(umap, nxb.X0 & ~1, nxb.Y0, nxb.Z0, c);
              if (PPASS) tma_prefetch_box(pmap, nxb.X0 & ~1, nxb.Y0, nxb.Z0, c);
            }
          }
        }
        else nxt = NextRows{first_field, (N - 1) * ni, (N - 1) * nj, (N - 1) * nk};
      }
    }
    if (GEN && SDME_GEN_GEO_PREF && MODE != MODE_MASS) {
      // general meshes: the element's J^-1 and w det J (10 Q doubles, read at the
      // points) on their way into L2 while the forward pass runs
      constexpr int LG = (10 * Q * 8 + 127) / 128 + 1;
      const char* bp = reinterpret_cast<const char*>(args.geo + eid * (10 * Q));
      for (int l = t; l < LG; l += T) prefetch_l2(bp + (l * 128 < 10 * Q * 8 - 8 ? l * 128 : 10 * Q * 8 - 8));
    }
    double Hu[QPT][9];
    if (UPASS) {
      const NextRows after_u = MODE == MODE_APPLY ? NextRows{args.p + eoff, X0, Y0, Z0} : nxt;
      const NextBox after_ub = MODE == MODE_APPLY ? NextBox{pmap, X0, Y0, Z0} : nxb;
      col_forward<N, WPE, MIR, false, VALS, TM, SUB, ISO>(tb, args.zero, g, args.u + eoff, X0, Y0, Z0, S, t, &buf, after_u, true, umap,
                                                after_ub, &ph);
#pragma unroll
      for (int r = 0; r < QPT; ++r) {
        const int q = t + r * T;
        if (q < Q) {
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int d = 0; d < 3; ++d) Hu[r][i * 3 + d] = S[L::qi(d, i, q)];
          if constexpr (GEN) {
            double J[3][3];
            gen_jinv<N>(args.geo, eid, q, J);
            gen_to_phys(Hu[r], J);
          }
        }
      }
      group_sync<WPE>(0);
    }
    if (MODE == MODE_PA && SDME_COL_PA_PREF) {
      // the element's stored point data (K, ln J: 80 Q bytes, 16-byte aligned)
      // on its way into L2 while the forward pass of p runs (2: the next
      // element's, a whole element ahead)
      constexpr int LPE = (kQpSlots * Q * 8 + 127) / 128 + 1;
      const bool first_it = base == (long long)blockIdx.x * SUB;
      if (SDME_COL_PA_PREF == 1 || first_it) {
        const char* bp = reinterpret_cast<const char*>(args.qpd + eid * (kQpSlots * Q));
        for (int l = t; l < LPE; l += T) prefetch_l2(bp + (l * 128 < kQpSlots * Q * 8 - 8 ? l * 128 : kQpSlots * Q * 8 - 8));
      }
      if (SDME_COL_PA_PREF == 2 && next_eid >= 0) {
        const char* bp = reinterpret_cast<const char*>(args.qpd + next_eid * (kQpSlots * Q));
        for (int l = t; l < LPE; l += T) prefetch_l2(bp + (l * 128 < kQpSlots * Q * 8 - 8 ? l * 128 : kQpSlots * Q * 8 - 8));
      }
    }
    if (PPASS)
      col_forward<N, WPE, MIR, VAL, VALS, TM, SUB, ISO>(tb, args.zero, g, args.p + eoff, X0, Y0, Z0, S, t, &buf, nxt, PGRAD, pmap, nxb,
                                              &ph);
#pragma unroll
    for (int r = 0; r < QPT; ++r) {
      const int q = t + r * T;
      if (q >= Q) continue;
      const double wdet = GEN ? __ldg(args.geo + eid * (10 * Q) + 9 * Q + q) : S[L::W + q];
      if (MODE == MODE_MASS) {
#pragma unroll
        for (int i = 0; i < 3; ++i) S[L::qi(3, i, q)] *= cmr * wdet;
        continue;
      }
      QpK s;
      if (MODE == MODE_PA) {
        const double* qd = args.qpd + eid * (kQpSlots * Q) + q;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) s.K[i][d] = __ldg(qd + (i * 3 + d) * Q);
        s.lnJ = __ldg(qd + 9 * Q);
      } else {
        qp_k(Hu[r], s);
        if (!(s.det > 0.0)) {
          const int a = q % N, b = (q / N) % N, c = q / (N * N);
          const long long ref = (GEN && args.elem_id) ? (long long)__ldg(args.elem_id + eid) : eid;
          atomicMin(args.inv_flag, (unsigned long long)ref * Q + (unsigned long long)((a * N + b) * N + c));
        }
      }
      if (MODE == MODE_SETUP) {
        double* qd = args.qpd + eid * (kQpSlots * Q) + q;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) qd[(i * 3 + d) * Q] = s.K[i][d];
        qd[9 * Q] = s.lnJ;
        continue;
      }
      if (MODE == MODE_FINT && GEN) {
        // flux back to the reference axes: wdet * P J^-T
        const double cK = g.lam * s.lnJ - g.mu;
        double J[3][3];
        gen_jinv<N>(args.geo, eid, q, J);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          double Pi[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) Pi[c] = fma(g.mu, s.F[i][c], cK * s.K[i][c]);
#pragma unroll
          for (int d = 0; d < 3; ++d) S[L::qi(d, i, q)] = wdet * fma(Pi[0], J[d][0], fma(Pi[1], J[d][1], Pi[2] * J[d][2]));
        }
      } else if (MODE == MODE_FINT) {
        const double cK = g.lam * s.lnJ - g.mu;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) S[L::qi(d, i, q)] = wdet * fma(g.mu, s.F[i][d], cK * s.K[i][d]);
      } else {
        double Hp[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) Hp[i][d] = S[L::qi(d, i, q)];
        double Jg[3][3];
        if constexpr (GEN) {
          gen_jinv<N>(args.geo, eid, q, Jg);
          gen_to_phys(&Hp[0][0], Jg);
        }
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
        const double cc = mu_k - lam_k * s.lnJ;
        const double lt = lam_k * tr;
        if constexpr (GEN) {
#pragma unroll
          for (int i = 0; i < 3; ++i) {
            double Pi[3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const double m2 = fma(M1[i][0], s.K[0][c], fma(M1[i][1], s.K[1][c], M1[i][2] * s.K[2][c]));
              Pi[c] = fma(cc, m2, fma(lt, s.K[i][c], mu_k * Hp[i][c]));
            }
#pragma unroll
            for (int d = 0; d < 3; ++d)
              S[L::qi(d, i, q)] = wdet * fma(Pi[0], Jg[d][0], fma(Pi[1], Jg[d][1], Pi[2] * Jg[d][2]));
          }
        } else {
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              const double m2 = fma(M1[i][0], s.K[0][d], fma(M1[i][1], s.K[1][d], M1[i][2] * s.K[2][d]));
              S[L::qi(d, i, q)] = wdet * fma(cc, m2, fma(lt, s.K[i][d], mu_k * Hp[i][d]));
            }
        }
        if (VAL) {
#pragma unroll
          for (int i = 0; i < 3; ++i) S[L::qi(3, i, q)] *= cmr * wdet;
        }
      }
    }
    group_sync<WPE>(0);
    if (MODE == MODE_SETUP) continue;
    double* evb = args.ev ? args.ev + eid * 3 * Q : nullptr;
    col_backward<N, WPE, MIR, VAL, VALS, TM, SUB, ISO>(tb, args.zero, g, args.y, X0, Y0, Z0, S, t, evb, PGRAD,
                                                  ghost ? nullptr : static_cast<const CUtensorMap*>(args.ty),
                                                  &waited);
  }
  // the reduce-adds have completed before the CTA (and its shared memory) retires
  if (TM && t == 0) bulk_wait_all();
}

}  // namespace sdme
