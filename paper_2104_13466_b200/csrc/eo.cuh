// Even-odd decomposition of the 1D contractions (sum factorisation).
//
// Every basis of the reference has a mirror symmetry at a symmetric Gauss rule
// (checked on the host, tools/run_configs.py & sdme_abi.cu:make_eo): in
// lattice-local order there is an involution sigma of the functions and
// signs s with
//   B[m-1-a][l] =  s_l B[a][sigma(l)],   D[m-1-a][l] = -s_l D[a][sigma(l)].
// Nodal GLL (MIR = 0): sigma(l) = n-1-l, s = +1.  Modal Jacobi / SDME with
// parity-split internal modes (MIR = 1): sigma swaps the two vertices and fixes
// the internal modes, s = +1, -1, +1, ... along l = 1..n-2.
// A contraction out = T v then needs only the "even" and "odd" combinations
// of the inputs and the mirrored output pairs:
//   S[a] = out[a] + out[m-1-a] = sum_e TS[a][e] E[e],   Dt[a] = out[a] - out[m-1-a] = sum_o TT[a][o] O[o]
// which roughly halves the multiply-adds (13 instead of 25 at n = m = 5;
// 41 instead of 81 at n = m = 9).  D-type operators (mirror sign -s) swap the
// roles of the E and O combinations.  The transposed (backward) contraction
// uses the same structure on the point side.  Tables are folded by 1/2 on
// the host so reconstruction is a single add / subtract.
#pragma once

namespace sdme {

template <int N, int MIR>
struct Mir {
  __host__ __device__ static constexpr int sig(int l) {
    return MIR == 0 ? N - 1 - l : (l == 0 ? N - 1 : (l == N - 1 ? 0 : l));
  }
  __host__ __device__ static constexpr int sg(int l) {
    return MIR == 0 ? 1 : ((l == 0 || l == N - 1) ? 1 : ((l % 2) ? 1 : -1));
  }
  __host__ __device__ static constexpr int count(int kind) {  // 0 pairs, 1 fixed +, 2 fixed -
    int c = 0;
    for (int l = 0; l < N; ++l) {
      const int r = sig(l);
      if (kind == 0 && l < r) ++c;
      if (kind == 1 && l == r && sg(l) > 0) ++c;
      if (kind == 2 && l == r && sg(l) < 0) ++c;
    }
    return c;
  }
  __host__ __device__ static constexpr int nth(int kind, int k) {
    int c = 0;
    for (int l = 0; l < N; ++l) {
      const int r = sig(l);
      const bool hit = (kind == 0 && l < r) || (kind == 1 && l == r && sg(l) > 0) ||
                       (kind == 2 && l == r && sg(l) < 0);
      if (hit) {
        if (c == k) return l;
        ++c;
      }
    }
    return -1;
  }
  static constexpr int NP = count(0), NFP = count(1), NFM = count(2);
  static constexpr int NE = NP + NFP;  // B-type even set (pair reps, fixed +)
  static constexpr int NO = NP + NFM;  // B-type odd set (pair reps, fixed -)
};

template <int M>
struct Half {
  static constexpr int H = M / 2, HP = (M + 1) / 2;
};

// forward tables of one operator: S rows HP x WS, T rows H x WT
template <int M, int WS, int WT>
struct EoFwd {
  double S[Half<M>::HP][WS > 0 ? WS : 1];
  double T[Half<M>::H > 0 ? Half<M>::H : 1][WT > 0 ? WT : 1];
};
// backward tables of one operator: YE rows WE x HP (point side), YO rows WO x H
template <int M, int WE, int WO>
struct EoBwd {
  double E[WE > 0 ? WE : 1][Half<M>::HP];
  double O[WO > 0 ? WO : 1][Half<M>::H > 0 ? Half<M>::H : 1];
};

template <int N, int M, int MIR>
struct TabEO {
  using Mr = Mir<N, MIR>;
  static constexpr int NE = Mr::NE, NO = Mr::NO;
  EoFwd<M, NE, NO> B;                 // forward values (B-type)
  EoFwd<M, NO, NE> Dx, Dy, Dz;        // forward physical derivatives (D-type)
  EoBwd<M, NE, NO> bBx, bBy, bBz;     // backward B w (z: det J), B-type
  EoBwd<M, NO, NE> bDx, bDy, bDz;     // backward D w 2/h (z: det J), D-type
};

// E/O combinations of an input pencil (B-type sets)
template <int N, int MIR>
__device__ __forceinline__ void eo_split(const double (&v)[N], double (&E)[Mir<N, MIR>::NE > 0 ? Mir<N, MIR>::NE : 1],
                                         double (&O)[Mir<N, MIR>::NO > 0 ? Mir<N, MIR>::NO : 1]) {
  using Mr = Mir<N, MIR>;
#pragma unroll
  for (int p = 0; p < Mr::NP; ++p) {
    const int l = Mr::nth(0, p), r = Mr::sig(l);
    if (Mr::sg(l) > 0) {
      E[p] = v[l] + v[r];
      O[p] = v[l] - v[r];
    } else {
      E[p] = v[l] - v[r];
      O[p] = v[l] + v[r];
    }
  }
#pragma unroll
  for (int f = 0; f < Mr::NFP; ++f) E[Mr::NP + f] = v[Mr::nth(1, f)];
#pragma unroll
  for (int f = 0; f < Mr::NFM; ++f) O[Mr::NP + f] = v[Mr::nth(2, f)];
}

// out = T v from the combinations (B-type: (ES, ET) = (E, O); D-type: (O, E))
template <int M, int WS, int WT>
__device__ __forceinline__ void eo_fwd(const EoFwd<M, WS, WT>& t, const double* ES, const double* ET,
                                       double (&out)[M]) {
  constexpr int H = Half<M>::H;
#pragma unroll
  for (int a = 0; a < H; ++a) {
    double s = 0.0, d = 0.0;
#pragma unroll
    for (int e = 0; e < WS; ++e) s = fma(t.S[a][e], ES[e], s);
#pragma unroll
    for (int o = 0; o < WT; ++o) d = fma(t.T[a][o], ET[o], d);
    out[a] = s + d;
    out[M - 1 - a] = s - d;
  }
  if (M % 2) {
    double s = 0.0;
#pragma unroll
    for (int e = 0; e < WS; ++e) s = fma(t.S[H][e], ES[e], s);
    out[H] = s;
  }
}

// point-side combinations of a backward input q[M]
template <int M>
__device__ __forceinline__ void eo_qsplit(const double (&q)[M], double (&qe)[Half<M>::HP],
                                          double (&qo)[Half<M>::H > 0 ? Half<M>::H : 1]) {
  constexpr int H = Half<M>::H;
#pragma unroll
  for (int a = 0; a < H; ++a) {
    qe[a] = q[a] + q[M - 1 - a];
    qo[a] = q[a] - q[M - 1 - a];
  }
  if (M % 2) qe[H] = q[H];
}

// Reconstruction of y = T^T q from the even / odd partial sums YE (WE) and
// YO (WO) of a B-type (F = +1) or D-type (F = -1) operator; y accumulated
// (ACC) or set.  For D-type the mirror sign is -s, so the fixed sets swap.
template <int N, int MIR, int F, int WE, int WO, bool ACC>
__device__ __forceinline__ void eo_recon(const double* YE, const double* YO, double (&y)[N]) {
  using Mr = Mir<N, MIR>;
#pragma unroll
  for (int p = 0; p < Mr::NP; ++p) {
    const int l = Mr::nth(0, p), r = Mr::sig(l);
    const double lo = YE[p] + YO[p], hi = YE[p] - YO[p];
    const bool plus = (F * Mr::sg(l)) > 0;
    if (ACC) {
      y[l] += lo;
      y[r] += plus ? hi : -hi;
    } else {
      y[l] = lo;
      y[r] = plus ? hi : -hi;
    }
  }
  constexpr int NFE = F > 0 ? Mr::NFP : Mr::NFM;  // fixed points in this type's even set
  constexpr int NFO = F > 0 ? Mr::NFM : Mr::NFP;
#pragma unroll
  for (int f = 0; f < NFE; ++f) {
    const int l = Mr::nth(F > 0 ? 1 : 2, f);
    if (ACC) y[l] += YE[Mr::NP + f];
    else y[l] = YE[Mr::NP + f];
  }
#pragma unroll
  for (int f = 0; f < NFO; ++f) {
    const int l = Mr::nth(F > 0 ? 2 : 1, f);
    if (ACC) y[l] += YO[Mr::NP + f];
    else y[l] = YO[Mr::NP + f];
  }
}

// y = T^T q for a B-type (F = +1) or D-type (F = -1) operator, y accumulated (ACC) or set
template <int N, int M, int MIR, int F, int WE, int WO, bool ACC>
__device__ __forceinline__ void eo_bwd(const EoBwd<M, WE, WO>& t, const double (&qe)[Half<M>::HP],
                                       const double (&qo)[Half<M>::H > 0 ? Half<M>::H : 1], double (&y)[N]) {
  constexpr int H = Half<M>::H, HP = Half<M>::HP;
  double YE[WE > 0 ? WE : 1], YO[WO > 0 ? WO : 1];
#pragma unroll
  for (int e = 0; e < WE; ++e) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < HP; ++a) s = fma(t.E[e][a], qe[a], s);
    YE[e] = s;
  }
#pragma unroll
  for (int o = 0; o < WO; ++o) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < H; ++a) s = fma(t.O[o][a], qo[a], s);
    YO[o] = s;
  }
  eo_recon<N, MIR, F, WE, WO, ACC>(YE, YO, y);
}

// y = T^T q of a B-type (F = +1) or D-type (F = -1) operator read from its
// *forward* tables: make_tabc stores the backward tables as their exact
// transposes (bwd E[e][a] = fwd S[a][e], O[o][a] = T[a][o]), so this is
// eo_bwd bit for bit with half as many distinct table constants
template <int N, int M, int MIR, int F, int WE, int WO, bool ACC>
__device__ __forceinline__ void eo_bwd_t(const EoFwd<M, WE, WO>& t, const double (&qe)[Half<M>::HP],
                                         const double (&qo)[Half<M>::H > 0 ? Half<M>::H : 1], double (&y)[N]) {
  constexpr int H = Half<M>::H, HP = Half<M>::HP;
  double YE[WE > 0 ? WE : 1], YO[WO > 0 ? WO : 1];
#pragma unroll
  for (int e = 0; e < WE; ++e) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < HP; ++a) s = fma(t.S[a][e], qe[a], s);
    YE[e] = s;
  }
#pragma unroll
  for (int o = 0; o < WO; ++o) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < H; ++a) s = fma(t.T[a][o], qo[a], s);
    YO[o] = s;
  }
  eo_recon<N, MIR, F, WE, WO, ACC>(YE, YO, y);
}

}  // namespace sdme
