// Operator dispatch and launch shapes for one polynomial order P (compiled
// once per P with -DSDME_ORDER=P by build.py, in parallel): element kernels
// (f_int, K.p, mass) and the Jacobi diagonal for m in {P+1, P+2}.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "ctx.cuh"
#include "element_col.cuh"
#include "element_diag.cuh"
#include "element_eo.cuh"
#include "element_gen.cuh"
#include "element_kernels.cuh"
#include "element_q5.cuh"
#include "element_q5d.cuh"
#include "element_v3.cuh"
#include "pcg_small.cuh"

#ifndef SDME_COL_MINB
#define SDME_COL_MINB 11  // resident 1-warp blocks per SM for the P = 4 collocated kernels
#endif

#ifndef SDME_Q5_MINB
#define SDME_Q5_MINB 3  // resident 4-warp quintet blocks per SM of the P = 4 kernel (168 registers)
#endif

#ifndef SDME_TMB_MINB
#define SDME_TMB_MINB 7  // max resident 2-warp blocks per SM of the TMA all-component kernels
#endif

#ifndef SDME_GEN_MINB
// resident blocks per SM asked of the general-mesh P = 4 kernels: K.p from u
// at the 168-register cap of 11-12 warps (12.5 -> 13.5 GDOF/s at 32^3,
// tools/gen_mesh_bench.py); f_int and the stored-data operator unconstrained
// (188 registers; the PA operator is 5% slower at the cap)
#define SDME_GEN_MINB 1
#endif
#ifndef SDME_GEN_APPLY_MINB
#define SDME_GEN_APPLY_MINB 11
#endif

#ifndef SDME_ORDER
#error "compile with -DSDME_ORDER=P"
#endif

using namespace sdme;
using Ops = SdmeOps;

namespace {

constexpr int kMaxDevices = 64;

// One cached value per CUDA device: kernel attributes (dynamic shared memory
// opt-in) and occupancy are per device, so they are set / queried for the
// device current at the launch, never assumed to be device 0.
struct PerDevice {
  int v[kMaxDevices];
  PerDevice() {
    for (int& x : v) x = -1;
  }
};

inline int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return (dev >= 0 && dev < kMaxDevices) ? dev : 0;
}

// resident CTAs of ``kern`` over the whole current device (persistent grid cap)
template <class K>
int resident_grid(PerDevice& cache, K kern, int threads, int smem) {
  const int dev = current_device();
  int& mb = cache.v[dev];
  if (mb < 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, smem);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    mb = std::max(1, nb) * sms;
  }
  return mb;
}

// v3 tables: weights, det J and dxi/dX folded per axis (element_v3.cuh)
template <int N, int M>
Tab3<N, M> make_tab3(const sdme_ctx* c) {
  Tab3<N, M> t;
  const Geo& g = c->geo;
  for (int a = 0; a < M; ++a) {
    const double w = c->w[a];
    for (int l = 0; l < N; ++l) {
      const double b = c->Bl[a * N + l], d = c->Dl[a * N + l];
      t.B[a][l] = b;
      t.Dx[a][l] = d * g.s[0];
      t.Dy[a][l] = d * g.s[1];
      t.Dz[a][l] = d * g.s[2];
      t.bBx[a][l] = b * w;
      t.bDx[a][l] = d * w * g.s[0];
      t.bBy[a][l] = b * w;
      t.bDy[a][l] = d * w * g.s[1];
      t.bBz[a][l] = b * w * g.detJ;
      t.bDz[a][l] = d * w * g.s[2] * g.detJ;
    }
  }
  return t;
}

// Launch shape of the v3 element kernels.  WPE warps per element, EPB
// elements per block, NC components per contraction stage, MINB minimum
// resident blocks per SM (register cap for __launch_bounds__).
template <int N, int M, int WPE_, int NC_, int EPB_, int MINB_, bool STG_ = false>
struct Shape {
  static constexpr int WPE = WPE_, NC = NC_, EPB = EPB_, MINB = MINB_;
  static constexpr bool STG = STG_;  // cp.async row staging (NC == 1)
};

template <int N, int M>
struct DefaultShape {
  static constexpr int bytes = V3<N, M, 1, 3>::PER * 8;
  static constexpr int WPE = bytes <= 40960 ? 1 : (bytes <= 65536 ? 4 : 8);
  // resident 2-warp blocks per SM for P = 2, 3 at m = P + 1 (register cap
  // 128 / 168: 16 / 12 warps per SM; tools/prof_c3.py), else unconstrained
  static constexpr int MINB = (N == 3 && M == 3) ? 8 : ((N == 4 && M == 4) ? 6 : 1);
  using type = Shape<N, M, WPE, 3, (WPE == 1 ? 2 : 1), MINB>;
};

// E-vector mode: y += gathered element boxes (after the single element launch)
template <int N>
void ev_gather(sdme_ctx* c, const OpArgs& a) {
  ++c->launches;  // the element launch
  const long long n = 3 * c->geo.Ns;
  const unsigned grid = (unsigned)std::min<long long>((n + 255) / 256, 148LL * 8);
  k_ev_gather<N><<<grid, 256, 0, c->st>>>(a.y, c->d_ev, c->geo, a.skip);
  ++c->launches;
}

template <int N, int M, class S, int MODE, bool VAL, class TB, bool TMB>
void launch_v3_k(sdme_ctx* c, const TB& tb, OpArgs a) {
  constexpr bool VALS = VAL || MODE == MODE_MASS;
  constexpr int smem = V3Smem<N, M, S::WPE, S::NC, VALS, S::STG, TMB>::PERS * 8 * S::EPB;
  constexpr int MINB = TMB && S::MINB > SDME_TMB_MINB ? SDME_TMB_MINB : S::MINB;  // TMA boxes: register cap (see DESIGN)
  auto kern = element_v3<N, M, S::WPE, S::NC, S::EPB, MINB, MODE, VAL, S::STG, TB, TMB>;
  static PerDevice grid_cache;  // per device: attribute + occupancy set once
  const int max_blocks = resident_grid(grid_cache, kern, S::EPB * S::WPE * 32, smem);
  if (MODE == MODE_SETUP || MODE == MODE_ENERGY) {
    // no scatter: one pass over all elements
    a.colour = -1;
    const long long need = (colour_count(c->geo, -1) + S::EPB - 1) / S::EPB;
    kern<<<(unsigned)std::min<long long>(need, max_blocks), S::EPB * S::WPE * 32, smem, c->st>>>(tb, c->geo, a);
    ++c->launches;
    return;
  }
  if (c->ev_mode) {
    a.colour = -1;
    a.ev = c->d_ev;
    const long long need = (colour_count(c->geo, -1) + S::EPB - 1) / S::EPB;
    kern<<<(unsigned)std::min<long long>(need, max_blocks), S::EPB * S::WPE * 32, smem, c->st>>>(tb, c->geo, a);
    if (c->ev_no_gather) ++c->launches;
    else ev_gather<N>(c, a);
    return;
  }
  for (int sp = 0; sp < 8 * c->nslab; ++sp) {
    const int col = colour_code(c->geo, sp % 8, sp / 8, c->nslab);
    if (col == -2) continue;
    const long long cnt = colour_count(c->geo, col);
    if (cnt == 0) continue;
    a.colour = col;
    const long long need = (cnt + S::EPB - 1) / S::EPB;
    const unsigned grid = (unsigned)std::min<long long>(need, max_blocks);
    kern<<<grid, S::EPB * S::WPE * 32, smem, c->st>>>(tb, c->geo, a);
    ++c->launches;
  }
}

// TMA element boxes for the all-component shape (small P) with even-odd
// tables on colour passes, when every vector of the mode has a tensor map;
// SDME_VARIANT=11 keeps the per-lane loads and RED (A/B only)
template <int N, int M, class S, int MODE, bool VAL, class TB = Tab3<N, M>>
void launch_v3(sdme_ctx* c, const TB& tb, OpArgs a) {
  constexpr bool tmb_ok = S::NC == 3 && S::WPE == 1 && !S::STG && !std::is_same<TB, Tab3<N, M>>::value &&
                          MODE != MODE_ENERGY;
  if constexpr (tmb_ok) {
    const bool maps = MODE == MODE_SETUP ? a.tu != nullptr
                                         : (a.ty && (MODE == MODE_PA || MODE == MODE_MASS || a.tu) &&
                                            (MODE == MODE_FINT || a.tp));
    if (maps && !c->ev_mode && c->variant != 11) {
      launch_v3_k<N, M, S, MODE, VAL, TB, true>(c, tb, a);
      return;
    }
  }
  launch_v3_k<N, M, S, MODE, VAL, TB, false>(c, tb, a);
}

template <int N, int M, class S, class TB = Tab3<N, M>>
void element_shape(sdme_ctx* c, int mode, const TB& tb, OpArgs a) {
  if (mode == MODE_SETUP) launch_v3<N, M, S, MODE_SETUP, false, TB>(c, tb, a);
  else if (mode == MODE_ENERGY) launch_v3<N, M, S, MODE_ENERGY, false, TB>(c, tb, a);
  else if (mode == MODE_PA && a.c_m != 0.0) launch_v3<N, M, S, MODE_PA, true, TB>(c, tb, a);
  else if (mode == MODE_PA) launch_v3<N, M, S, MODE_PA, false, TB>(c, tb, a);
  else if (mode == MODE_FINT) launch_v3<N, M, S, MODE_FINT, false, TB>(c, tb, a);
  else if (mode == MODE_APPLY && a.c_m != 0.0) launch_v3<N, M, S, MODE_APPLY, true, TB>(c, tb, a);
  else if (mode == MODE_APPLY) launch_v3<N, M, S, MODE_APPLY, false, TB>(c, tb, a);
  else launch_v3<N, M, S, MODE_MASS, true, TB>(c, tb, a);
}

// Even-odd forward / backward tables of one 1D operator T (m x n, rows =
// points, columns = lattice-local functions) with the mirror structure
// Mir<n, MIR>: pairs first, then the fixed points whose sign (F * s) is + (even
// set) or - (odd set); F = +1 for B-type, -1 for D-type operators.  Folded by
// 1/2 so the reconstruction is one add / subtract (eo.cuh).
template <int N, int M, int MIR>
struct EoBuild {
  using Mr = Mir<N, MIR>;
  static constexpr int H = M / 2, HP = (M + 1) / 2;
  static int set_of(int F, bool even, int idx) {
    if (idx < Mr::NP) return Mr::nth(0, idx);
    const int kind = (F > 0) == even ? 1 : 2;
    return Mr::nth(kind, idx - Mr::NP);
  }
  template <class Dst>
  static void fwd(Dst& dst, const double (&T)[M][N], int F) {
    constexpr int WS = sizeof(dst.S[0]) / sizeof(double), WT = sizeof(dst.T[0]) / sizeof(double);
    const int nS = F > 0 ? Mr::NE : Mr::NO, nT = F > 0 ? Mr::NO : Mr::NE;
    for (int a = 0; a < HP; ++a)
      for (int e = 0; e < WS; ++e) {
        double v = 0.0;
        if (e < nS) {
          const int l = set_of(F, true, e), r = Mr::sig(l);
          v = e < Mr::NP ? 0.5 * (T[a][l] + F * Mr::sg(l) * T[a][r]) : T[a][l];
        }
        dst.S[a][e] = v;
      }
    for (int a = 0; a < H; ++a)
      for (int o = 0; o < WT; ++o) {
        double v = 0.0;
        if (o < nT) {
          const int l = set_of(F, false, o), r = Mr::sig(l);
          v = o < Mr::NP ? 0.5 * (T[a][l] - F * Mr::sg(l) * T[a][r]) : T[a][l];
        }
        dst.T[a][o] = v;
      }
  }
  template <class Dst>
  static void bwd(Dst& dst, const double (&T)[M][N], int F) {
    constexpr int WE = sizeof(dst.E) / sizeof(dst.E[0]), WO = sizeof(dst.O) / sizeof(dst.O[0]);
    const int nE = F > 0 ? Mr::NE : Mr::NO, nO = F > 0 ? Mr::NO : Mr::NE;
    for (int e = 0; e < WE; ++e)
      for (int a = 0; a < HP; ++a) {
        double v = 0.0;
        if (e < nE) {
          const int l = set_of(F, true, e);
          v = (a < H) ? 0.5 * (T[a][l] + T[M - 1 - a][l]) : T[a][l];
        }
        dst.E[e][a] = v;
      }
    for (int o = 0; o < WO; ++o)
      for (int a = 0; a < (H > 0 ? H : 1); ++a) {
        double v = 0.0;
        if (o < nO && a < H) {
          const int l = set_of(F, false, o);
          v = 0.5 * (T[a][l] - T[M - 1 - a][l]);
        }
        dst.O[o][a] = v;
      }
  }
};

// backward tables of a square (M = N) operator as the transposed forward ones
template <int M, int WS, int WT>
void eo_transpose(EoBwd<M, WS, WT>& b, const EoFwd<M, WS, WT>& f) {
  for (int e = 0; e < (WS > 0 ? WS : 1); ++e)
    for (int a = 0; a < Half<M>::HP; ++a) b.E[e][a] = f.S[a][e];
  for (int o = 0; o < (WT > 0 ? WT : 1); ++o)
    for (int a = 0; a < (Half<M>::H > 0 ? Half<M>::H : 1); ++a) b.O[o][a] = f.T[a][o];
}

// Even-odd tables (eo.cuh) from the lattice-order 1D tables, with the same
// folding of weights, det J and 2/h as make_tab3.
template <int N, int M, int MIR>
TabEO<N, M, MIR> make_tabeo(const sdme_ctx* c) {
  const Geo& g = c->geo;
  double Bv[M][N], Dv[3][M][N], bB[3][M][N], bD[3][M][N];
  for (int a = 0; a < M; ++a)
    for (int l = 0; l < N; ++l) {
      const double b = c->Bl[a * N + l], d = c->Dl[a * N + l], w = c->w[a];
      Bv[a][l] = b;
      for (int ax = 0; ax < 3; ++ax) {
        const double jz = ax == 2 ? g.detJ : 1.0;
        Dv[ax][a][l] = d * g.s[ax];
        bB[ax][a][l] = b * w * jz;
        bD[ax][a][l] = d * w * g.s[ax] * jz;
      }
    }
  using EB = EoBuild<N, M, MIR>;
  auto fwd = [](auto& dst, const double (&T)[M][N], int F) { EB::fwd(dst, T, F); };
  auto bwd = [](auto& dst, const double (&T)[M][N], int F) { EB::bwd(dst, T, F); };
  TabEO<N, M, MIR> t;
  fwd(t.B, Bv, 1);
  fwd(t.Dx, Dv[0], -1);
  fwd(t.Dy, Dv[1], -1);
  fwd(t.Dz, Dv[2], -1);
  bwd(t.bBx, bB[0], 1);
  bwd(t.bBy, bB[1], 1);
  bwd(t.bBz, bB[2], 1);
  bwd(t.bDx, bD[0], -1);
  bwd(t.bDy, bD[1], -1);
  bwd(t.bDz, bD[2], -1);
  return t;
}



// Component-serial staged shape for P >= 5: enough warps per element that the
// element's shared memory (points, stage scratch, staged rows) is shared by
// 4 or 8 warps.
template <int N, int M>
struct LargeShape {
  // enough warps that one round covers a stage's M^2 (or N M) pencils
  static constexpr int WPE = (M * M + 31) / 32 > 8 ? 8 : (M * M + 31) / 32;
  using type = Shape<N, M, WPE, 1, 1, 1, true>;
};

// even-odd tables when the 1D tables mirror (ctx->mir), else the plain ones
template <int N, int M, class S>
void element_eo_or_plain(sdme_ctx* c, int mode, const Tab3<N, M>& tb, OpArgs a) {
  if (c->mir == 0)
    element_shape<N, M, S>(c, mode, make_tabeo<N, M, 0>(c), a);
  else if (c->mir == 1)
    element_shape<N, M, S>(c, mode, make_tabeo<N, M, 1>(c), a);
  else
    element_shape<N, M, S>(c, mode, tb, a);
}

template <int N, int MIR>
void col_modes(sdme_ctx* c, int mode, OpArgs a);

// every vector of the mode has a TMA tensor map (launch_col's box path)
inline bool col_tma_ok(const sdme_ctx* c, int mode, const OpArgs& a) {
  if (c->variant == 11) return false;
  if (mode == MODE_SETUP) return a.tu != nullptr;
  return a.ty && (mode == MODE_PA || mode == MODE_MASS || a.tu) && (mode == MODE_FINT || a.tp);
}

template <int N, int M>
void element_impl(sdme_ctx* c, int mode, const double* u, const double* p, double* y, double ck, double cm) {
  const Tab3<N, M> tb = make_tab3<N, M>(c);
  OpArgs a{u, p, y, ck, cm, 0, c->d_flag, c->cur_skip};
  a.qpd = mode == MODE_ENERGY ? y : c->d_qpd;  // MODE_ENERGY: y is the per-element energy buffer
  a.tu = sdme_tmap_of(c, u);
  a.tp = sdme_tmap_of(c, p);
  a.ty = mode == MODE_ENERGY ? nullptr : sdme_tmap_of(c, y);
  if constexpr (N <= 5) {
    // E-vector mode (small meshes, one launch over all elements): latency
    // shape, four warps per element, all three components per stage
    if (c->ev_mode && c->variant != 6) {
      element_eo_or_plain<N, M, Shape<N, M, 4, 3, 1, 1>>(c, mode, tb, a);
      return;
    }
  }
  if constexpr (N == 5 && M == 5) {
    // P = 4, m = 5 (BASELINE config 2); schedule history in profiles/variants_r01.txt
    // (the 3-component, 12-warp and unstaged shapes measured there are template
    // arguments of this same kernel; the rejected column-resident v4 and
    // column-fused v5 were removed).
    using SK = Shape<N, M, 1, 1, 1, 11, true>;
    // f_int and K.p: collocated sum factorisation (element_col.cuh) unless
    // SDME_VARIANT=10; other modes and non-mirrored tables: component-serial,
    // cp.async-staged rows, even-odd contractions, 11 warps/SM
    if ((mode == MODE_FINT || mode == MODE_APPLY || mode == MODE_PA || mode == MODE_SETUP || mode == MODE_MASS) &&
        c->variant != 10 && c->mir >= 0) {
      if (c->mir == 0) col_modes<N, 0>(c, mode, a);
      else col_modes<N, 1>(c, mode, a);
      return;
    }
    element_eo_or_plain<N, M, SK>(c, mode, tb, a);
    return;
  } else if constexpr (N >= 6) {
    if constexpr (N == M) {
      if ((mode == MODE_FINT || mode == MODE_APPLY || mode == MODE_PA || mode == MODE_SETUP || mode == MODE_MASS) &&
          c->variant != 10 && c->mir >= 0) {
        if (c->mir == 0) col_modes<N, 0>(c, mode, a);
        else col_modes<N, 1>(c, mode, a);
        return;
      }
    }
    element_eo_or_plain<N, M, typename LargeShape<N, M>::type>(c, mode, tb, a);
    return;
  } else {
    // small P: all three components per stage (more pencils per warp), even-odd
    if constexpr (N == M && N == 4) {
      // P = 3: collocated, one element per half-warp, TMA boxes (swizzled
      // layout, ColLay::SW): 2.42 -> 1.98 ms per K.p (profiles/variants_r01.txt)
      if ((mode == MODE_FINT || mode == MODE_APPLY || mode == MODE_PA || mode == MODE_SETUP || mode == MODE_MASS) &&
          c->variant != 10 && c->mir >= 0 && !c->ev_mode && col_tma_ok(c, mode, a)) {
        if (c->mir == 0) col_modes<N, 0>(c, mode, a);
        else col_modes<N, 1>(c, mode, a);
        return;
      }
    }
    element_eo_or_plain<N, M, typename DefaultShape<N, M>::type>(c, mode, tb, a);
  }
}

// squared 1D tables of the diagonal kernel (element_diag.cuh): per axis
// w B^2, w B D (2/h), w D^2 (2/h)^2, det J folded into z
template <int N, int M>
TabD<N, M> make_tabd(const sdme_ctx* c) {
  TabD<N, M> t;
  const Geo& g = c->geo;
  for (int a = 0; a < M; ++a)
    for (int l = 0; l < N; ++l) {
      const double b = c->Bl[a * N + l], d = c->Dl[a * N + l], w = c->w[a];
      for (int ax = 0; ax < 3; ++ax) {
        const double s = g.s[ax], jz = ax == 2 ? g.detJ : 1.0;
        double(&T)[3][M][N] = ax == 0 ? t.x : (ax == 1 ? t.y : t.z);
        T[0][a][l] = w * b * b * jz;
        T[1][a][l] = w * b * d * s * jz;
        T[2][a][l] = w * d * d * s * s * jz;
      }
    }
  return t;
}

// collocated tables (element_col.cuh, m = n): B, D^ = D B^-1 per axis (x 2/h)
template <int N, int MIR>
TabC<N, MIR> make_tabc(const sdme_ctx* c) {
  const Geo& g = c->geo;
  double Bv[N][N], Dv[N][N], inv[N][N], a[N][2 * N];
  for (int r = 0; r < N; ++r)
    for (int l = 0; l < N; ++l) {
      Bv[r][l] = c->Bl[r * N + l];
      Dv[r][l] = c->Dl[r * N + l];
    }
  // B^-1 by Gauss-Jordan with partial pivoting (n <= 9, cond(B) <= 34)
  for (int r = 0; r < N; ++r)
    for (int l = 0; l < 2 * N; ++l) a[r][l] = l < N ? Bv[r][l] : (l - N == r ? 1.0 : 0.0);
  for (int col = 0; col < N; ++col) {
    int piv = col;
    for (int r = col + 1; r < N; ++r)
      if (std::fabs(a[r][col]) > std::fabs(a[piv][col])) piv = r;
    for (int l = 0; l < 2 * N; ++l) std::swap(a[col][l], a[piv][l]);
    const double d = a[col][col];
    for (int l = 0; l < 2 * N; ++l) a[col][l] /= d;
    for (int r = 0; r < N; ++r)
      if (r != col) {
        const double f = a[r][col];
        for (int l = 0; l < 2 * N; ++l) a[r][l] -= f * a[col][l];
      }
  }
  for (int r = 0; r < N; ++r)
    for (int l = 0; l < N; ++l) inv[r][l] = a[r][N + l];
  double Dh[3][N][N];
  for (int r = 0; r < N; ++r)
    for (int q = 0; q < N; ++q) {
      double s = 0.0;
      for (int l = 0; l < N; ++l) s += Dv[r][l] * inv[l][q];
      for (int ax = 0; ax < 3; ++ax) Dh[ax][r][q] = s * g.s[ax];
    }
  TabC<N, MIR> t;
  EoBuild<N, N, MIR>::fwd(t.B, Bv, 1);
  EoBuild<N, N, 0>::fwd(t.Dx, Dh[0], -1);
  EoBuild<N, N, 0>::fwd(t.Dy, Dh[1], -1);
  EoBuild<N, N, 0>::fwd(t.Dz, Dh[2], -1);
  EoBuild<N, N, MIR>::bwd(t.bB, Bv, 1);
  EoBuild<N, N, 0>::bwd(t.bDx, Dh[0], -1);
  EoBuild<N, N, 0>::bwd(t.bDy, Dh[1], -1);
  EoBuild<N, N, 0>::bwd(t.bDz, Dh[2], -1);
  if (N <= 5) {
    // P <= 4: the backward tables are the forward ones transposed, entry for
    // entry (by the mirror symmetry EoBuild::bwd gives the same numbers up to
    // the last bit).  The quintet kernel (element_q5) reads the forward tables
    // in its backward pass -- half the table constants -- and so matches
    // element_col<5> bit for bit; element_col itself does so for N <= 5.
    // Higher orders keep the EoBuild::bwd bits.
    eo_transpose(t.bB, t.B);
    eo_transpose(t.bDx, t.Dx);
    eo_transpose(t.bDy, t.Dy);
    eo_transpose(t.bDz, t.Dz);
  }
  for (int q = 0; q < N; ++q) t.wq[q] = c->w[q];
  t.detJ = g.detJ;
  return t;
}

template <int N, int MODE, bool VAL, int MIR, bool TM, bool ISO = false>
void launch_col_k(sdme_ctx* c, const TabC<N, MIR>& tb, OpArgs a) {
  constexpr int WPE = LargeShape<N, N>::WPE;  // one round per stage
  constexpr int T = 32 * WPE;
  // N * N <= 16 pencils per stage: two elements per warp (TMA path)
  constexpr int SUB = (TM && WPE == 1 && N * N <= 16) ? 2 : 1;
  constexpr int smem = SUB * ColPer<N, VAL, TM>::PERP * 8;
  auto kern = element_col<N, WPE, (WPE == 1 ? SDME_COL_MINB : 1), MODE, VAL, MIR, TM, false, SUB, ISO>;
  static PerDevice grid_cache;  // per device: attribute + occupancy set once
  const int max_blocks = resident_grid(grid_cache, kern, T, smem);
  if (MODE == MODE_SETUP || c->ev_mode) {
    // setup: no scatter, one pass over all elements; E-vector mode: boxes + gather
    a.colour = -1;
    if (MODE != MODE_SETUP) a.ev = c->d_ev;
    kern<<<(unsigned)std::min<long long>((colour_count(c->geo, -1) + SUB - 1) / SUB, max_blocks), T, smem, c->st>>>(
        tb, c->geo, a);
    if (MODE == MODE_SETUP || c->ev_no_gather) ++c->launches;
    else ev_gather<N>(c, a);
    return;
  }
  // TMA passes: programmatic dependent launch -- pass k+1 starts its u / p
  // forward work while pass k drains (each CTA waits before its first
  // reduce-add into y); the first pass too when the launch before it is the
  // PDL-triggering zeroing of y (c->pdl_first).  Not inside graph capture
  // (the PCG graph's passes follow kernels that write p).
  bool pdl = TM && c->pdl && !c->capturing;
  bool first = true;
  // z-slab schedule (colour_code): K.p from u and the mass run the 8 colour
  // passes slab by slab over 8 z-slabs, so the faces a slab's passes share stay
  // in L2 -- with PDL filling the extra partial waves this costs no time and
  // cuts K.p DRAM traffic 4.69 -> 1.90 GB at config 2 (SDME_SLABS overrides)
  // (P = 6 / 8 K.p: 2.02 / 1.98 ms at 8 slabs, 1.97 / 1.98 at 4, 1.95 / 1.93 at 2; tools/run_configs.py c3)
  const int nslab = c->nslab_env ? c->nslab : ((TM && (MODE == MODE_APPLY || MODE == MODE_MASS)) ? (N >= 7 ? 2 : 8) : 1);
  for (int sp = 0; sp < 8 * nslab; ++sp) {
    const int col = colour_code(c->geo, sp % 8, sp / 8, nslab);
    if (col == -2) continue;
    const long long cnt = colour_count(c->geo, col);
    if (cnt == 0) continue;
    a.colour = col;
    const unsigned grid = (unsigned)std::min<long long>((cnt + SUB - 1) / SUB, max_blocks);
    if (pdl && (!first || c->pdl_first)) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(T);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = c->st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tb, c->geo, a);
      if (e != cudaSuccess && c->launch_err == cudaSuccess) c->launch_err = e;
    } else {
      kern<<<grid, T, smem, c->st>>>(tb, c->geo, a);
    }
    first = false;
    ++c->launches;
  }
  c->pdl_first = false;
}

// SDME_Q5_ISO=0: never the one-derivative-table (ISO) instances (A/B)
inline bool q5_iso_enabled() {
  static const bool on = [] {
    const char* e = getenv("SDME_Q5_ISO");
    return !(e && e[0] == '0');
  }();
  return on;
}

// P = 4 with tensor maps: five elements per 4-warp CTA (element_q5.cuh);
// SDME_VARIANT=12 keeps the warp-per-element kernel (A/B only)
template <int MODE, bool VAL, int MIR, bool ISO>
void launch_q5_iso(sdme_ctx* c, const TabC<5, MIR>& tb, OpArgs a) {
  using L = Q5Lay<MODE, VAL>;
  constexpr int T = 128, smem = L::PER * 8;
  constexpr int MINB = (227 * 1024) / (smem + 1024) < SDME_Q5_MINB ? (227 * 1024) / (smem + 1024) : SDME_Q5_MINB;
  auto kern = element_q5<MINB, MODE, VAL, MIR, ISO>;
  static PerDevice grid_cache;
  const int max_blocks = resident_grid(grid_cache, kern, T, smem);
  if (MODE == MODE_SETUP) {
    a.colour = -1;
    const long long nq = (colour_count(c->geo, -1) + L::E - 1) / L::E;
    kern<<<(unsigned)std::min<long long>(nq, max_blocks), T, smem, c->st>>>(tb, c->geo, a);
    ++c->launches;
    return;
  }
  bool pdl = c->pdl && !c->capturing;
  bool first = true;
  // z slabs (DRAM traffic): measured on this kernel K.p 1.589 / 1.597 / 1.575 /
  // 1.603 ms and mass 0.732 / 0.688 / 0.658 / 0.714 ms for 1 / 2 / 4 / 8 slabs, f_int flat
  // K.p keeps 8: 1.7% slower than 4 but 1.89 instead of 3.18 GB of DRAM traffic per call
  // f_int: 1.108 / 1.125 / 1.107 / 1.132 ms for 1 / 2 / 4 / 8 slabs; 4 for its DRAM traffic (3.2 GB at 1)
  const int nslab = c->nslab_env ? c->nslab
                                 : (MODE == MODE_APPLY ? 8 : ((MODE == MODE_MASS || MODE == MODE_FINT) ? 4 : 1));
  for (int sp = 0; sp < 8 * nslab; ++sp) {
    const int col = colour_code(c->geo, sp % 8, sp / 8, nslab);
    if (col == -2) continue;
    const long long cnt = colour_count(c->geo, col);
    if (cnt == 0) continue;
    a.colour = col;
    const unsigned grid = (unsigned)std::min<long long>((cnt + L::E - 1) / L::E, max_blocks);
    if (pdl && (!first || c->pdl_first)) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(T);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = c->st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tb, c->geo, a);
      if (e != cudaSuccess && c->launch_err == cudaSuccess) c->launch_err = e;
    } else {
      kern<<<grid, T, smem, c->st>>>(tb, c->geo, a);
    }
    first = false;
    ++c->launches;
  }
  c->pdl_first = false;
}

// Cubic elements (hx = hy = hz: one derivative table for the three axes) keep
// all 25 table constants in uniform registers for the whole kernel; otherwise
// the 49 constants are re-read from the constant bank per component loop
// (OpArgs::zero).  SDME_Q5_ISO=0 forces the general instance (A/B).
template <int MODE, bool VAL, int MIR>
void launch_q5(sdme_ctx* c, const TabC<5, MIR>& tb, OpArgs a) {
  const Geo& g = c->geo;
  if (q5_iso_enabled() && g.s[0] == g.s[1] && g.s[1] == g.s[2]) launch_q5_iso<MODE, VAL, MIR, true>(c, tb, a);
  else launch_q5_iso<MODE, VAL, MIR, false>(c, tb, a);
}

// TMA box loads / bulk reduce-add (tma.cuh) when every vector of the mode has
// a tensor map and the colour passes scatter (not E-vector mode).  An FP64 box
// must start 16-byte aligned (tools/micro/tma_f64.cu), so boxes start at the
// even x at or below the element (odd P: rows shifted by one, box n + 2 wide).
// SDME_VARIANT=11 keeps the cp.async / RED kernel (A/B only).
// P = 5 (box pitch 8 doubles: 8-way bank conflicts on the row reads; measured
// 2.93 vs 2.72 ms) keeps the cp.async kernel; P = 7 (pitch 10) 2.39 vs 2.84 ms.
template <int N, int MODE, bool VAL, int MIR>
void launch_col(sdme_ctx* c, const TabC<N, MIR>& tb, OpArgs a) {
  if constexpr ((N & 1) || BoxW<N>::BW % 4 == 2) {
    const bool maps = MODE == MODE_SETUP ? a.tu != nullptr
                                         : (a.ty && (MODE == MODE_PA || MODE == MODE_MASS || a.tu) &&
                                            (MODE == MODE_FINT || a.tp));
    if (maps && !c->ev_mode && c->variant != 11) {
      if constexpr (N == 5) {
        // The stored-data operator too (round 2): with its point data (K, ln J)
        // prefetched into L2 one quintet ahead and loaded into registers before
        // the forward pass of p (element_q5.cuh, SDME_PA_PREF) it runs at 1.35 ms
        // against 1.50 ms for the warp-per-element kernel without prefetch
        // (1.38 with its own L2 prefetch), and with the mass term, two CTAs
        // per SM, at 1.49 against 1.67 (1.54) ms (tools/op_times.py).
        if (c->variant != 12) {
          launch_q5<MODE, VAL, MIR>(c, tb, a);
          return;
        }
      }
      if constexpr (N <= 5) {
        // cubic elements: one derivative table (ISO instance; with the forward
        // tables also serving the backward pass, 16 / 25 table constants at
        // P = 3 / 4 -- they stay in uniform registers for the whole kernel)
        const Geo& g = c->geo;
        if (q5_iso_enabled() && g.s[0] == g.s[1] && g.s[1] == g.s[2]) {
          launch_col_k<N, MODE, VAL, MIR, true, true>(c, tb, a);
          return;
        }
      }
      launch_col_k<N, MODE, VAL, MIR, true>(c, tb, a);
      return;
    }
  }
  launch_col_k<N, MODE, VAL, MIR, false>(c, tb, a);
}

// collocated path: f_int, K.p (from u or from stored quadrature data)
template <int N, int MIR>
void col_modes(sdme_ctx* c, int mode, OpArgs a) {
  const TabC<N, MIR> tb = make_tabc<N, MIR>(c);
  if (mode == MODE_FINT) launch_col<N, MODE_FINT, false, MIR>(c, tb, a);
  else if (mode == MODE_SETUP) launch_col<N, MODE_SETUP, false, MIR>(c, tb, a);
  else if (mode == MODE_APPLY && a.c_m != 0.0) launch_col<N, MODE_APPLY, true, MIR>(c, tb, a);
  else if (mode == MODE_APPLY) launch_col<N, MODE_APPLY, false, MIR>(c, tb, a);
  else if (mode == MODE_PA && a.c_m != 0.0) launch_col<N, MODE_PA, true, MIR>(c, tb, a);
  else if (mode == MODE_MASS) launch_col<N, MODE_MASS, true, MIR>(c, tb, a);
  else launch_col<N, MODE_PA, false, MIR>(c, tb, a);
}

// P = 4, m = 5 with tensor maps: the diagonal on the quintet schedule
// (element_q5d.cuh); SDME_VARIANT=13 keeps element_diag3 (A/B only)
template <int MIR, bool ISO>
void launch_q5_diag(sdme_ctx* c, const double* u, double* d, double ck, double cm, const void* tu, const void* td_map) {
  using L = Q5DLay;
  constexpr int T = 128, smem = L::PER * 8;
  auto kern = element_q5_diag<3, MIR, ISO>;
  static PerDevice grid_cache;
  const int max_blocks = resident_grid(grid_cache, kern, T, smem);
  const TabC<5, MIR> tb = make_tabc<5, MIR>(c);
  const TabD<5, 5> td = make_tabd<5, 5>(c);
  OpArgs a{u, nullptr, d, ck, cm, 0, c->d_flag};
  a.tu = tu;
  a.ty = td_map;
  for (int sp = 0; sp < 8; ++sp) {
    const int col = colour_code(c->geo, sp, 0, 1);
    if (col == -2) continue;
    const long long cnt = colour_count(c->geo, col);
    if (cnt == 0) continue;
    a.colour = col;
    const unsigned grid = (unsigned)std::min<long long>((cnt + L::E - 1) / L::E, max_blocks);
    kern<<<grid, T, smem, c->st>>>(tb, td, c->geo, a);
    ++c->launches;
  }
}

template <int N, int M>
void diag_impl(sdme_ctx* c, const double* u, double* d, double ck, double cm) {
  if constexpr (N == 5 && M == 5) {
    const void* tu = sdme_tmap_of(c, u);
    const void* tdm = sdme_tmap_of(c, d);
    if (ck != 0.0 && tu && tdm && !c->ev_mode && c->mir >= 0 && c->variant != 13 && c->variant != 11) {
      const Geo& g = c->geo;
      const bool iso = g.s[0] == g.s[1] && g.s[1] == g.s[2];
      if (c->mir == 0) {
        if (iso) launch_q5_diag<0, true>(c, u, d, ck, cm, tu, tdm);
        else launch_q5_diag<0, false>(c, u, d, ck, cm, tu, tdm);
      } else {
        if (iso) launch_q5_diag<1, true>(c, u, d, ck, cm, tu, tdm);
        else launch_q5_diag<1, false>(c, u, d, ck, cm, tu, tdm);
      }
      return;
    }
  }
  constexpr int WPE = LargeShape<N, M>::WPE;  // one round per stage
  constexpr int smem = DiagLay<N, M, WPE>::PER * 8;
  auto kern = element_diag3<N, M, WPE, 1, 1>;
  static PerDevice grid_cache;  // per device: attribute + occupancy set once
  const int max_blocks = resident_grid(grid_cache, kern, WPE * 32, smem);
  const Tab3<N, M> tb = make_tab3<N, M>(c);
  const TabD<N, M> td = make_tabd<N, M>(c);
  OpArgs a{u, nullptr, d, ck, cm, 0, c->d_flag};
  if (c->ev_mode) {
    a.colour = -1;
    a.ev = c->d_ev;
    kern<<<(unsigned)std::min<long long>(colour_count(c->geo, -1), max_blocks), WPE * 32, smem, c->st>>>(
        tb, td, c->geo, a);
    ev_gather<N>(c, a);
    return;
  }
  for (int sp = 0; sp < 8 * c->nslab; ++sp) {
    const int col = colour_code(c->geo, sp % 8, sp / 8, c->nslab);
    if (col == -2) continue;
    const long long cnt = colour_count(c->geo, col);
    if (cnt == 0) continue;
    a.colour = col;
    kern<<<(unsigned)std::min<long long>(cnt, max_blocks), WPE * 32, smem, c->st>>>(tb, td, c->geo, a);
    ++c->launches;
  }
}

template <int N>
void pcg_small_attr() {
  static PerDevice done;
  int& d = done.v[current_device()];
  if (d < 0) {
    cudaFuncSetAttribute(k_pcg_small<N>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    d = 1;
  }
}

template <int N>
cudaLaunchConfig_t pcg_small_config(sdme_ctx* c, cudaLaunchAttribute* at) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kSmallCta);
  cfg.blockDim = dim3(kSmallThreads);
  cfg.stream = c->st;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kSmallCta;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  // + programmatic dependent of the E-vector element kernel before it (SDME_PDL=0: plain)
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = c->pdl ? 2 : 1;
  return cfg;
}

template <int N>
int pcg_small_fits_impl(sdme_ctx* c) {
  pcg_small_attr<N>();
  cudaLaunchAttribute at[2];
  cudaLaunchConfig_t cfg = pcg_small_config<N>(c, at);
  int clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&clusters, k_pcg_small<N>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return clusters > 0 ? 1 : 0;
}

template <int N>
void pcg_small_impl(sdme_ctx* c, double* x, double* r, double* p, double* ap, const double* dinv,
                    cudaGraphConditionalHandle cond, int has_cond) {
  pcg_small_attr<N>();
  cudaLaunchAttribute at[2];
  cudaLaunchConfig_t cfg = pcg_small_config<N>(c, at);
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_pcg_small<N>, x, r, p, ap, dinv, (const double*)c->d_ev,
                                           c->geo, c->d_scal, c->d_status, cond, has_cond);
  if (e != cudaSuccess && c->launch_err == cudaSuccess) c->launch_err = e;
  ++c->launches;
}

// ------------------------------------------------ general meshes (F4)
// element_gen.cuh: gather -> element_col<..., GEN> -> deterministic assembly

template <int N, int MODE, bool VAL, int MIR>
void launch_col_gen(sdme_ctx* c, const TabC<N, MIR>& tb, OpArgs a) {
  constexpr int WPE = LargeShape<N, N>::WPE;
  constexpr int T = 32 * WPE;
  constexpr int smem = ColLay<N, VAL>::PER * 8;
  constexpr int MINB = WPE != 1 ? 1 : (MODE == MODE_APPLY ? SDME_GEN_APPLY_MINB : SDME_GEN_MINB);
  auto kern = element_col<N, WPE, MINB, MODE, VAL, MIR, false, true>;
  static PerDevice grid_cache;  // per device: attribute + occupancy set once
  const int max_blocks = resident_grid(grid_cache, kern, T, smem);
  a.colour = -1;
  kern<<<(unsigned)std::min<long long>(colour_count(c->geo, -1), max_blocks), T, smem, c->st>>>(tb, c->geo, a);
  ++c->launches;
}

template <int N, int MIR>
void gen_modes(sdme_ctx* c, int mode, OpArgs a) {
  const TabC<N, MIR> tb = make_tabc<N, MIR>(c);  // geo.s = 1, det J = 1: reference-coordinate tables
  if (mode == MODE_FINT) launch_col_gen<N, MODE_FINT, false, MIR>(c, tb, a);
  else if (mode == MODE_SETUP) launch_col_gen<N, MODE_SETUP, false, MIR>(c, tb, a);
  else if (mode == MODE_APPLY && a.c_m != 0.0) launch_col_gen<N, MODE_APPLY, true, MIR>(c, tb, a);
  else if (mode == MODE_APPLY) launch_col_gen<N, MODE_APPLY, false, MIR>(c, tb, a);
  else if (mode == MODE_PA && a.c_m != 0.0) launch_col_gen<N, MODE_PA, true, MIR>(c, tb, a);
  else if (mode == MODE_MASS) launch_col_gen<N, MODE_MASS, true, MIR>(c, tb, a);
  else launch_col_gen<N, MODE_PA, false, MIR>(c, tb, a);
}

inline unsigned gen_grid(long long n) { return (unsigned)std::min<long long>((n + 255) / 256, 148LL * 16); }

template <int N>
void gen_element_impl(sdme_ctx* c, int mode, const double* u, const double* p, double* y, double ck, double cm) {
  constexpr int Q = N * N * N;
  const long long ns = (long long)c->geo.nx * 3 * Q;
  const int* skip = c->cur_skip;
  OpArgs a{c->d_evu, c->d_evp, y, ck, cm, -1, c->d_flag, skip};
  a.geo = c->d_geom;
  a.elem_id = c->d_elem_id;
  a.qpd = c->d_qpd;
  a.ev = c->d_ev;
  if (mode == MODE_APPLY) {
    k_gen_gather2<<<gen_grid(ns), 256, 0, c->st>>>(c->d_evu, u, c->d_evp, p, c->d_dof, ns, skip);
    ++c->launches;
  } else if (mode == MODE_FINT || mode == MODE_SETUP) {
    k_gen_gather<<<gen_grid(ns), 256, 0, c->st>>>(c->d_evu, u, c->d_dof, ns, skip);
    ++c->launches;
  } else if (mode == MODE_PA || mode == MODE_MASS) {
    k_gen_gather<<<gen_grid(ns), 256, 0, c->st>>>(c->d_evp, p, c->d_dof, ns, skip);
    ++c->launches;
  }
  if (c->mir == 0) gen_modes<N, 0>(c, mode, a);
  else gen_modes<N, 1>(c, mode, a);
  if (mode != MODE_SETUP) {
    k_gen_assemble<<<gen_grid(c->nvec), 256, 0, c->st>>>(y, c->d_ev, c->d_aptr, c->d_aslot, c->nvec, skip, false,
                                                         c->d_asm_rows);
    ++c->launches;
  }
}

// squared 1D tables without weights (w det J is per point on general meshes)
template <int N>
TabD<N, N> make_tabd_gen(const sdme_ctx* c) {
  TabD<N, N> t;
  for (int a = 0; a < N; ++a)
    for (int l = 0; l < N; ++l) {
      const double b = c->Bl[a * N + l], d = c->Dl[a * N + l];
      for (int ax = 0; ax < 3; ++ax) {
        double(&T)[3][N][N] = ax == 0 ? t.x : (ax == 1 ? t.y : t.z);
        T[0][a][l] = b * b;
        T[1][a][l] = b * d;
        T[2][a][l] = d * d;
      }
    }
  return t;
}

template <int N, int MIR>
void gen_diag_launch(sdme_ctx* c, OpArgs a) {
  constexpr int WPE = LargeShape<N, N>::WPE;
  constexpr int smem = DiagGenLay<N, WPE, MIR>::PER * 8;
  auto kern = element_diag_gen<N, WPE, MIR>;
  static PerDevice grid_cache;  // per device: attribute + occupancy set once
  const int max_blocks = resident_grid(grid_cache, kern, 32 * WPE, smem);
  kern<<<(unsigned)std::min<long long>(colour_count(c->geo, -1), max_blocks), 32 * WPE, smem, c->st>>>(
      make_tabc<N, MIR>(c), make_tabd_gen<N>(c), c->geo, a);
  ++c->launches;
}

template <int N>
void gen_diag_impl(sdme_ctx* c, const double* u, double* d, double ck, double cm) {
  constexpr int Q = N * N * N;
  const long long ns = (long long)c->geo.nx * 3 * Q;
  OpArgs a{c->d_evu, nullptr, d, ck, cm, -1, c->d_flag};
  a.geo = c->d_geom;
  a.elem_id = c->d_elem_id;
  a.ev = c->d_ev;
  if (ck != 0.0) {
    k_gen_gather<<<gen_grid(ns), 256, 0, c->st>>>(c->d_evu, u, c->d_dof, ns, nullptr);
    ++c->launches;
  }
  if (c->mir == 0) gen_diag_launch<N, 0>(c, a);
  else gen_diag_launch<N, 1>(c, a);
  k_gen_assemble<<<gen_grid(c->nvec), 256, 0, c->st>>>(d, c->d_ev, c->d_aptr, c->d_aslot, c->nvec, nullptr,
                                                       true, c->d_asm_rows);
  ++c->launches;
}

template <int N>
const Ops* gen_ops_for() {
  static const Ops o{&gen_element_impl<N>, &gen_diag_impl<N>, nullptr, nullptr};
  return &o;
}

template <int N, int M>
const Ops* ops_for() {
  static const Ops o{&element_impl<N, M>, &diag_impl<N, M>, &pcg_small_impl<N>, &pcg_small_fits_impl<N>};
  return &o;
}

}  // namespace

#define SDME_CAT2(a, b) a##b
#define SDME_CAT(a, b) SDME_CAT2(a, b)
const SdmeOps* SDME_CAT(sdme_ops_p, SDME_ORDER)(int m) {
  if (m == SDME_ORDER + 1) return ops_for<SDME_ORDER + 1, SDME_ORDER + 1>();
  if (m == SDME_ORDER + 2) return ops_for<SDME_ORDER + 1, SDME_ORDER + 2>();
  return nullptr;
}

// general meshes: m = P + 1 (collocated kernels), P >= 2
const SdmeOps* SDME_CAT(sdme_ops_gen_p, SDME_ORDER)(int m) {
#if SDME_ORDER >= 2
  if (m == SDME_ORDER + 1) return gen_ops_for<SDME_ORDER + 1>();
#endif
  (void)m;
  return nullptr;
}
