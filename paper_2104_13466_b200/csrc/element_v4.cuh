// Element kernels v4 ("column-resident points") for m*m <= 32 (P <= 4 at m = P+1).
//
// v3's limiter at config 2 is the shared-memory pipe (profiles/ncu_apply_r01_v3b.txt:
// l1tex 77%, ~1,560 wavefronts per element).  A third of that traffic is the
// point buffer: the z stage writes grad u / grad p to shared memory, the point
// stage reads them back in a different thread mapping, writes the flux, and
// the backward z stage reads the flux again.  v4 keeps every point value in
// the registers of the thread that produced it: lane (b, a) owns the column
// of m points (a, b, c = 0..m-1), for all three components, from the forward
// z stage through the constitutive work to the backward z stage.  The x/y
// stages stay in shared memory (component-serial, as v3 NC=1), the point
// buffer disappears (6.4 KB instead of 19.6 KB of shared memory per element at
// P=4), and each lane has m independent points of ILP in the point work.
// Arithmetic and summation order per output are identical to v3, so results
// are bit-identical to the v3 kernels.
#pragma once
#include "element_v3.cuh"

namespace sdme {

template <int N, int M>
struct V4 {
  static_assert(M * M <= 32, "v4 needs one warp lane per point column");
  using Ly = Lay<N, M, 1>;
  static constexpr int XS = N * Ly::sx;
  static constexpr int XO = 2 * XS;              // x-stage scratch, one component
  static constexpr int YS = N * Ly::sy;
  static constexpr int YO = 3 * YS;              // y-stage scratch, one component
  static constexpr int PER = XO + YO;            // doubles of shared memory per element
  __device__ static int xi(int s, int k, int j, int a) { return s * XS + k * Ly::sx + j * M + a; }
  __device__ static int yi(int s, int k, int ba) { return s * YS + k * Ly::sy + ba; }
};

// x and y stages of one component of a field -> Y scratch.  Rows (k, j) of the
// element box start at base + k*sk + j*sj: global lattice rows (GLOBAL_SRC) or
// the cp.async-staged box in shared memory.
template <int N, int M, bool GRAD, bool GLOBAL_SRC>
__device__ __forceinline__ void v4_xy(const Tab3<N, M>& tb, const double* __restrict__ base, long long sk,
                                      long long sj, double* Xs, double* Ys, int t) {
  using C = V4<N, M>;
  if (t < N * N) {
    const int k = t / N, j = t % N;
    const double* row = base + k * sk + j * sj;
    double v[N];
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = GLOBAL_SRC ? __ldg(row + i) : row[i];
#pragma unroll
    for (int a = 0; a < M; ++a) {
      double b0 = 0.0, b1 = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        b0 = fma(tb.B[a][i], v[i], b0);
        if (GRAD) b1 = fma(tb.Dx[a][i], v[i], b1);
      }
      Xs[C::xi(0, k, j, a)] = b0;
      if (GRAD) Xs[C::xi(1, k, j, a)] = b1;
    }
  }
  __syncwarp();
  if (t < N * M) {
    const int k = t / M, a = t % M;
    double x0[N], x1[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      x0[j] = Xs[C::xi(0, k, j, a)];
      if (GRAD) x1[j] = Xs[C::xi(1, k, j, a)];
    }
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
      Ys[C::yi(0, k, b * M + a)] = bb;
      if (GRAD) {
        Ys[C::yi(1, k, b * M + a)] = db;
        Ys[C::yi(2, k, b * M + a)] = bd;
      }
    }
  }
  __syncwarp();
}

// z stage of one component into the lane's column registers
template <int N, int M, bool GRAD, bool VAL>
__device__ __forceinline__ void v4_z(const Tab3<N, M>& tb, const double* Ys, int t, double (&G)[3][M],
                                     double (&V)[M]) {
  using C = V4<N, M>;
  if (t < M * M) {
    double y0[N], y1[N], y2[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      y0[k] = Ys[C::yi(0, k, t)];
      if (GRAD) {
        y1[k] = Ys[C::yi(1, k, t)];
        y2[k] = Ys[C::yi(2, k, t)];
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
      if (GRAD) {
        G[0][c] = gx;
        G[1][c] = gy;
        G[2][c] = gz;
      }
      if (VAL) V[c] = vv;
    }
  }
  __syncwarp();
}

// backward of one component: column registers -> z' (shared) -> y' -> x' -> RED
template <int N, int M, bool GRAD, bool VAL>
__device__ __forceinline__ void v4_back(const Tab3<N, M>& tb, const Geo& g, double* __restrict__ dst, int comp,
                                        int X0, int Y0, int Z0, double* Xs, double* Ys, int t,
                                        const double (&Fq)[3][M], const double (&Vq)[M]) {
  using C = V4<N, M>;
  if (t < M * M) {
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double hx = 0.0, hy = 0.0, hz = 0.0;
#pragma unroll
      for (int c = 0; c < M; ++c) {
        if (GRAD) {
          hx = fma(tb.bBz[c][k], Fq[0][c], hx);
          hy = fma(tb.bBz[c][k], Fq[1][c], hy);
          hz = fma(tb.bDz[c][k], Fq[2][c], hz);
        }
        if (VAL) hz = fma(tb.bBz[c][k], Vq[c], hz);
      }
      if (GRAD) {
        Ys[C::yi(0, k, t)] = hx;
        Ys[C::yi(1, k, t)] = hy;
      }
      Ys[C::yi(2, k, t)] = hz;
    }
  }
  __syncwarp();
  if (t < N * M) {
    const int k = t / M, a = t % M;
    double hx[M], hy[M], hz[M];
#pragma unroll
    for (int b = 0; b < M; ++b) {
      if (GRAD) {
        hx[b] = Ys[C::yi(0, k, b * M + a)];
        hy[b] = Ys[C::yi(1, k, b * M + a)];
      }
      hz[b] = Ys[C::yi(2, k, b * M + a)];
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
      if (GRAD) Xs[C::xi(0, k, j, a)] = jx;
      Xs[C::xi(1, k, j, a)] = jyz;
    }
  }
  __syncwarp();
  if (t < N * N) {
    const int k = t / N, j = t % N;
    double jx[M], jyz[M];
#pragma unroll
    for (int a = 0; a < M; ++a) {
      if (GRAD) jx[a] = Xs[C::xi(0, k, j, a)];
      jyz[a] = Xs[C::xi(1, k, j, a)];
    }
    const int Z = Z0 + k, Y = Y0 + j;
    const bool chk = touches_dirichlet(g, comp, X0, Y0, Z0, N);
    double* row = dst + comp * g.Ns + ((long long)Z * g.Ly + Y) * g.Lx + X0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < M; ++a) {
        if (GRAD) acc = fma(tb.bDx[a][i], jx[a], acc);
        acc = fma(tb.bBx[a][i], jyz[a], acc);
      }
      if (!chk || !constrained(g, comp, X0 + i, Y, Z)) red_add(row + i, acc);
    }
  }
  __syncwarp();
}


// stage the 3-component (P+1)^3 box of one field into shared memory, [comp][k][j][i]
template <int N>
__device__ __forceinline__ void v4_stage_box(const Geo& g, const double* __restrict__ src, int X0, int Y0, int Z0,
                                             double* box, int t) {
#pragma unroll
  for (int r = 0; r < (3 * N * N * N + 31) / 32; ++r) {
    const int w = t + 32 * r;
    if (w < 3 * N * N * N) {
      const int comp = w / (N * N * N), rem = w % (N * N * N);
      const int k = rem / (N * N), j = (rem / N) % N, i = rem % N;
      cp_async8(box + w, src + comp * g.Ns + ((long long)(Z0 + k) * g.Ly + (Y0 + j)) * g.Lx + X0 + i);
    }
  }
}

// One colour pass, one warp per element, MINB blocks of one warp per SM.
// ASYNC: the next element's u and p boxes are staged into shared memory with
// cp.async while the current element computes (double-buffered).
template <int N, int M, int MINB, int MODE, bool VAL, bool ASYNC, bool GUS = false>
__global__ void __launch_bounds__(32, MINB) element_v4(const __grid_constant__ Tab3<N, M> tb,
                                                         const __grid_constant__ Geo g, OpArgs args) {
  using C = V4<N, M>;
  extern __shared__ double smem[];
  const int t = threadIdx.x;
  double* Xs = smem;
  double* Ys = smem + C::XO;
  constexpr int BOX = 3 * N * N * N;
  double* Ub = smem + C::PER;              // [2][BOX] (ASYNC only)
  double* Pb = Ub + 2 * BOX;               // [2][BOX]
  // GUS (apply mode): grad u parked lane-private in shared memory, [9*M][32]
  double* Gs = smem + C::PER + (ASYNC ? 4 * BOX : 0);
  constexpr bool PARK = GUS && MODE == MODE_APPLY;
  constexpr bool NEED_U = MODE != MODE_MASS, NEED_P = MODE != MODE_FINT;
  if (args.skip && *(volatile const int*)args.skip) return;
  const long long cnt = colour_count(g, args.colour);
  const long long stride = gridDim.x;
  const double mu_k = args.c_k * g.mu, lam_k = args.c_k * g.lam;
  const double cmr = args.c_m * g.rho;
  const int a = t % M, b = (t / M) % M;  // this lane's point column (valid for t < M*M)
  if (ASYNC && (long long)blockIdx.x < cnt) {
    int ei, ej, ek;
    colour_element(g, args.colour, blockIdx.x, ei, ej, ek);
    if (NEED_U) v4_stage_box<N>(g, args.u, (N - 1) * ei, (N - 1) * ej, (N - 1) * ek, Ub, t);
    if (NEED_P) v4_stage_box<N>(g, args.p, (N - 1) * ei, (N - 1) * ej, (N - 1) * ek, Pb, t);
    cp_async_commit();
  }
  int buf = 0;
  for (long long idx = blockIdx.x; idx < cnt; idx += stride, buf ^= 1) {
    int ei, ej, ek;
    colour_element(g, args.colour, idx, ei, ej, ek);
    const int X0 = (N - 1) * ei, Y0 = (N - 1) * ej, Z0 = (N - 1) * ek;
    if (ASYNC) {
      if (idx + stride < cnt) {
        int ni, nj, nk;
        colour_element(g, args.colour, idx + stride, ni, nj, nk);
        if (NEED_U) v4_stage_box<N>(g, args.u, (N - 1) * ni, (N - 1) * nj, (N - 1) * nk, Ub + (buf ^ 1) * BOX, t);
        if (NEED_P) v4_stage_box<N>(g, args.p, (N - 1) * ni, (N - 1) * nj, (N - 1) * nk, Pb + (buf ^ 1) * BOX, t);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncwarp();
    } else if (idx + stride < cnt) {
      int ni, nj, nk;
      colour_element(g, args.colour, idx + stride, ni, nj, nk);
      if (MODE != MODE_MASS) v3_prefetch<N, 32>(g, args.u, (N - 1) * ni, (N - 1) * nj, (N - 1) * nk, t);
      if (MODE != MODE_FINT) v3_prefetch<N, 32>(g, args.p, (N - 1) * ni, (N - 1) * nj, (N - 1) * nk, t);
    }
    // column registers: Gu[comp][d][c], Gp[comp][d][c] (flux in place), Vp[comp][c]
    double Gu[3][3][M], Gp[3][3][M], Vp[3][M];
    if (MODE != MODE_MASS) {
#pragma unroll
      for (int comp = 0; comp < 3; ++comp) {
        if (ASYNC)
          v4_xy<N, M, true, false>(tb, Ub + buf * BOX + comp * N * N * N, N * N, N, Xs, Ys, t);
        else
          v4_xy<N, M, true, true>(tb, args.u + comp * g.Ns + ((long long)Z0 * g.Ly + Y0) * g.Lx + X0,
                                  (long long)g.Ly * g.Lx, g.Lx, Xs, Ys, t);
        v4_z<N, M, true, false>(tb, Ys, t, Gu[comp], Vp[comp]);
        if (PARK && t < M * M) {
#pragma unroll
          for (int d = 0; d < 3; ++d)
#pragma unroll
            for (int c = 0; c < M; ++c) Gs[((comp * 3 + d) * M + c) * 32 + t] = Gu[comp][d][c];
        }
      }
    }
    if (MODE != MODE_FINT) {
      constexpr bool GRADP = (MODE == MODE_APPLY);
      constexpr bool VALP = VAL || MODE == MODE_MASS;
#pragma unroll
      for (int comp = 0; comp < 3; ++comp) {
        if (ASYNC)
          v4_xy<N, M, GRADP, false>(tb, Pb + buf * BOX + comp * N * N * N, N * N, N, Xs, Ys, t);
        else
          v4_xy<N, M, GRADP, true>(tb, args.p + comp * g.Ns + ((long long)Z0 * g.Ly + Y0) * g.Lx + X0,
                                   (long long)g.Ly * g.Lx, g.Lx, Xs, Ys, t);
        v4_z<N, M, GRADP, VALP>(tb, Ys, t, Gp[comp], Vp[comp]);
      }
    }
    // point work on the lane's column
    if (t < M * M) {
#pragma unroll
      for (int c = 0; c < M; ++c) {
        if (MODE == MODE_MASS) {
#pragma unroll
          for (int i = 0; i < 3; ++i) Vp[i][c] *= cmr;
          continue;
        }
        double H[9];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) H[i * 3 + d] = PARK ? Gs[((i * 3 + d) * M + c) * 32 + t] : Gu[i][d][c];
        QpK s;
        qp_k(H, s);
        if (!(s.det > 0.0)) {
          const long long e = ((long long)ek * g.ny + ej) * g.nx + ei;
          atomicMin(args.inv_flag, (unsigned long long)e * (M * M * M) + (unsigned long long)((a * M + b) * M + c));
        }
        if (MODE == MODE_FINT) {
          const double cK = g.lam * s.lnJ - g.mu;
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int d = 0; d < 3; ++d) Gu[i][d][c] = fma(g.mu, s.F[i][d], cK * s.K[i][d]);
        } else {
          double Hp[3][3];
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int d = 0; d < 3; ++d) Hp[i][d] = Gp[i][d][c];
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
#pragma unroll
          for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              const double m2 = fma(M1[i][0], s.K[0][d], fma(M1[i][1], s.K[1][d], M1[i][2] * s.K[2][d]));
              Gp[i][d][c] = fma(cc, m2, fma(lt, s.K[i][d], mu_k * Hp[i][d]));
            }
          if (VAL) {
#pragma unroll
            for (int i = 0; i < 3; ++i) Vp[i][c] *= cmr;
          }
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      if (MODE == MODE_MASS)
        v4_back<N, M, false, true>(tb, g, args.y, comp, X0, Y0, Z0, Xs, Ys, t, Gp[comp], Vp[comp]);
      else if (MODE == MODE_FINT)
        v4_back<N, M, true, false>(tb, g, args.y, comp, X0, Y0, Z0, Xs, Ys, t, Gu[comp], Vp[comp]);
      else
        v4_back<N, M, true, VAL>(tb, g, args.y, comp, X0, Y0, Z0, Xs, Ys, t, Gp[comp], Vp[comp]);
    }
  }
}

}  // namespace sdme
