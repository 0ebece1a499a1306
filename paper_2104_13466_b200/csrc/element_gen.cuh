// General hexahedral meshes: element gather / assembly through
// index tables and the Jacobi diagonal with per-point geometry.
//
// A general-mesh context keeps vectors in the reference's free-DOF order.  An
// operator application is
//   k_gen_gather   x (free) -> element boxes [elem][comp][z][y][x], signed
//                  (gather, femcore.py:302-306)
//   element_col<..., GEN>  the collocated kernel on those boxes, per-point J^-1
//                  and w det J (build_tables, femcore.py:73-81), results as
//                  element boxes
//   k_gen_assemble y[f] += sum of the signed element entries of f, in element
//                  order: the reference's np.add.at order (femcore.py:318-321),
//                  deterministic, no atomics
#pragma once
#include "element_col.cuh"
#include "element_diag.cuh"

namespace sdme {

// ev[s] = sign * x[free] (0 on constrained entries); dof[s] = 2*free + neg or -1
static __global__ void __launch_bounds__(256) k_gen_gather(double* __restrict__ ev, const double* __restrict__ x,
                                                    const int* __restrict__ dof, long long n, const int* skip) {
  if (skip && *(volatile const int*)skip) return;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int d = __ldg(dof + i);
    double v = 0.0;
    if (d >= 0) {
      v = __ldg(x + (d >> 1));
      if (d & 1) v = -v;
    }
    ev[i] = v;
  }
}

// two fields through one read of the index table (K.p from u: u and p)
static __global__ void __launch_bounds__(256) k_gen_gather2(double* __restrict__ eva, const double* __restrict__ xa,
                                                     double* __restrict__ evb, const double* __restrict__ xb,
                                                     const int* __restrict__ dof, long long n, const int* skip) {
  if (skip && *(volatile const int*)skip) return;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int d = __ldg(dof + i);
    double va = 0.0, vb = 0.0;
    if (d >= 0) {
      va = __ldg(xa + (d >> 1));
      vb = __ldg(xb + (d >> 1));
      if (d & 1) va = -va, vb = -vb;
    }
    eva[i] = va;
    evb[i] = vb;
  }
}

// y[f] += sum_k sign_k ev[slot_k] over the CSR entries of f (increasing element);
// unsigned for a diagonal (sign_k^2 = 1).  CSR row r belongs to DOF rows[r]
// (rows: the locality order of the rows, nullptr = identity)
static __global__ void __launch_bounds__(256) k_gen_assemble(double* __restrict__ y, const double* __restrict__ ev,
                                                      const long long* __restrict__ ptr,
                                                      const int* __restrict__ slot, long long n, const int* skip,
                                                      bool diagonal = false, const int* __restrict__ rows = nullptr) {
  if (skip && *(volatile const int*)skip) return;
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (long long)gridDim.x * blockDim.x) {
    const long long f = rows ? __ldg(rows + r) : r;
    double s = 0.0;
    for (long long k = __ldg(ptr + r), e = __ldg(ptr + r + 1); k < e; ++k) {
      const int sl = __ldg(slot + k);
      const double v = __ldg(ev + (sl >> 1));
      s += ((sl & 1) && !diagonal) ? -v : v;
    }
    y[f] += s;
  }
}

// Jacobi diagonal on a general mesh, one element per CTA of WPE warps:
// reference-coordinate grad u by the collocated forward pass, material
// gradient through J^-1, the diagonal-block coefficients of element_diag3
// turned back to the reference axes (T = J^-1 M J^-T, times w det J), and
// the 6 squared-table chains per component (tables without weights; the
// weights are in w det J).  Output: element boxes (assembled by
// k_gen_assemble).  Once per PCG solve: a plain, unsplit schedule.
template <int N, int WPE, int MIR>
struct DiagGenLay {
  using L = ColLay<N, false>;
  static constexpr int Q = N * N * N;
  static constexpr int A = L::PER, ZS = A + 19 * Q, YS = ZS + Q, PER = YS + Q;
};

template <int N, int WPE, int MIR>
__global__ void __launch_bounds__(32 * WPE, 1) element_diag_gen(const __grid_constant__ TabC<N, MIR> tb,
                                                                const __grid_constant__ TabD<N, N> td,
                                                                const __grid_constant__ Geo g, OpArgs args) {
  using L = ColLay<N, false>;
  using DL = DiagGenLay<N, WPE, MIR>;
  constexpr int T = 32 * WPE, Q = N * N * N;
  extern __shared__ __align__(128) double smem[];
  double* S = smem;
  double* A = S + DL::A;
  double* Zs = S + DL::ZS;
  double* Ys = S + DL::YS;
  const int t = threadIdx.x;
  int buf = 0;
  const long long cnt = colour_count(g, -1);
  const bool stiff = args.c_k != 0.0;
  const double cmr = args.c_m * g.rho;
  int* tab = reinterpret_cast<int*>(S + L::TAB);
  for (int q = t; q < Q; q += T) tab[q] = q;
  group_sync<WPE>(0);
  for (long long eid = blockIdx.x; eid < cnt; eid += gridDim.x) {
    if (stiff) {
      col_stage<N, T>(g, args.u + eid * 3 * Q, 0, 0, 0, 0, S + L::R + buf * Q, t, tab);
      col_forward<N, WPE, MIR, false, false>(tb, args.zero, g, args.u + eid * 3 * Q, 0, 0, 0, S, t, &buf,
                                             NextRows{nullptr, 0, 0, 0}, true);
    }
    for (int q = t; q < Q; q += T) {
      const double wdet = __ldg(args.geo + eid * (10 * Q) + 9 * Q + q);
      double coef[3][6];
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int tt = 0; tt < 6; ++tt) coef[i][tt] = 0.0;
      if (stiff) {
        double J[3][3], H[3][3];
        gen_jinv<N>(args.geo, eid, q, J);
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int d = 0; d < 3; ++d) H[i][d] = S[L::qi(d, i, q)];
        gen_to_phys(&H[0][0], J);
        QpState st;
        qp_state(H, g.mu, g.lam, st);
        if (!(st.detF > 0.0)) {
          const int a = q % N, b = (q / N) % N, c = q / (N * N);
          const long long ref = args.elem_id ? __ldg(args.elem_id + eid) : eid;
          atomicMin(args.inv_flag, (unsigned long long)ref * Q + (unsigned long long)((a * N + b) * N + c));
        }
        const double cc = g.mu - g.lam * st.lnJ;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          double FC[3];
#pragma unroll
          for (int d = 0; d < 3; ++d)
            FC[d] = st.F[i][0] * st.Ci[0][d] + st.F[i][1] * st.Ci[1][d] + st.F[i][2] * st.Ci[2][d];
          const double fcf = FC[0] * st.F[i][0] + FC[1] * st.F[i][1] + FC[2] * st.F[i][2];
          double Mm[3][3];  // material block M_c1c2 = A^i + S
#pragma unroll
          for (int c1 = 0; c1 < 3; ++c1)
#pragma unroll
            for (int c2 = 0; c2 < 3; ++c2)
              Mm[c1][c2] = g.lam * FC[c1] * FC[c2] + cc * (fcf * st.Ci[c1][c2] + FC[c2] * FC[c1]) + st.S[c1][c2];
          double JM[3][3];  // J^-1 M
#pragma unroll
          for (int d = 0; d < 3; ++d)
#pragma unroll
            for (int c2 = 0; c2 < 3; ++c2)
              JM[d][c2] = J[d][0] * Mm[0][c2] + J[d][1] * Mm[1][c2] + J[d][2] * Mm[2][c2];
#pragma unroll
          for (int tt = 0; tt < 6; ++tt) {
            const int d = pair_d(tt), e = pair_e(tt);
            const double Tde = JM[d][0] * J[e][0] + JM[d][1] * J[e][1] + JM[d][2] * J[e][2];
            coef[i][tt] = args.c_k * (d == e ? 1.0 : 2.0) * wdet * Tde;
          }
        }
      }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int tt = 0; tt < 6; ++tt) A[(i * 6 + tt) * Q + q] = coef[i][tt];
      A[18 * Q + q] = cmr * wdet;
    }
    group_sync<WPE>(0);
#pragma unroll 1
    for (int comp = 0; comp < 3; ++comp) {
      constexpr int NR = (N * N + T - 1) / T;
      double acc[NR][N];
#pragma unroll
      for (int r = 0; r < NR; ++r)
#pragma unroll
        for (int i = 0; i < N; ++i) acc[r][i] = 0.0;
#pragma unroll 1
      for (int tt = 0; tt < 6; ++tt) {
        if (!stiff && tt != 2) continue;  // mass only: the (z, z) chain carries it
        const int d = pair_d(tt), e = pair_e(tt);
        const int tx = (d == 0) + (e == 0), ty = (d == 1) + (e == 1), tz = (d == 2) + (e == 2);
        const double* cf = A + (comp * 6 + tt) * Q;
        const double* cm = A + 18 * Q;
        for (int w = t; w < N * N; w += T) {  // z': column (b, a) over c
#pragma unroll
          for (int k = 0; k < N; ++k) {
            double h = 0.0;
#pragma unroll
            for (int c = 0; c < N; ++c) {
              h = fma(td.z[tz][c][k], cf[c * N * N + w], h);
              if (tt == 2) h = fma(td.z[0][c][k], cm[c * N * N + w], h);
            }
            Zs[k * N * N + w] = h;
          }
        }
        group_sync<WPE>(0);
        for (int w = t; w < N * N; w += T) {  // y': item (k, a) over b
          const int k = w / N, a = w % N;
#pragma unroll
          for (int j = 0; j < N; ++j) {
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < N; ++b) s = fma(td.y[ty][b][j], Zs[(k * N + b) * N + a], s);
            Ys[(k * N + j) * N + a] = s;
          }
        }
        group_sync<WPE>(0);
#pragma unroll
        for (int r = 0; r < NR; ++r) {  // x': item (k, j) over a
          const int w = t + r * T;
          if (w >= N * N) continue;
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double s = acc[r][i];
#pragma unroll
            for (int a = 0; a < N; ++a) s = fma(td.x[tx][a][i], Ys[w * N + a], s);
            acc[r][i] = s;
          }
        }
        group_sync<WPE>(0);
      }
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int w = t + r * T;
        if (w >= N * N) continue;
        double* er = args.ev + (eid * 3 + comp) * Q + w * N;
#pragma unroll
        for (int i = 0; i < N; ++i) er[i] = acc[r][i];
      }
    }
    group_sync<WPE>(0);
  }
}

}  // namespace sdme
