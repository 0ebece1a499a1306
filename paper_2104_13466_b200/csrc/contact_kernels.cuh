// Penalty contact against a rigid plane on a box face (K8).
//
// Replaces PenaltyContact._gaps / evaluate_forces (contact.py:87-128) for a
// tagged side of a structured box: face quadrature with qf x qf Gauss points
// (default P+1, contact.py:81-83), current position x = X + N u, gap
// g = (x - point).n, active where g < 0 (strict), pressure t_N = -eps g, nodal
// force sum_q warea t_N N_f n.  Only the lattice plane of the face carries
// non-zero face traces, so the work is a 2D contraction on that plane.
// Faces are processed in 4 colour passes (in-plane parity) so the
// read-modify-write scatter is race-free and bit-reproducible.
//
// Implicit contact (contact.py:120-140, dynamics.py:268-284): with the active
// set of the last force evaluation (stored gaps), the contact stiffness
// K_c = eps sum_{q active} warea N_f N_g (n n^T) is applied matrix-free
// (CONTACT_APPLY: y += K_c p) and its diagonal added to the Jacobi
// preconditioner (CONTACT_DIAG: d += eps sum_q warea act N_f^2 n_c^2).
#pragma once
#include <cuda_runtime.h>
#include "contact_types.cuh"
#include "element_kernels.cuh"

namespace sdme {

__global__ void __launch_bounds__(128) k_contact(const __grid_constant__ FaceTab ft,
                                                 const __grid_constant__ Geo g, ContactArgs ca) {
  const int axis = ca.axis;
  const int d1 = axis == 0 ? 1 : 0;
  const int d2 = axis == 2 ? 1 : 2;
  const int ne[3] = {g.nx, g.ny, g.nz};
  const int n1 = ne[d1], n2 = ne[d2];
  const int c1 = ca.colour & 1, c2 = (ca.colour >> 1) & 1;
  const int m1 = (n1 - c1 + 1) >> 1, m2 = (n2 - c2 + 1) >> 1;
  const long long fid = blockIdx.x;
  if (m1 <= 0 || m2 <= 0 || fid >= (long long)m1 * m2) return;
  if (ca.skip && *(volatile const int*)ca.skip) return;
  const int f1 = 2 * (int)(fid % m1) + c1;
  const int f2 = 2 * (int)(fid / m1) + c2;
  const int n = ft.n, qf = ft.qf, P = n - 1;
  const int L[3] = {g.Lx, g.Ly, g.Lz};
  const int plane = ca.side ? L[axis] - 1 : 0;

  __shared__ double su[3][kMaxN * kMaxN];
  __shared__ double stn[kMaxQF * kMaxQF];

  // gather the face plane coefficients (n x n per component) of u (force) or p (apply)
  for (int t = threadIdx.x; t < (ca.mode == CONTACT_DIAG ? 0 : 3 * n * n); t += blockDim.x) {
    const int comp = t / (n * n), r = t % (n * n);
    const int l1 = r / n, l2 = r % n;
    int c[3];
    c[axis] = plane;
    c[d1] = P * f1 + l1;
    c[d2] = P * f2 + l2;
    su[comp][r] = ca.u[comp * g.Ns + ((long long)c[2] * g.Ly + c[1]) * g.Px + c[0]];
  }
  __syncthreads();
  // points: gap and pressure (force), or eps warea (n . N p) on the active set (apply),
  // or eps warea on the active set (diag)
  for (int t = threadIdx.x; t < qf * qf; t += blockDim.x) {
    const int a = t / qf, b = t % qf;
    const double warea = ft.W[a] * ft.W[b] * 0.25 * ca.h[d1] * ca.h[d2];
    if (ca.mode != CONTACT_FORCE) {
      const bool act = ca.gaps[((long long)f2 * n1 + f1) * qf * qf + t] < 0.0;
      double pn = 1.0;
      if (ca.mode == CONTACT_APPLY) {
        pn = 0.0;
#pragma unroll
        for (int comp = 0; comp < 3; ++comp) {
          double v = 0.0;
          for (int l1 = 0; l1 < n; ++l1) {
            double sv = 0.0;
            for (int l2 = 0; l2 < n; ++l2) sv = fma(ft.B[b][l2], su[comp][l1 * n + l2], sv);
            v = fma(ft.B[a][l1], sv, v);
          }
          pn = fma(v, ca.normal[comp], pn);
        }
      }
      stn[t] = act ? ca.eps * pn * warea : 0.0;
      continue;
    }
    double x[3];
    x[axis] = ca.origin[axis] + (ca.side ? ne[axis] * ca.h[axis] : 0.0);
    x[d1] = ca.origin[d1] + (f1 + 0.5 * (ft.X[a] + 1.0)) * ca.h[d1];
    x[d2] = ca.origin[d2] + (f2 + 0.5 * (ft.X[b] + 1.0)) * ca.h[d2];
    double gap = 0.0;
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      double v = 0.0;
      for (int l1 = 0; l1 < n; ++l1) {
        double s = 0.0;
        for (int l2 = 0; l2 < n; ++l2) s = fma(ft.B[b][l2], su[comp][l1 * n + l2], s);
        v = fma(ft.B[a][l1], s, v);
      }
      gap = fma(x[comp] + v - ca.point[comp], ca.normal[comp], gap);
    }
    stn[t] = gap < 0.0 ? -ca.eps * gap * warea : 0.0;
    ca.gaps[((long long)f2 * n1 + f1) * qf * qf + t] = gap;
  }
  __syncthreads();
  // nodal force on the plane
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
    const int l1 = t / n, l2 = t % n;
    // diag: squared traces (N_f^2), otherwise the traces themselves
    const bool sq = ca.mode == CONTACT_DIAG;
    double s = 0.0;
    for (int a = 0; a < qf; ++a) {
      double sb = 0.0;
      for (int b = 0; b < qf; ++b) sb = fma(sq ? ft.B[b][l2] * ft.B[b][l2] : ft.B[b][l2], stn[a * qf + b], sb);
      s = fma(sq ? ft.B[a][l1] * ft.B[a][l1] : ft.B[a][l1], sb, s);
    }
    int c[3];
    c[axis] = plane;
    c[d1] = P * f1 + l1;
    c[d2] = P * f2 + l2;
    const long long off = ((long long)c[2] * g.Ly + c[1]) * g.Px + c[0];
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      if (ca.normal[comp] != 0.0 && !constrained(g, comp, c[0], c[1], c[2]))
        ca.fc[comp * g.Ns + off] += s * (sq ? ca.normal[comp] * ca.normal[comp] : ca.normal[comp]);
    }
  }
}

}  // namespace sdme
