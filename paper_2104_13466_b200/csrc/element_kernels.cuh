// Shared pieces of the element kernels (sm_100a): geometry, operator
// arguments, Dirichlet masks, colour classes, the C-form neo-Hookean point
// state of the diagonal kernel, and the E-vector gather.
//
// The kernels replace the dense per-element path of the reference
//   femcore.py:87-106  deformation_state / element_internal_force   (f_int)
//   femcore.py:116-146 _b_matrix / element_tangent, consumer a@p     (K.p)
//   femcore.py:149-156 element_mass, mass_full @ a_trial             (mass)
//   solver.py:105-110  diagonal of the assembled effective operator  (diag)
// by O(n^4) sum-factorised contractions plus O(m^3) point work
// (element_v3.cuh, element_eo.cuh, element_diag.cuh).
//
// Data layout: every global vector is a lattice of
// Lx*Ly*Lz points per displacement component, component-major, x fastest,
// rows padded to the even pitch Px (the pad column is held at 0 like a
// Dirichlet point; host-side lattice arrays stay dense, Lx per row).
// Element (i,j,k) owns the (P+1)^3 box starting at (P*i, P*j, P*k).  The 1D
// tables arrive permuted to *lattice-local* order (column l = lattice offset l),
// so an element gather is a strided box with no index table.
//
// Assembly is deterministic: elements are processed in 8 colour passes (parity
// of i, j, k); elements of one colour share no lattice point, so within a pass
// every point receives at most one contribution (RED.ADD never contends) and
// the summation order at every point is fixed by the colour order.  Small
// meshes instead store element boxes (E-vector) and gather them in a fixed
// order (k_ev_gather).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sdme {

struct Geo {
  int nx, ny, nz;     // elements per axis
  int Lx, Ly, Lz;     // lattice points per axis (P*n+1)
  int Px;             // x pitch of the device lattice (Lx rounded up to even: 16-byte rows for TMA)
  long long Ns;       // points per component plane
  double s[3];        // dxi/dX = 2/h per axis
  double detJ;        // h_x h_y h_z / 8
  double mu, lam, rho;
  int dmask[3];       // Dirichlet face bits per component (xmin,xmax,ymin,ymax,zmin,zmax)
  int serp;           // 1: odd colour passes run their elements in reverse order
};

// MODE_SETUP stores K = F^-T and ln J at every quadrature point (OpArgs::qpd);
// MODE_PA is K.p from those stored values (the PCG operator: u is fixed
// during a solve, so the u pass and the point inverse/log are done once).
// MODE_ENERGY writes the element strain energy sum_q w_q det J psi(F) to qpd[e]
// (p carries the 1D rule weights in that mode).
enum Mode { MODE_FINT = 0, MODE_APPLY = 1, MODE_MASS = 2, MODE_PA = 3, MODE_SETUP = 4, MODE_ENERGY = 5 };
constexpr int kQpSlots = 10;  // K (9) + ln J per point, [elem][slot][q]

struct OpArgs {
  const double* u;    // linearisation point (FINT, APPLY, DIAG)
  const double* p;    // direction (APPLY) or field (MASS)
  double* y;          // accumulated output (RMW per colour pass)
  double c_k, c_m;    // y += c_k K p + c_m M p   (APPLY); y += c_m M p (MASS)
  int colour;         // bit0: i parity, bit1: j parity, bit2: k parity
  unsigned long long* inv_flag;  // atomicMin(elem*nq + qp) on det F <= 0
  const int* skip = nullptr;     // if set and non-zero: return at once (stopped PCG graph)
  double* ev = nullptr;          // E-vector mode (colour < 0): element boxes stored, not scattered
  double* qpd = nullptr;         // quadrature data (MODE_SETUP writes, MODE_PA reads)
  // TMA tensor maps (CUtensorMap in global memory) of u, p, y for the
  // box-load / reduce-add element kernels; nullptr: per-lane staging and RED
  const void* tu = nullptr;
  const void* tp = nullptr;
  const void* ty = nullptr;
  // general meshes (element_gen.cuh): per element and point J^-1 (9 slots) and
  // w det J ([elem][10][Q]); u / p are then E-vector boxes [elem][comp][Q]
  const double* geo = nullptr;
  const int* elem_id = nullptr;  // general meshes: reference element id of a storage position (nullptr: same)
  // always 0; a value the compiler cannot fold.  Kernels add zero * (loop
  // counter) to the address of their 1D tables inside a loop so that the
  // table reads stay constant-bank loads (LDCU) in the loop body: hoisted,
  // the ~100 table doubles overflow the uniform register file and ptxas
  // shuffles them through vector registers (R2UR / MOV.SPILL, 18% of the
  // K.p kernel's instructions, ncu) and local memory
  int zero = 0;
};

// Orders from which the kernels re-read their tables (measured, tools/run_configs.py
// c3, tools/op_times.py): the collocated kernels at P >= 4 (P = 6 K.p
// 2.10 -> 2.02 ms, P = 8 2.16 -> 1.98 ms; P = 3: 1.97 -> 2.03 ms, so not
// below); the all-component v3 kernels never (P = 2 K.p 3.66 -> 3.74 ms,
// diagonal at P = 4 4.98 -> 5.30 ms, config 1 unchanged: few multiply-adds
// per table constant there)
#ifndef SDME_COL_RELOAD_MIN_N
#define SDME_COL_RELOAD_MIN_N 5
#endif
#ifndef SDME_V3_RELOAD_MIN_N
#define SDME_V3_RELOAD_MIN_N 99
#endif

// the tables again, through an offset (always 0) that varies with the loop:
// their reads stay LDCU in the loop body (OpArgs::zero)
template <class T>
__device__ __forceinline__ const T& reload_tab(const T& tb, int off) {
  return *reinterpret_cast<const T*>(reinterpret_cast<const char*>(&tb) + off);
}

__device__ __forceinline__ bool constrained(const Geo& g, int comp, int X, int Y, int Z) {
  const int m = g.dmask[comp];
  return ((m & 1) && X == 0) || ((m & 2) && X == g.Lx - 1) || ((m & 4) && Y == 0) ||
         ((m & 8) && Y == g.Ly - 1) || ((m & 16) && Z == 0) || ((m & 32) && Z == g.Lz - 1);
}

// True when the element box starting at (X0, Y0, Z0) with N points per edge
// touches a Dirichlet plane of component comp (warp-uniform fast path).
__device__ __forceinline__ bool touches_dirichlet(const Geo& g, int comp, int X0, int Y0, int Z0, int N) {
  const int m = g.dmask[comp];
  if (!m) return false;
  return ((m & 1) && X0 == 0) || ((m & 2) && X0 + N - 1 == g.Lx - 1) || ((m & 4) && Y0 == 0) ||
         ((m & 8) && Y0 + N - 1 == g.Ly - 1) || ((m & 16) && Z0 == 0) || ((m & 32) && Z0 + N - 1 == g.Lz - 1);
}

// Element of this block slot, for the given colour pass.  Returns false past the end.
// colour >= 0: the elements of one parity class (8-colour passes);
// colour < 0: every element in lexicographic order (E-vector mode).
__device__ __forceinline__ bool colour_element(const Geo& g, int colour, long long idx,
                                               int& ei, int& ej, int& ek) {
  if (colour < 0) {
    if (idx >= (long long)g.nx * g.ny * g.nz) return false;
    ei = (int)(idx % g.nx);
    const long long r = idx / g.nx;
    ej = (int)(r % g.ny);
    ek = (int)(r / g.ny);
    return true;
  }
  // colour code: parity bits 0-2, optional z-slab [izlo, izhi) of the
  // colour's element layers in bits 3-16 / 17-30 (0, 0: all layers)
  const int cx = colour & 1, cy = (colour >> 1) & 1, cz = (colour >> 2) & 1;
  const int nex = (g.nx - cx + 1) >> 1, ney = (g.ny - cy + 1) >> 1, nez = (g.nz - cz + 1) >> 1;
  int izlo = (colour >> 3) & 0x3fff, izhi = (colour >> 17) & 0x3fff;
  if (izhi == 0) izlo = 0, izhi = nez;
  if (izhi > nez) izhi = nez;
  if (nex <= 0 || ney <= 0 || izhi <= izlo) return false;
  const long long cnt = (long long)nex * ney * (izhi - izlo);
  if (idx >= cnt) return false;
  // serpentine pass order: the passes run in Gray-code colour order
  // (colour_of_pass: consecutive passes are face neighbours) and sweep the mesh
  // in alternating directions (odd popcount = odd pass), so a pass starts
  // where the previous one ended and finds their shared faces still in L2
  if (g.serp && (__popc(colour & 7) & 1)) idx = cnt - 1 - idx;
  int ix, iy, iz;
  if (cnt <= 0x7fffffffLL) {
    // 32-bit unsigned division (a 64-bit divide is a ~70-instruction
    // subroutine, and this runs twice per element: current and next)
    const unsigned id = (unsigned)idx, ux = (unsigned)nex, uy = (unsigned)ney;
    const unsigned r = id / ux;
    ix = (int)(id - r * ux);
    const unsigned q = r / uy;
    iy = (int)(r - q * uy);
    iz = izlo + (int)q;
  } else {
    ix = (int)(idx % nex);
    const long long r = idx / nex;
    iy = (int)(r % ney);
    iz = izlo + (int)(r / ney);
  }
  ei = 2 * ix + cx;
  ej = 2 * iy + cy;
  ek = 2 * iz + cz;
  return true;
}

// launch order of the 8 colour passes: Gray code 0 1 3 2 6 7 5 4 (each pass
// flips one parity bit, i.e. shares faces with the previous one)
__host__ __device__ constexpr int colour_of_pass(int pass) { return pass ^ (pass >> 1); }

__host__ __device__ inline long long colour_count(const Geo& g, int colour) {
  if (colour < 0) return (long long)g.nx * g.ny * g.nz;
  const int cx = colour & 1, cy = (colour >> 1) & 1, cz = (colour >> 2) & 1;
  const long long nex = (g.nx - cx + 1) >> 1, ney = (g.ny - cy + 1) >> 1, nez = (g.nz - cz + 1) >> 1;
  long long izlo = (colour >> 3) & 0x3fff, izhi = (colour >> 17) & 0x3fff;
  if (izhi == 0) izlo = 0, izhi = nez;
  if (izhi > nez) izhi = nez;
  if (nex <= 0 || ney <= 0 || izhi <= izlo) return 0;
  return nex * ney * (izhi - izlo);
}

// colour code of pass `pass` over z-slab `slab` of `nslab` (element layers
// split evenly in the colour's own layer index)
inline int colour_code(const Geo& g, int pass, int slab, int nslab) {
  const int c = colour_of_pass(pass);
  if (nslab <= 1) return c;
  const int nez = (g.nz - ((c >> 2) & 1) + 1) >> 1;
  const int lo = (int)((long long)nez * slab / nslab), hi = (int)((long long)nez * (slab + 1) / nslab);
  if (hi <= lo) return -2;  // empty slab
  return c | (lo << 3) | (hi << 17);
}

// ---------------------------------------------------------------------------
// Per-qp constitutive work (neo-Hookean, material.py:65-105).

struct QpState {
  double F[3][3];
  double Ci[3][3];
  double S[3][3];
  double lnJ;
  double detF;
};

__device__ __forceinline__ void qp_state(const double H[3][3], double mu, double lam, QpState& st) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) st.F[i][j] = H[i][j] + (i == j ? 1.0 : 0.0);
  const double(&F)[3][3] = st.F;
  st.detF = F[0][0] * (F[1][1] * F[2][2] - F[1][2] * F[2][1]) -
            F[0][1] * (F[1][0] * F[2][2] - F[1][2] * F[2][0]) +
            F[0][2] * (F[1][0] * F[2][1] - F[1][1] * F[2][0]);
  // C = F^T F (symmetric)
  double C00 = F[0][0] * F[0][0] + F[1][0] * F[1][0] + F[2][0] * F[2][0];
  double C11 = F[0][1] * F[0][1] + F[1][1] * F[1][1] + F[2][1] * F[2][1];
  double C22 = F[0][2] * F[0][2] + F[1][2] * F[1][2] + F[2][2] * F[2][2];
  double C01 = F[0][0] * F[0][1] + F[1][0] * F[1][1] + F[2][0] * F[2][1];
  double C12 = F[0][1] * F[0][2] + F[1][1] * F[1][2] + F[2][1] * F[2][2];
  double C02 = F[0][0] * F[0][2] + F[1][0] * F[1][2] + F[2][0] * F[2][2];
  // adjugate / det
  double A00 = C11 * C22 - C12 * C12;
  double A01 = C02 * C12 - C01 * C22;
  double A02 = C01 * C12 - C02 * C11;
  double A11 = C00 * C22 - C02 * C02;
  double A12 = C01 * C02 - C00 * C12;
  double A22 = C00 * C11 - C01 * C01;
  double detC = C00 * A00 + C01 * A01 + C02 * A02;
  double inv = 1.0 / detC;
  st.Ci[0][0] = A00 * inv; st.Ci[1][1] = A11 * inv; st.Ci[2][2] = A22 * inv;
  st.Ci[0][1] = st.Ci[1][0] = A01 * inv;
  st.Ci[1][2] = st.Ci[2][1] = A12 * inv;
  st.Ci[0][2] = st.Ci[2][0] = A02 * inv;
  st.lnJ = 0.5 * log(detC);
  const double a = lam * st.lnJ - mu;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) st.S[i][j] = a * st.Ci[i][j] + (i == j ? mu : 0.0);
}

// E-vector mode: y += sum of the element boxes covering each lattice point.
// Along each axis a point lies in one element (interior offset) or two (a
// shared plane: offset P in the left element, 0 in the right one); the up to
// 8 contributions are summed in a fixed (z, y, x, ascending element) order,
// so results are bit-reproducible.  Constrained points are left untouched.
__device__ __forceinline__ int ev_cands(int X, int P, int n, int (&e)[2], int (&o)[2]) {
  const int q = X / P, r = X - q * P;
  if (r != 0) { e[0] = q; o[0] = r; return 1; }
  if (q == 0) { e[0] = 0; o[0] = 0; return 1; }
  if (q == n) { e[0] = n - 1; o[0] = P; return 1; }
  e[0] = q - 1; o[0] = P; e[1] = q; o[1] = 0;
  return 2;
}

// gathered value of lattice entry idx (comp-major); false on constrained points
// (E-vector mode only: meshes of <= kEvMaxElements elements, so 32-bit index math)
template <int N>
__device__ __forceinline__ bool ev_point(const double* __restrict__ ev, const Geo& g, long long idx_, double& s) {
  constexpr int P = N - 1, B = N * N * N;
  const int idx = (int)idx_, ns = (int)g.Ns;
  const int comp = idx / ns;
  const int r = idx - comp * ns;
  const int rxy = r / g.Px, X = r - rxy * g.Px;
  if (X >= g.Lx) return false;  // pitch padding
  const int Z = rxy / g.Ly, Y = rxy - Z * g.Ly;
  if (constrained(g, comp, X, Y, Z)) return false;
  int ex[2], ox[2], ey[2], oy[2], ez[2], oz[2];
  const int nx = ev_cands(X, P, g.nx, ex, ox), ny = ev_cands(Y, P, g.ny, ey, oy),
            nz = ev_cands(Z, P, g.nz, ez, oz);
  // all (up to 8) loads issued before the fixed-order sum
  double v[8];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const bool ok = a < nz && b < ny && c < nx;
        const int e = (ez[a & (nz - 1)] * g.ny + ey[b & (ny - 1)]) * g.nx + ex[c & (nx - 1)];
        v[(a * 2 + b) * 2 + c] =
            ok ? ev[(long long)(e * 3 + comp) * B + (oz[a & (nz - 1)] * N + oy[b & (ny - 1)]) * N +
                    ox[c & (nx - 1)]]
               : 0.0;
      }
  s = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += v[t];
  return true;
}

template <int N>
__global__ void __launch_bounds__(256) k_ev_gather(double* __restrict__ y, const double* __restrict__ ev,
                                                   const __grid_constant__ Geo g, const int* skip) {
  if (skip && *(volatile const int*)skip) return;
  const long long total = 3 * g.Ns;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    double s;
    if (ev_point<N>(ev, g, idx, s)) y[idx] += s;
  }
}

}  // namespace sdme
