// Contact face tables and launch arguments (header-only; kernels in
// contact_kernels.cuh) -- shared with the context object (ctx.cuh).
#pragma once

namespace sdme {

constexpr int kMaxN = 9;    // P <= 8
constexpr int kMaxQF = 12;  // face rule points per direction

struct FaceTab {
  double B[kMaxQF][kMaxN];  // lattice-local function values at face rule points
  double W[kMaxQF];
  double X[kMaxQF];         // rule points (reference coordinate)
  int n, qf;
};

enum { CONTACT_FORCE = 0, CONTACT_APPLY = 1, CONTACT_DIAG = 2 };

struct ContactArgs {
  int axis, side;           // face normal axis (0..2) and side (0 = min, 1 = max)
  double origin[3];
  double h[3];
  double point[3], normal[3];
  double eps;
  const double* u;
  double* fc;               // accumulated force (RMW)
  double* gaps;             // [face][qf*qf], reference face/point order
  int colour;               // bit0: parity along d1, bit1: along d2
  int mode;                 // CONTACT_FORCE / CONTACT_APPLY (u -> p) / CONTACT_DIAG
  const int* skip;          // PCG status word: return at once when set
};

}  // namespace sdme
