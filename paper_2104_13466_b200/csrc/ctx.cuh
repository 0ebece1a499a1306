// Internal: the context object shared by the C-ABI translation unit and the
// per-order operator translation units (ops.cu, compiled once per P).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "contact_types.cuh"
#include "element_kernels.cuh"

struct sdme_ctx;

// meshes with at most this many element points (elements x (P+1)^3) use
// E-vector mode (sdme_ctx::ev_mode): 4096 elements at P = 4; measured with the
// TMA colour passes, tools/ev_crossover.py: P = 4 16^3 EV 79 vs 103 us, 24^3
// 237 vs 188 us; P = 6 64x8x8 (4096 elements) EV 197 vs 187 us
constexpr long long kEvMaxPoints = 4096LL * 125;
constexpr long long kEvMaxElements = kEvMaxPoints / 8;  // bound for the 32-bit index math (P = 1)

// Operator entry points of one (P, m) instantiation.
struct SdmeOps {
  void (*element)(sdme_ctx*, int mode, const double* u, const double* p, double* y, double ck, double cm);
  void (*diag)(sdme_ctx*, const double* u, double* d, double ck, double cm);
  // small-mesh PCG iteration tail after an E-vector element launch (pcg_small.cuh)
  void (*pcg_small)(sdme_ctx*, double* x, double* r, double* p, double* ap, const double* dinv,
                    cudaGraphConditionalHandle cond, int has_cond);
  // 1 if the 16-CTA cluster of pcg_small can be placed on the current device
  // (cudaOccupancyMaxActiveClusters > 0; 0 e.g. under MIG / MPS partitions)
  int (*pcg_small_fits)(sdme_ctx*);
};

struct sdme_ctx {
  int P = 0, m = 0, n = 0;
  sdme::Geo geo{};
  double h[3]{}, origin[3]{};
  std::vector<double> Bl, Dl, w;  // lattice-local order, m x n
  cudaStream_t st = nullptr;
  // side stream + fork / join events: the contact force of an explicit step
  // runs beside the f_int colour passes (sdme_explicit_steps; created on first use)
  cudaStream_t st_side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  long long nvec = 0;             // 3 * Ns (device vector length, pitched rows)
  long long nlat = 0;             // 3 * Lx * Ly * Lz (dense host lattice arrays)
  std::vector<double*> vecs;
  std::vector<void*> vec_tmaps;  // device CUtensorMap per vector (element box TMA), parallel to vecs
  int* d_perm = nullptr;
  int* d_iperm = nullptr;          // free index -> pitched lattice index (gather form of lattice -> free)
  int64_t n_free = 0;
  unsigned char* d_free = nullptr;  // 1 on free lattice dofs
  double* d_fbuf = nullptr;         // staging for free-order vectors
  double* d_partial = nullptr;
  double* d_scal = nullptr;
  double* h_scal = nullptr;         // pinned
  unsigned long long* d_flag = nullptr;   // [0] element inversion, [1] non-positive diagonal
  unsigned long long* d_dflag = nullptr;  // d_flag + 1
  unsigned long long* h_flag = nullptr;
  double* d_gaps = nullptr;
  long long gaps_cap = 0;
  double* h_gaps = nullptr;
  // PCG scratch vectors (lazily allocated ids)
  int v_r = -1, v_p = -1, v_ap = -1, v_dinv = -1, v_tmp = -1;
  const SdmeOps* ops = nullptr;
  int err_code = 0;
  int64_t err_elem = -1;
  int err_qp = -1;
  std::string err_msg;
  int64_t launches = 0;
  int variant = 0;  // schedule variant (SDME_VARIANT env), tuning only
  bool pcg_start = true;  // start of a solve as two fused launches (SDME_PCG_START=0: nine separate ones)
  int chain_mode = -1;  // PCG iteration sequence (SDME_PCG_CHAIN env bit mask; -1: by size, sdme_abi.cu)
  int nslab = 1;    // colour passes per z-slab (SDME_SLABS env): 8 * nslab launches per operator
  bool nslab_env = false;  // SDME_SLABS given: it overrides the per-mode default of the TMA passes
  int mir = -1;     // mirror structure of the 1D tables: 0 nodal, 1 modal/SDME, -1 none (no even-odd)
  int* d_status = nullptr;  // PCG status word (device) and its pinned mirror
  int* h_status = nullptr;
  const int* cur_skip = nullptr;  // element kernels exit early when *cur_skip != 0 (PCG graph)
  // E-vector mode (small meshes): one launch over all elements writing their
  // boxes to d_ev, then a deterministic gather -- instead of 8 colour passes
  bool ev_mode = false;
  bool ev_no_gather = false;
  int pcg_warm = 0;
  int small_fits = -1;
  // programmatic dependent launch of the TMA colour passes (SDME_PDL=0 disables);
  // pdl_first: the next operator's first pass may overlap the zeroing of y
  // (k_zero_pdl); capturing: inside a graph capture (PDL off)
  bool pdl = true;
  bool pdl_first = false;
  bool capturing = false;  // pcg_small cluster placement on this device (-1: not queried yet)
  cudaError_t launch_err = cudaSuccess;  // a failed cudaLaunchKernelEx, reported by check_launch  // operator kinds whose launch setup ran (sdme_pcg)
  // instantiated PCG graph, reused while the solve's operands are the same
  cudaGraph_t pcg_graph = nullptr;
  cudaGraphExec_t pcg_exec = nullptr;
  struct PcgKey {
    const double* u = nullptr;
    const double* x = nullptr;
    double ck = 0.0, cm = 0.0;
    bool pa = false;
    bool contact = false;
    double eps = 0.0;
    unsigned long long cgen = 0;  // contact generation (face tables, plane, gaps buffer) captured
    bool operator==(const PcgKey& o) const {
      return u == o.u && x == o.x && ck == o.ck && cm == o.cm && pa == o.pa && contact == o.contact &&
             eps == o.eps && cgen == o.cgen;
    }
  } pcg_key;
  long long pcg_per_iter = 0;
  bool pcg_direct = false;  // SDME_PCG_DIRECT: no graph (profiling aid)
  // implicit contact: face tables / parameters of the last sdme_contact call
  // (its gaps in d_gaps define the active set of the contact stiffness)
  sdme::FaceTab c_ft{};
  sdme::ContactArgs c_ca{};
  bool c_ready = false;
  // bumped whenever c_ft / c_ca (other than the per-call u / fc pointers) or
  // d_gaps change, so a cached PCG graph never replays a stale contact node
  unsigned long long c_gen = 0;
  bool pcg_contact = false;  // sdme_pcg adds K_c (and its diagonal)  // element launch leaves A p in d_ev (small PCG path gathers)
  double* d_ev = nullptr;
  // stored quadrature data of the PCG linearisation point (MODE_SETUP / MODE_PA)
  double* d_qpd = nullptr;
  double* d_energy = nullptr;  // per-element strain energy (sdme_strain_energy)
  bool pa = true;  // SDME_PA=0 disables (the PCG then applies K(u) from scratch)
  // general mesh (sdme_create_mesh): vectors in the reference free order,
  // elements gathered / assembled through index tables (element_gen.cuh)
  // pipelined batch K.p with host buffers (sdme_apply_batch): copy streams,
  // double-buffered free-order staging, events
  struct Batch {
    cudaStream_t h2d = nullptr, h2d2 = nullptr, d2h = nullptr;  // u / p copies on separate streams
    double* su[2] = {nullptr, nullptr};
    double* sp[2] = {nullptr, nullptr};
    double* sy[2] = {nullptr, nullptr};
    cudaEvent_t ev_h2d[2] = {}, ev_h2d2[2] = {}, ev_in_free[2] = {}, ev_comp[2] = {}, ev_out_free[2] = {};
    int u = -1, p = -1, y = -1;  // lattice vectors
  };
  Batch* batch = nullptr;
  bool gen = false;
  int* d_dof = nullptr;           // [elem][comp][Q] 2*free + neg, or -1
  long long* d_aptr = nullptr;    // assembly CSR over free DOFs
  int* d_aslot = nullptr;
  double* d_geom = nullptr;       // [elem][10][Q] J^-1, w det J
  int* d_elem_id = nullptr;       // storage position -> reference element id (nullptr: identity)
  int* d_asm_rows = nullptr;      // assembly CSR row -> free DOF (nullptr: identity)
  double* d_evu = nullptr;        // gathered element boxes of u and p
  double* d_evp = nullptr;
};

// TMA tensor map (device address) of a context vector, nullptr if none
const void* sdme_tmap_of(const sdme_ctx* c, const double* v);

// per-order operator tables (ops.cu, one object file per P)
const SdmeOps* sdme_ops_p1(int m);
const SdmeOps* sdme_ops_p2(int m);
const SdmeOps* sdme_ops_p3(int m);
const SdmeOps* sdme_ops_p4(int m);
const SdmeOps* sdme_ops_p5(int m);
const SdmeOps* sdme_ops_p6(int m);
const SdmeOps* sdme_ops_p7(int m);
const SdmeOps* sdme_ops_p8(int m);
// general-mesh operator tables (ops.cu; m = P + 1, P >= 2)
const SdmeOps* sdme_ops_gen_p1(int m);
const SdmeOps* sdme_ops_gen_p2(int m);
const SdmeOps* sdme_ops_gen_p3(int m);
const SdmeOps* sdme_ops_gen_p4(int m);
const SdmeOps* sdme_ops_gen_p5(int m);
const SdmeOps* sdme_ops_gen_p6(int m);
const SdmeOps* sdme_ops_gen_p7(int m);
const SdmeOps* sdme_ops_gen_p8(int m);
