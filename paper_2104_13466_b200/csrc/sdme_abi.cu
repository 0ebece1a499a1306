// C-ABI implementation: context, device vectors, operator dispatch over (P, m),
// the Jacobi-PCG driver (solver.py:129-170), explicit step and contact.
// Build: see paper_2104_13466_b200/build.py (nvcc -gencode arch=compute_100a,code=sm_100a).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sdme.h"
#include "contact_kernels.cuh"
#include "element_kernels.cuh"
#include "vector_kernels.cuh"
#include "pcg_small.cuh"

#include "ctx.cuh"

using namespace sdme;

namespace {

constexpr unsigned long long kNoFlag = ~0ull;
using Ops = SdmeOps;

int set_err(sdme_ctx* c, int code, const std::string& msg, int64_t elem = -1, int qp = -1) {
  if (c) {
    c->err_code = code;
    c->err_msg = msg;
    c->err_elem = elem;
    c->err_qp = qp;
  }
  return code;
}

#define CK(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return set_err(ctx, SDME_CUDA_ERROR, std::string(#call ": ") + cudaGetErrorString(e_)); \
  } while (0)

int check_launch(sdme_ctx* ctx) {
  cudaError_t e = cudaGetLastError();
  if (ctx->launch_err != cudaSuccess) {
    if (e == cudaSuccess) e = ctx->launch_err;
    ctx->launch_err = cudaSuccess;
  }
  if (e != cudaSuccess) return set_err(ctx, SDME_CUDA_ERROR, std::string("launch: ") + cudaGetErrorString(e));
  return SDME_OK;
}

inline int grid_for(long long n, int threads = 256) {
  long long g = (n + threads - 1) / threads;
  return (int)std::max<long long>(1, std::min<long long>(g, 148LL * 16));
}

// Mirror structure of the lattice-order tables (eo.cuh); -1 if none applies.
int detect_mirror(const sdme_ctx* c) {
  const int n = c->n, m = c->m, P = c->P;
  for (int mir = 0; mir < 2; ++mir) {
    auto sig = [&](int l) { return mir == 0 ? n - 1 - l : (l == 0 ? n - 1 : (l == n - 1 ? 0 : l)); };
    auto sg = [&](int l) { return mir == 0 ? 1 : ((l == 0 || l == n - 1) ? 1 : ((l % 2) ? 1 : -1)); };
    double scale = 0.0;
    for (double v : c->Bl) scale = std::max(scale, std::fabs(v));
    for (double v : c->Dl) scale = std::max(scale, std::fabs(v));
    bool ok = true;
    for (int a = 0; a < m && ok; ++a) {
      if (std::fabs(c->w[a] - c->w[m - 1 - a]) > 1e-14 * std::fabs(c->w[a])) ok = false;
      for (int l = 0; l < n && ok; ++l) {
        const double b1 = c->Bl[(m - 1 - a) * n + l], b2 = sg(l) * c->Bl[a * n + sig(l)];
        const double d1 = c->Dl[(m - 1 - a) * n + l], d2 = -sg(l) * c->Dl[a * n + sig(l)];
        if (std::fabs(b1 - b2) > 1e-13 * scale || std::fabs(d1 - d2) > 1e-13 * scale) ok = false;
      }
    }
    (void)P;
    if (ok) return mir;
  }
  return -1;
}

const Ops* select_ops(int P, int m) {
  switch (P) {
    case 1: return sdme_ops_p1(m);
    case 2: return sdme_ops_p2(m);
    case 3: return sdme_ops_p3(m);
    case 4: return sdme_ops_p4(m);
    case 5: return sdme_ops_p5(m);
    case 6: return sdme_ops_p6(m);
    case 7: return sdme_ops_p7(m);
    case 8: return sdme_ops_p8(m);
    default: return nullptr;
  }
}

double* vec(sdme_ctx* c, int id) {
  if (id < 0 || id >= (int)c->vecs.size()) return nullptr;
  return c->vecs[id];
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)f;
  }();
  return fn;
}

// Tensor map of one lattice vector for the element box TMA (tma.cuh): 4D
// (x, y, z, component) FP64, pitched rows (Px), box (BW, n, n, 1) with BW the
// even width that covers n points from the even x at or below the element's
// start (n + 1 for odd n, n + 2 for even n; 16-byte box rows); elements outside
// (Lx, Ly, Lz) are zero-filled on load and dropped on reduce.  nullptr if
// unavailable.
void* make_tmap(sdme_ctx* ctx, double* p) {
  if (ctx->gen || getenv("SDME_NO_TMA")) return nullptr;
  auto enc = tmap_encoder();
  if (!enc) return nullptr;
  const Geo& g = ctx->geo;
  const int n = ctx->n, rp = (n + 2) & ~1;  // BoxW<n>: even width covering n points from an even start
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)g.Lx, (cuuint64_t)g.Ly, (cuuint64_t)g.Lz, 3};
  cuuint64_t strides[3] = {(cuuint64_t)g.Px * 8, (cuuint64_t)g.Px * g.Ly * 8, (cuuint64_t)g.Ns * 8};
  cuuint32_t box[4] = {(cuuint32_t)rp, (cuuint32_t)n, (cuuint32_t)n, 1}, es[4] = {1, 1, 1, 1};
  if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return nullptr;
  void* d = nullptr;
  if (cudaMalloc(&d, sizeof(CUtensorMap)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, &m, sizeof(CUtensorMap), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  return d;
}

int alloc_vec(sdme_ctx* ctx, int* id) {
  double* p = nullptr;
  CK(cudaMalloc(&p, ctx->nvec * sizeof(double)));
  CK(cudaMemsetAsync(p, 0, ctx->nvec * sizeof(double), ctx->st));
  void* tm = make_tmap(ctx, p);
  for (size_t i = 0; i < ctx->vecs.size(); ++i)
    if (!ctx->vecs[i]) {
      ctx->vecs[i] = p;
      ctx->vec_tmaps[i] = tm;
      *id = (int)i;
      return SDME_OK;
    }
  ctx->vecs.push_back(p);
  ctx->vec_tmaps.push_back(tm);
  *id = (int)ctx->vecs.size() - 1;
  return SDME_OK;
}

int ensure(sdme_ctx* ctx, int& id) {
  if (id >= 0) return SDME_OK;
  return alloc_vec(ctx, &id);
}

// deterministic dot into d_scal[slot]
int dot_into(sdme_ctx* ctx, const double* a, const double* b, int slot) {
  DotArgs<1> da{{a}, {b}};
  k_dots<1><<<kRedBlocks, kRedThreads, 0, ctx->st>>>(da, ctx->nvec, ctx->d_partial);
  k_finish<1><<<1, kRedThreads, 0, ctx->st>>>(ctx->d_partial, ctx->d_scal + slot);
  ctx->launches += 2;
  return check_launch(ctx);
}

int read_scalars(sdme_ctx* ctx) {
  CK(cudaMemcpyAsync(ctx->h_scal, ctx->d_scal, S_COUNT * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return SDME_OK;
}

int reset_flag(sdme_ctx* ctx) {
  CK(cudaMemsetAsync(ctx->d_flag, 0xFF, sizeof(kNoFlag), ctx->st));  // = kNoFlag; no pageable H2D (implicit stream sync)
  return SDME_OK;
}

int flag_error(sdme_ctx* ctx, unsigned long long f) {
  if (f != kNoFlag) {
    const long long nq = (long long)ctx->m * ctx->m * ctx->m;
    const int64_t e = (int64_t)(f / nq);
    const int q = (int)(f % nq);
    char buf[128];
    snprintf(buf, sizeof buf, "element %lld inverted at quadrature point %d", (long long)e, q);
    return set_err(ctx, SDME_INVERSION, buf, e, q);
  }
  return SDME_OK;
}

int check_flag(sdme_ctx* ctx) {
  CK(cudaMemcpyAsync(ctx->h_flag, ctx->d_flag, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return flag_error(ctx, ctx->h_flag[0]);
}

// y = A p  with A = c_k K(u) + c_m M (y zeroed first)
// y = 0 before an operator's colour passes: a PDL-triggering kernel, so the
// first pass overlaps it (box contexts with tensor maps, outside captures)
int zero_output(sdme_ctx* ctx, double* y) {
  if (ctx->pdl && !ctx->capturing && !ctx->ev_mode && !ctx->gen && sdme_tmap_of(ctx, y)) {
    k_zero_pdl<<<148 * 4, 256, 0, ctx->st>>>(y, ctx->nvec);
    ++ctx->launches;
    ctx->pdl_first = true;
    return SDME_OK;
  }
  CK(cudaMemsetAsync(y, 0, ctx->nvec * sizeof(double), ctx->st));
  return SDME_OK;
}

int apply_raw(sdme_ctx* ctx, const double* u, const double* p, double* y, double ck, double cm) {
  if (int rc = zero_output(ctx, y)) return rc;
  if (ck != 0.0)
    ctx->ops->element(ctx, MODE_APPLY, u, p, y, ck, cm);
  else
    ctx->ops->element(ctx, MODE_MASS, nullptr, p, y, 0.0, cm);
  return check_launch(ctx);
}

}  // namespace

// the 4 in-plane colour passes of one contact evaluation / apply / diagonal
void launch_contact(sdme_ctx* ctx, ContactArgs ca) {
  const int ne[3] = {ctx->geo.nx, ctx->geo.ny, ctx->geo.nz};
  const int d1 = ca.axis == 0 ? 1 : 0, d2 = ca.axis == 2 ? 1 : 2;
  for (int col = 0; col < 4; ++col) {
    const int m1 = (ne[d1] - (col & 1) + 1) >> 1, m2 = (ne[d2] - ((col >> 1) & 1) + 1) >> 1;
    if (m1 <= 0 || m2 <= 0) continue;
    ca.colour = col;
    k_contact<<<m1 * m2, 128, 0, ctx->st>>>(ctx->c_ft, ctx->geo, ca);
    ++ctx->launches;
  }
}

// y += K_c p (CONTACT_APPLY) or y += diag(K_c) (CONTACT_DIAG), active set of
// the last sdme_contact evaluation
void contact_op(sdme_ctx* ctx, int mode, const double* p, double* y, const int* skip) {
  ContactArgs ca = ctx->c_ca;
  ca.mode = mode;
  ca.u = p;
  ca.fc = y;
  ca.skip = skip;
  launch_contact(ctx, ca);
}

// quadrature-data buffer for MODE_SETUP / MODE_PA (allocated on first use;
// false -- and the PCG applies K(u) from scratch -- if it does not fit)
bool ensure_qpd(sdme_ctx* ctx) {
  if (ctx->d_qpd) return true;
  const long long ne = (long long)ctx->geo.nx * ctx->geo.ny * ctx->geo.nz;
  const size_t bytes = (size_t)ne * kQpSlots * ctx->m * ctx->m * ctx->m * sizeof(double);
  if (cudaMalloc(&ctx->d_qpd, bytes) != cudaSuccess) {
    cudaGetLastError();
    ctx->d_qpd = nullptr;
    ctx->pa = false;
    return false;
  }
  return true;
}

// SDME_PCG_CHAIN bit mask (A/B): 1 fused vector kernels (k_pcg_update2 / k_pcg_p2),
// 2 the vector kernels as programmatic dependents, 4 the first colour pass
// overlaps the zeroing of A p.  The colour passes always carry PDL edges (in
// the captured graph too: config 5 SDME_H 0.090 -> 0.073 s per step, one
// iteration at 32^3 385 -> 339 us).  Measured (one iteration at 64^3 / 32^3 /
// 16^3 in us, config 5 SDME_H in s per step): 0: 2511 / 339 / 96.0, 0.0730;
// 1: 2522 / 337 / 93.6, 0.0715; 3: 2562 / 342 / 93.4, 0.0778 (dependents
// spinning in griddepcontrol.wait take issue slots from the HBM-bound kernel
// they wait for); 5: 2515 / 333 / 93.7, 0.0720 (default); 7: 2559 / 339 / 93.5, 0.0775.
// Bit 8 (with bit 1): k_pcg_p2 also zeroes A p for the next iteration (no zeroing launch;
// the first pass then follows k_pcg_p2 plainly): 64^3 / 32^3 / 16^3 2475 / 332 / 89.0 us and
// config-5 size 152.4 us per iteration against 2455 / 336 / 95.9 and 159.4 for mode 5 --
// so 9 up to 2^24 vector entries and 5 above (chain_mode_of).  Read per context.
inline int chain_mode_of(const sdme_ctx* c) {
  return c->chain_mode >= 0 ? c->chain_mode : (c->nvec <= (1LL << 24) ? 9 : 5);
}

// launch as a programmatic dependent of the previous kernel on the stream
template <class... KArgs, class... Args>
void launch_chain(sdme_ctx* ctx, void (*kern)(KArgs...), int grid, int block, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = ctx->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.numAttrs = (chain_mode_of(ctx) & 2) ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  if (e != cudaSuccess && ctx->launch_err == cudaSuccess) ctx->launch_err = e;
}

// One PCG iteration on ctx->st: E-vector element launch + one cluster kernel
// (small meshes) or the 7-kernel sequence.  Every kernel returns at once when
// the status word is set; the last one clears the graph's loop condition.
void enqueue_pcg_iteration(sdme_ctx* ctx, const double* pu, double* px, double* r, double* p, double* ap,
                           double* dinv, double c_k, double c_m, bool pa, bool withc,
                           cudaGraphConditionalHandle cond, int has_cond) {
  const int kmode = pa ? MODE_PA : MODE_APPLY;
  // (the cluster tail gathers A p itself, so K_c p needs the general sequence)
  if (ctx->small_fits < 0) ctx->small_fits = ctx->ops->pcg_small_fits ? ctx->ops->pcg_small_fits(ctx) : 0;
  const bool small = ctx->ev_mode && ctx->nvec <= kSmallPcgMax && ctx->ops->pcg_small && ctx->small_fits && !withc;
  ctx->cur_skip = ctx->d_status;
  if (small) {
    // E-vector element launch, then one cluster kernel for the rest
    ctx->ev_no_gather = true;
    if (c_k != 0.0)
      ctx->ops->element(ctx, kmode, pu, p, ap, c_k, c_m);
    else
      ctx->ops->element(ctx, MODE_MASS, nullptr, p, ap, 0.0, c_m);
    ctx->ev_no_gather = false;
    ctx->ops->pcg_small(ctx, px, r, p, ap, dinv, cond, has_cond);
  } else {
    if (ctx->pdl) {
      // fused sequence, every kernel a programmatic dependent of its predecessor
      // (vector_kernels.cuh); the first colour pass of a TMA operator overlaps
      // the zeroing of A p like the passes overlap one another
      // bit 8 (with the fused kernels): k_pcg_p2 zeroes A p for the next
      // iteration, sdme_pcg once before the first
      const bool p2_zeroes = (chain_mode_of(ctx) & 9) == 9;
      const bool tm_first = (chain_mode_of(ctx) & 4) && !p2_zeroes && !ctx->ev_mode && !ctx->gen && sdme_tmap_of(ctx, ap);
      if (!p2_zeroes)
        launch_chain(ctx, k_zero_chain, grid_for(ctx->nvec), 256, ap, ctx->nvec, (const int*)ctx->d_status);
      const bool cap = ctx->capturing;
      ctx->capturing = false;  // PDL edges between the passes, inside a capture too
      ctx->pdl_first = tm_first;
      if (c_k != 0.0)
        ctx->ops->element(ctx, kmode, pu, p, ap, c_k, c_m);
      else
        ctx->ops->element(ctx, MODE_MASS, nullptr, p, ap, 0.0, c_m);
      ctx->pdl_first = false;
      ctx->capturing = cap;
      if (withc) contact_op(ctx, CONTACT_APPLY, p, ap, ctx->d_status);
      if (!(chain_mode_of(ctx) & 1)) {
        launch_chain(ctx, k_pcg_pap_chain, kRedBlocks, kRedThreads, (const double*)p, (const double*)ap, ctx->nvec,
                     ctx->d_partial, (const int*)ctx->d_status);
        k_pcg_alpha<<<1, kRedThreads, 0, ctx->st>>>(ctx->d_partial, ctx->d_scal, ctx->d_status);
        k_pcg_update<<<kRedBlocks, kRedThreads, 0, ctx->st>>>(px, r, p, ap, dinv, ctx->d_scal, ctx->nvec,
                                                              ctx->d_partial, ctx->d_status);
        k_pcg_check<<<1, kRedThreads, 0, ctx->st>>>(ctx->d_partial, ctx->d_scal, ctx->d_status);
        k_pcg_p<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(p, r, dinv, ctx->d_scal, ctx->nvec, ctx->d_status, cond,
                                                           has_cond);
        ctx->launches += 6;
        ctx->cur_skip = nullptr;
        return;
      }
      double* part2 = ctx->d_partial + 2 * kRedBlocks;
      launch_chain(ctx, k_pcg_pap_chain, kRedBlocks, kRedThreads, (const double*)p, (const double*)ap, ctx->nvec,
                   ctx->d_partial, (const int*)ctx->d_status);
      launch_chain(ctx, k_pcg_update2, kRedBlocks, kRedThreads, px, r, (const double*)p, (const double*)ap,
                   (const double*)dinv, ctx->d_scal, ctx->nvec, (const double*)ctx->d_partial, part2, ctx->d_status);
      launch_chain(ctx, k_pcg_p2, grid_for(ctx->nvec), kRedThreads, p, (const double*)r, (const double*)dinv,
                   ctx->d_scal, ctx->nvec, (const double*)part2, ctx->d_status, cond, has_cond,
                   p2_zeroes ? ap : (double*)nullptr);
      ctx->launches += p2_zeroes ? 3 : 4;
      ctx->cur_skip = nullptr;
      return;
    }
    k_zero<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(ap, ctx->nvec, ctx->d_status);
    if (c_k != 0.0)
      ctx->ops->element(ctx, kmode, pu, p, ap, c_k, c_m);
    else
      ctx->ops->element(ctx, MODE_MASS, nullptr, p, ap, 0.0, c_m);
    if (withc) contact_op(ctx, CONTACT_APPLY, p, ap, ctx->d_status);
    k_pcg_pap<<<kRedBlocks, kRedThreads, 0, ctx->st>>>(p, ap, ctx->nvec, ctx->d_partial, ctx->d_status);
    k_pcg_alpha<<<1, kRedThreads, 0, ctx->st>>>(ctx->d_partial, ctx->d_scal, ctx->d_status);
    k_pcg_update<<<kRedBlocks, kRedThreads, 0, ctx->st>>>(px, r, p, ap, dinv, ctx->d_scal, ctx->nvec,
                                                          ctx->d_partial, ctx->d_status);
    k_pcg_check<<<1, kRedThreads, 0, ctx->st>>>(ctx->d_partial, ctx->d_scal, ctx->d_status);
    k_pcg_p<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(p, r, dinv, ctx->d_scal, ctx->nvec, ctx->d_status,
                                                       cond, has_cond);
    ctx->launches += 6;
  }
  ctx->cur_skip = nullptr;
}

// The whole PCG solve as one CUDA graph: a conditional while-node whose body
// is one iteration; the iteration's last kernel clears the condition once the
// status word is set, so the host waits once per solve.  Small meshes
// (E-vector mode) run the iteration as one element launch + one cluster
// kernel (pcg_small.cuh); others as the 7-kernel sequence.
int build_pcg_graph(sdme_ctx* ctx, const double* pu, double* px, double* r, double* p, double* ap, double* dinv,
                    double c_k, double c_m, bool pa, bool withc) {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  CK(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle cond;
  CK(cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = cond;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t loop;
  CK(cudaGraphAddNode(&loop, graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  const long long l0 = ctx->launches;
  CK(cudaStreamBeginCaptureToGraph(ctx->st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  // plain launches inside the graph for the 7-kernel sequence; the fused
  // sequence adds its own PDL edges, captured as such
  ctx->capturing = true;
  enqueue_pcg_iteration(ctx, pu, px, r, p, ap, dinv, c_k, c_m, pa, withc, cond, 1);
  ctx->capturing = false;
  const cudaError_t ce = cudaStreamEndCapture(ctx->st, &body);
  const long long per_iter = ctx->launches - l0;
  ctx->launches = l0;
  if (ce != cudaSuccess) {
    cudaGraphDestroy(graph);
    return set_err(ctx, SDME_CUDA_ERROR, std::string("graph capture: ") + cudaGetErrorString(ce));
  }
  if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
    cudaGraphDestroy(graph);
    return set_err(ctx, SDME_CUDA_ERROR, "graph instantiate failed");
  }
  ctx->pcg_graph = graph;
  ctx->pcg_exec = exec;
  ctx->pcg_per_iter = per_iter;
  return SDME_OK;
}

// =========================================================================
const void* sdme_tmap_of(const sdme_ctx* c, const double* v) {
  if (!v) return nullptr;
  for (size_t i = 0; i < c->vecs.size(); ++i)
    if (c->vecs[i] == v) return c->vec_tmaps[i];
  return nullptr;
}

extern "C" {

int sdme_create(const sdme_desc* d, sdme_ctx** out) {
  if (!d || !out) return SDME_BAD_ARGUMENT;
  *out = nullptr;
  const Ops* ops = select_ops(d->P, d->m);
  if (!ops || d->nx < 1 || d->ny < 1 || d->nz < 1 || !(d->hx > 0) || !(d->hy > 0) || !(d->hz > 0) ||
      !d->B || !d->D || !d->w)
    return SDME_BAD_ARGUMENT;
  sdme_ctx* ctx = new sdme_ctx();
  ctx->ops = ops;
  if (const char* v = getenv("SDME_VARIANT")) ctx->variant = atoi(v);
  if (const char* v = getenv("SDME_PCG_CHAIN")) ctx->chain_mode = atoi(v);
  if (const char* v = getenv("SDME_PCG_START")) ctx->pcg_start = atoi(v) != 0;
  if (const char* v = getenv("SDME_SLABS")) {
    ctx->nslab = std::max(1, std::min(atoi(v), 64));
    ctx->nslab_env = true;
  }
  if (const char* v = getenv("SDME_PCG_DIRECT")) ctx->pcg_direct = atoi(v) != 0;
  if (const char* v = getenv("SDME_PA")) ctx->pa = atoi(v) != 0;
  if (const char* v = getenv("SDME_PDL")) ctx->pdl = atoi(v) != 0;
  ctx->P = d->P;
  ctx->m = d->m;
  ctx->n = d->P + 1;
  const int n = ctx->n, m = ctx->m, P = d->P;
  // reference function order [left, right, internal 2..P] -> lattice offset l
  auto func_of = [&](int l) { return l == 0 ? 0 : (l == P ? 1 : l + 1); };
  ctx->Bl.resize(m * n);
  ctx->Dl.resize(m * n);
  ctx->w.assign(d->w, d->w + m);
  for (int a = 0; a < m; ++a)
    for (int l = 0; l < n; ++l) {
      ctx->Bl[a * n + l] = d->B[a * n + func_of(l)];
      ctx->Dl[a * n + l] = d->D[a * n + func_of(l)];
    }
  ctx->mir = detect_mirror(ctx);
  Geo& g = ctx->geo;
  g.nx = d->nx; g.ny = d->ny; g.nz = d->nz;
  g.Lx = P * d->nx + 1; g.Ly = P * d->ny + 1; g.Lz = P * d->nz + 1;
  g.Px = (g.Lx + 1) & ~1;  // even pitch: 16-byte aligned rows (TMA tensor maps)
  g.Ns = (long long)g.Px * g.Ly * g.Lz;
  g.s[0] = 2.0 / d->hx; g.s[1] = 2.0 / d->hy; g.s[2] = 2.0 / d->hz;
  g.detJ = d->hx * d->hy * d->hz / 8.0;
  g.mu = d->mu; g.lam = d->lambda_lame; g.rho = d->rho0;
  for (int c = 0; c < 3; ++c) g.dmask[c] = d->dirichlet_mask[c];
  g.serp = 1;
  if (const char* v = getenv("SDME_SERPENTINE")) g.serp = atoi(v) != 0;
  ctx->h[0] = d->hx; ctx->h[1] = d->hy; ctx->h[2] = d->hz;
  for (int c = 0; c < 3; ++c) ctx->origin[c] = d->origin[c];
  ctx->nvec = 3 * g.Ns;
  ctx->nlat = 3LL * g.Lx * g.Ly * g.Lz;
  ctx->n_free = d->n_free;

  auto fail = [&](int code) {
    sdme_destroy(ctx);
    return code;
  };
  if (cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking) != cudaSuccess) return fail(SDME_CUDA_ERROR);
  if (cudaMalloc(&ctx->d_partial, kRedBlocks * 4 * sizeof(double)) != cudaSuccess) return fail(SDME_CUDA_ERROR);
  if (cudaMalloc(&ctx->d_scal, 16 * sizeof(double)) != cudaSuccess) return fail(SDME_CUDA_ERROR);
  if (cudaMallocHost(&ctx->h_scal, 16 * sizeof(double)) != cudaSuccess) return fail(SDME_CUDA_ERROR);
  if (cudaMalloc(&ctx->d_flag, 2 * sizeof(unsigned long long)) != cudaSuccess) return fail(SDME_CUDA_ERROR);
  ctx->d_dflag = ctx->d_flag + 1;
  // E-vector mode for meshes too small to fill the GPU with 8 colour passes
  // (each pass would hold < 1 element per SM slot); SDME_EV=0/1 forces it.
  {
    const long long ne = (long long)g.nx * g.ny * g.nz;
    ctx->ev_mode = ne * n * n * n <= kEvMaxPoints;
    if (const char* v = getenv("SDME_EV")) ctx->ev_mode = atoi(v) != 0;
    if (ctx->ev_mode &&
        cudaMalloc(&ctx->d_ev, (size_t)ne * 3 * n * n * n * sizeof(double)) != cudaSuccess)
      return fail(SDME_CUDA_ERROR);
  }
  if (cudaMallocHost(&ctx->h_flag, 2 * sizeof(unsigned long long)) != cudaSuccess) return fail(SDME_CUDA_ERROR);
  if (cudaMalloc(&ctx->d_status, sizeof(int)) != cudaSuccess) return fail(SDME_CUDA_ERROR);
  if (cudaMallocHost(&ctx->h_status, sizeof(int)) != cudaSuccess) return fail(SDME_CUDA_ERROR);
  // free mask from the Dirichlet planes
  {
    std::vector<unsigned char> fm(ctx->nvec, 1);
    if (g.Px > g.Lx)  // pitch padding is never free
      for (long long r = 0; r < 3LL * g.Ly * g.Lz; ++r)
        for (int X = g.Lx; X < g.Px; ++X) fm[r * g.Px + X] = 0;
    for (int c = 0; c < 3; ++c) {
      const int mk = g.dmask[c];
      if (!mk) continue;
      for (int Z = 0; Z < g.Lz; ++Z)
        for (int Y = 0; Y < g.Ly; ++Y)
          for (int X = 0; X < g.Lx; ++X) {
            const bool cons = ((mk & 1) && X == 0) || ((mk & 2) && X == g.Lx - 1) || ((mk & 4) && Y == 0) ||
                              ((mk & 8) && Y == g.Ly - 1) || ((mk & 16) && Z == 0) || ((mk & 32) && Z == g.Lz - 1);
            if (cons) fm[c * g.Ns + ((long long)Z * g.Ly + Y) * g.Px + X] = 0;
          }
    }
    if (cudaMalloc(&ctx->d_free, ctx->nvec) != cudaSuccess) return fail(SDME_CUDA_ERROR);
    if (cudaMemcpy(ctx->d_free, fm.data(), ctx->nvec, cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(SDME_CUDA_ERROR);
  }
  if (d->perm) {
    if (d->n_free <= 0) return fail(SDME_BAD_ARGUMENT);
    // dense host permutation (Lx per row) -> pitched device rows, -1 on the padding
    std::vector<int> pp(ctx->nvec, -1);
    for (long long r = 0; r < 3LL * g.Ly * g.Lz; ++r)
      for (int X = 0; X < g.Lx; ++X) pp[r * g.Px + X] = d->perm[r * g.Lx + X];
    if (cudaMalloc(&ctx->d_perm, ctx->nvec * sizeof(int)) != cudaSuccess) return fail(SDME_CUDA_ERROR);
    if (cudaMemcpy(ctx->d_perm, pp.data(), ctx->nvec * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(SDME_CUDA_ERROR);
    if (cudaMalloc(&ctx->d_fbuf, d->n_free * sizeof(double)) != cudaSuccess) return fail(SDME_CUDA_ERROR);
    if (cudaMalloc(&ctx->d_iperm, d->n_free * sizeof(int)) != cudaSuccess) return fail(SDME_CUDA_ERROR);
    k_invert_perm<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(ctx->d_iperm, ctx->d_perm, ctx->nvec);
    if (cudaStreamSynchronize(ctx->st) != cudaSuccess) return fail(SDME_CUDA_ERROR);
  }
  *out = ctx;
  return SDME_OK;
}

void batch_free(sdme_ctx* ctx);  // sdme_apply_batch state (below)

// general hexahedral mesh context (element_gen.cuh)
int sdme_create_mesh(const sdme_mesh_desc* d, sdme_ctx** out) {
  if (!d || !out) return SDME_BAD_ARGUMENT;
  *out = nullptr;
  if (d->P < 2 || d->P > 8 || d->m != d->P + 1 || d->n_elems < 1 || d->n_free < 1 || !d->B || !d->D || !d->w ||
      !d->dof || !d->asm_ptr || !d->asm_slot || !d->geom)
    return SDME_BAD_ARGUMENT;
  const Ops* ops = nullptr;
  switch (d->P) {
    case 2: ops = sdme_ops_gen_p2(d->m); break;
    case 3: ops = sdme_ops_gen_p3(d->m); break;
    case 4: ops = sdme_ops_gen_p4(d->m); break;
    case 5: ops = sdme_ops_gen_p5(d->m); break;
    case 6: ops = sdme_ops_gen_p6(d->m); break;
    case 7: ops = sdme_ops_gen_p7(d->m); break;
    case 8: ops = sdme_ops_gen_p8(d->m); break;
    default: break;
  }
  if (!ops) return SDME_BAD_ARGUMENT;
  sdme_ctx* ctx = new sdme_ctx();
  ctx->ops = ops;
  ctx->gen = true;
  if (const char* v = getenv("SDME_PCG_DIRECT")) ctx->pcg_direct = atoi(v) != 0;
  if (const char* v = getenv("SDME_PA")) ctx->pa = atoi(v) != 0;
  if (const char* v = getenv("SDME_PDL")) ctx->pdl = atoi(v) != 0;
  const int P = d->P, n = P + 1, m = d->m;
  ctx->P = P;
  ctx->m = m;
  ctx->n = n;
  auto func_of = [&](int l) { return l == 0 ? 0 : (l == P ? 1 : l + 1); };
  ctx->Bl.resize(m * n);
  ctx->Dl.resize(m * n);
  ctx->w.assign(d->w, d->w + m);
  for (int a = 0; a < m; ++a)
    for (int l = 0; l < n; ++l) {
      ctx->Bl[a * n + l] = d->B[a * n + func_of(l)];
      ctx->Dl[a * n + l] = d->D[a * n + func_of(l)];
    }
  ctx->mir = detect_mirror(ctx);
  auto fail = [&](int code) {
    sdme_destroy(ctx);
    return code;
  };
  if (ctx->mir < 0) return fail(SDME_BAD_ARGUMENT);  // every reference basis mirrors
  Geo& g = ctx->geo;
  // elements as a row; one element box is a dense n^3 "lattice" (the staged
  // copies of element_col read E-vector boxes through the same code)
  g.nx = (int)d->n_elems; g.ny = 1; g.nz = 1;
  g.Lx = g.Ly = g.Lz = n; g.Px = n;
  g.Ns = (long long)n * n * n;
  g.s[0] = g.s[1] = g.s[2] = 1.0;
  g.detJ = 1.0;
  g.mu = d->mu; g.lam = d->lambda_lame; g.rho = d->rho0;
  ctx->nvec = d->n_free;
  ctx->nlat = d->n_free;
  ctx->n_free = d->n_free;
  const long long ns = d->n_elems * 3 * g.Ns;
  const long long nnz = d->asm_ptr[d->n_free];
  if (cudaStreamCreateWithFlags(&ctx->st, cudaStreamNonBlocking) != cudaSuccess) return fail(SDME_CUDA_ERROR);
  bool ok = cudaMalloc(&ctx->d_partial, kRedBlocks * 4 * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&ctx->d_scal, 16 * sizeof(double)) == cudaSuccess &&
            cudaMallocHost(&ctx->h_scal, 16 * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&ctx->d_flag, 2 * sizeof(unsigned long long)) == cudaSuccess &&
            cudaMallocHost(&ctx->h_flag, 2 * sizeof(unsigned long long)) == cudaSuccess &&
            cudaMalloc(&ctx->d_status, sizeof(int)) == cudaSuccess &&
            cudaMallocHost(&ctx->h_status, sizeof(int)) == cudaSuccess &&
            cudaMalloc(&ctx->d_free, ctx->nvec) == cudaSuccess &&
            cudaMalloc(&ctx->d_ev, ns * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&ctx->d_evu, ns * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&ctx->d_evp, ns * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&ctx->d_dof, ns * sizeof(int)) == cudaSuccess &&
            cudaMalloc(&ctx->d_aptr, (d->n_free + 1) * sizeof(long long)) == cudaSuccess &&
            cudaMalloc(&ctx->d_aslot, std::max<long long>(nnz, 1) * sizeof(int)) == cudaSuccess &&
            cudaMalloc(&ctx->d_geom, d->n_elems * 10 * g.Ns * sizeof(double)) == cudaSuccess;
  if (!ok) return fail(SDME_CUDA_ERROR);
  ctx->d_dflag = ctx->d_flag + 1;
  ok = cudaMemset(ctx->d_free, 1, ctx->nvec) == cudaSuccess &&
       cudaMemcpy(ctx->d_dof, d->dof, ns * sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(ctx->d_aptr, d->asm_ptr, (d->n_free + 1) * sizeof(long long), cudaMemcpyHostToDevice) ==
           cudaSuccess &&
       cudaMemcpy(ctx->d_aslot, d->asm_slot, nnz * sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess &&
       cudaMemcpy(ctx->d_geom, d->geom, d->n_elems * 10 * g.Ns * sizeof(double), cudaMemcpyHostToDevice) ==
           cudaSuccess;
  if (ok && d->elem_id)
    ok = cudaMalloc(&ctx->d_elem_id, d->n_elems * sizeof(int)) == cudaSuccess &&
         cudaMemcpy(ctx->d_elem_id, d->elem_id, d->n_elems * sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess;
  if (ok && d->asm_rows)
    ok = cudaMalloc(&ctx->d_asm_rows, d->n_free * sizeof(int)) == cudaSuccess &&
         cudaMemcpy(ctx->d_asm_rows, d->asm_rows, d->n_free * sizeof(int), cudaMemcpyHostToDevice) == cudaSuccess;
  if (!ok) return fail(SDME_CUDA_ERROR);
  *out = ctx;
  return SDME_OK;
}

int sdme_destroy(sdme_ctx* ctx) {
  if (!ctx) return SDME_OK;
  if (ctx->st) cudaStreamSynchronize(ctx->st);
  batch_free(ctx);
  for (double* p : ctx->vecs)
    if (p) cudaFree(p);
  for (void* p : ctx->vec_tmaps)
    if (p) cudaFree(p);
  cudaFree(ctx->d_perm);
  cudaFree(ctx->d_iperm);
  cudaFree(ctx->d_free);
  cudaFree(ctx->d_dof);
  cudaFree(ctx->d_aptr);
  cudaFree(ctx->d_aslot);
  cudaFree(ctx->d_elem_id);
  cudaFree(ctx->d_asm_rows);
  cudaFree(ctx->d_geom);
  cudaFree(ctx->d_evu);
  cudaFree(ctx->d_evp);
  cudaFree(ctx->d_ev);
  cudaFree(ctx->d_qpd);
  cudaFree(ctx->d_energy);
  if (ctx->pcg_exec) cudaGraphExecDestroy(ctx->pcg_exec);
  if (ctx->pcg_graph) cudaGraphDestroy(ctx->pcg_graph);
  cudaFree(ctx->d_fbuf);
  cudaFree(ctx->d_partial);
  cudaFree(ctx->d_scal);
  cudaFree(ctx->d_flag);
  cudaFree(ctx->d_gaps);
  if (ctx->h_scal) cudaFreeHost(ctx->h_scal);
  if (ctx->h_flag) cudaFreeHost(ctx->h_flag);
  cudaFree(ctx->d_status);
  if (ctx->h_status) cudaFreeHost(ctx->h_status);
  if (ctx->h_gaps) cudaFreeHost(ctx->h_gaps);
  if (ctx->st_side) cudaStreamDestroy(ctx->st_side);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->st) cudaStreamDestroy(ctx->st);
  delete ctx;
  return SDME_OK;
}

int sdme_lattice_size(const sdme_ctx* ctx, int64_t* n) {
  if (!ctx || !n) return SDME_BAD_ARGUMENT;
  *n = ctx->nlat;
  return SDME_OK;
}

int sdme_last_error(const sdme_ctx* ctx, int64_t* elem, int* qp, char* msg, size_t n) {
  if (!ctx) return SDME_BAD_ARGUMENT;
  if (elem) *elem = ctx->err_elem;
  if (qp) *qp = ctx->err_qp;
  if (msg && n) {
    strncpy(msg, ctx->err_msg.c_str(), n - 1);
    msg[n - 1] = 0;
  }
  return ctx->err_code;
}

int sdme_vec_alloc(sdme_ctx* ctx, int* id) {
  if (!ctx || !id) return SDME_BAD_ARGUMENT;
  return alloc_vec(ctx, id);
}

int sdme_vec_free(sdme_ctx* ctx, int id) {
  double* p = ctx ? vec(ctx, id) : nullptr;
  if (!p) return SDME_BAD_ARGUMENT;
  CK(cudaStreamSynchronize(ctx->st));
  cudaFree(p);
  ctx->vecs[id] = nullptr;
  if (ctx->vec_tmaps[id]) cudaFree(ctx->vec_tmaps[id]);
  ctx->vec_tmaps[id] = nullptr;
  return SDME_OK;
}

int sdme_vec_upload(sdme_ctx* ctx, int id, const double* host) {
  double* p = ctx ? vec(ctx, id) : nullptr;
  if (!p || !host) return SDME_BAD_ARGUMENT;
  // dense host rows (Lx doubles) -> pitched device rows (Px doubles)
  const Geo& g = ctx->geo;
  if (ctx->gen)  // general mesh: free-DOF arrays
    CK(cudaMemcpyAsync(p, host, ctx->nvec * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  else
    CK(cudaMemcpy2DAsync(p, g.Px * sizeof(double), host, g.Lx * sizeof(double), g.Lx * sizeof(double),
                         3LL * g.Ly * g.Lz, cudaMemcpyHostToDevice, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return SDME_OK;
}

int sdme_vec_download(sdme_ctx* ctx, int id, double* host) {
  double* p = ctx ? vec(ctx, id) : nullptr;
  if (!p || !host) return SDME_BAD_ARGUMENT;
  const Geo& g = ctx->geo;
  if (ctx->gen)
    CK(cudaMemcpyAsync(host, p, ctx->nvec * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
  else
    CK(cudaMemcpy2DAsync(host, g.Lx * sizeof(double), p, g.Px * sizeof(double), g.Lx * sizeof(double),
                         3LL * g.Ly * g.Lz, cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return SDME_OK;
}

int sdme_vec_upload_free(sdme_ctx* ctx, int id, const double* host) {
  if (ctx && ctx->gen) return sdme_vec_upload(ctx, id, host);
  double* p = ctx ? vec(ctx, id) : nullptr;
  if (!p || !host || !ctx->d_perm) return set_err(ctx, SDME_BAD_ARGUMENT, "no permutation / bad vector");
  CK(cudaMemcpyAsync(ctx->d_fbuf, host, ctx->n_free * sizeof(double), cudaMemcpyHostToDevice, ctx->st));
  k_free_to_lattice<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(p, ctx->d_fbuf, ctx->d_perm, ctx->nvec);
  ++ctx->launches;
  CK(cudaStreamSynchronize(ctx->st));
  return check_launch(ctx);
}

int sdme_vec_download_free(sdme_ctx* ctx, int id, double* host) {
  if (ctx && ctx->gen) return sdme_vec_download(ctx, id, host);
  double* p = ctx ? vec(ctx, id) : nullptr;
  if (!p || !host || !ctx->d_perm) return set_err(ctx, SDME_BAD_ARGUMENT, "no permutation / bad vector");
  k_lattice_to_free<<<grid_for(ctx->n_free), 256, 0, ctx->st>>>(ctx->d_fbuf, p, ctx->d_iperm, ctx->n_free);
  ++ctx->launches;
  CK(cudaMemcpyAsync(host, ctx->d_fbuf, ctx->n_free * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  return check_launch(ctx);
}

int sdme_vec_fill(sdme_ctx* ctx, int id, double value) {
  double* p = ctx ? vec(ctx, id) : nullptr;
  if (!p) return SDME_BAD_ARGUMENT;
  // value on free points, 0 on Dirichlet points
  k_fill_masked<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(p, ctx->d_free, value, ctx->nvec);
  ++ctx->launches;
  return check_launch(ctx);
}

int sdme_vec_copy(sdme_ctx* ctx, int dst, int src) {
  double* a = ctx ? vec(ctx, dst) : nullptr;
  double* b = ctx ? vec(ctx, src) : nullptr;
  if (!a || !b) return SDME_BAD_ARGUMENT;
  CK(cudaMemcpyAsync(a, b, ctx->nvec * sizeof(double), cudaMemcpyDeviceToDevice, ctx->st));
  return SDME_OK;
}

int sdme_vec_lincomb(sdme_ctx* ctx, int y, int nterms, const double* c, const int* x) {
  double* py = ctx ? vec(ctx, y) : nullptr;
  if (!py || nterms < 0 || nterms > 6) return SDME_BAD_ARGUMENT;
  LinComb lc{};
  lc.nt = nterms;
  for (int t = 0; t < nterms; ++t) {
    lc.x[t] = vec(ctx, x[t]);
    if (!lc.x[t]) return SDME_BAD_ARGUMENT;
    lc.c[t] = c[t];
  }
  k_lincomb<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(lc, py, ctx->nvec);
  ++ctx->launches;
  return check_launch(ctx);
}

int sdme_vec_mul(sdme_ctx* ctx, int out, int a, int b) {
  double* po = ctx ? vec(ctx, out) : nullptr;
  double* pa = ctx ? vec(ctx, a) : nullptr;
  double* pb = ctx ? vec(ctx, b) : nullptr;
  if (!po || !pa || !pb) return SDME_BAD_ARGUMENT;
  k_mul<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(po, pa, pb, ctx->nvec);
  ++ctx->launches;
  return check_launch(ctx);
}

int sdme_vec_dot(sdme_ctx* ctx, int a, int b, double* out) {
  double* pa = ctx ? vec(ctx, a) : nullptr;
  double* pb = ctx ? vec(ctx, b) : nullptr;
  if (!pa || !pb || !out) return SDME_BAD_ARGUMENT;
  int rc = dot_into(ctx, pa, pb, S_SCRATCH);
  if (rc) return rc;
  rc = read_scalars(ctx);
  if (rc) return rc;
  *out = ctx->h_scal[S_SCRATCH];
  return SDME_OK;
}

int sdme_vec_reciprocal(sdme_ctx* ctx, int dst, int src) {
  double* a = ctx ? vec(ctx, dst) : nullptr;
  double* b = ctx ? vec(ctx, src) : nullptr;
  if (!a || !b) return SDME_BAD_ARGUMENT;
  CK(cudaMemsetAsync(ctx->d_flag, 0xFF, sizeof(kNoFlag), ctx->st));  // = kNoFlag; no pageable H2D (implicit stream sync)
  k_invert_diag<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(a, b, ctx->d_free, ctx->nvec, ctx->d_flag);
  ++ctx->launches;
  CK(cudaMemcpyAsync(ctx->h_flag, ctx->d_flag, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaStreamSynchronize(ctx->st));
  if (*ctx->h_flag != kNoFlag)
    return set_err(ctx, SDME_BAD_DIAGONAL, "diagonal preconditioner needs positive diagonal entries",
                   (int64_t)*ctx->h_flag, -1);
  return check_launch(ctx);
}

int sdme_fint(sdme_ctx* ctx, int u, int r) {
  double* pu = ctx ? vec(ctx, u) : nullptr;
  double* pr = ctx ? vec(ctx, r) : nullptr;
  if (!pu || !pr) return SDME_BAD_ARGUMENT;
  int rc = reset_flag(ctx);
  if (rc) return rc;
  if ((rc = zero_output(ctx, pr))) return rc;
  ctx->ops->element(ctx, MODE_FINT, pu, nullptr, pr, 1.0, 0.0);
  rc = check_launch(ctx);
  if (rc) return rc;
  return check_flag(ctx);
}

int sdme_apply(sdme_ctx* ctx, int u, int p, int y, double c_k, double c_m) {
  double* pu = ctx ? vec(ctx, u) : nullptr;
  double* pp = ctx ? vec(ctx, p) : nullptr;
  double* py = ctx ? vec(ctx, y) : nullptr;
  if ((!pu && c_k != 0.0) || !pp || !py || py == pp) return SDME_BAD_ARGUMENT;
  int rc = reset_flag(ctx);
  if (rc) return rc;
  rc = apply_raw(ctx, pu, pp, py, c_k, c_m);
  if (rc) return rc;
  return c_k != 0.0 ? check_flag(ctx) : SDME_OK;
}

int sdme_mass(sdme_ctx* ctx, int a, int y) {
  double* pa = ctx ? vec(ctx, a) : nullptr;
  double* py = ctx ? vec(ctx, y) : nullptr;
  if (!pa || !py || pa == py) return SDME_BAD_ARGUMENT;
  return apply_raw(ctx, nullptr, pa, py, 0.0, 1.0);
}

// One Newton iterate's residual of newmark_run (dynamics.py:213-226) as one
// enqueued sequence with a single host synchronisation: [uk += du]; tmp = uk -
// u; atr = b1 tmp - b2 v - b3 a; tmp = f_int(uk); psi = M atr; psi = s load -
// tmp - psi; ||psi||.  The same kernels in the same order as the separate
// calls, so results are bit-identical to them.
int sdme_newmark_residual(sdme_ctx* ctx, int uk, int du, int u, int v, int a, int load, double s_load, double b1,
                          double b2, double b3, int atr, int tmp, int psi, double* norm) {
  if (!ctx || !norm) return SDME_BAD_ARGUMENT;
  double *puk = vec(ctx, uk), *pu = vec(ctx, u), *pv = vec(ctx, v), *pa = vec(ctx, a);
  double *patr = vec(ctx, atr), *ptmp = vec(ctx, tmp), *ppsi = vec(ctx, psi);
  double* pdu = du >= 0 ? vec(ctx, du) : nullptr;
  double* pl = load >= 0 ? vec(ctx, load) : nullptr;
  if (!puk || !pu || !pv || !pa || !patr || !ptmp || !ppsi || (du >= 0 && !pdu) || (load >= 0 && !pl))
    return SDME_BAD_ARGUMENT;
  const int grid = grid_for(ctx->nvec);
  auto lincomb = [&](double* y, std::initializer_list<std::pair<double, const double*>> terms) {
    LinComb lc{};
    lc.nt = 0;
    for (auto& t : terms) {
      lc.c[lc.nt] = t.first;
      lc.x[lc.nt] = t.second;
      ++lc.nt;
    }
    k_lincomb<<<grid, 256, 0, ctx->st>>>(lc, y, ctx->nvec);
    ++ctx->launches;
  };
  if (pdu) lincomb(puk, {{1.0, puk}, {1.0, pdu}});
  lincomb(ptmp, {{1.0, puk}, {-1.0, pu}});
  lincomb(patr, {{b1, ptmp}, {-b2, pv}, {-b3, pa}});
  int rc = reset_flag(ctx);
  if (rc) return rc;
  if ((rc = zero_output(ctx, ptmp))) return rc;
  ctx->ops->element(ctx, MODE_FINT, puk, nullptr, ptmp, 1.0, 0.0);
  if ((rc = apply_raw(ctx, nullptr, patr, ppsi, 0.0, 1.0))) return rc;
  if (pl)
    lincomb(ppsi, {{s_load, pl}, {-1.0, ptmp}, {-1.0, ppsi}});
  else
    lincomb(ppsi, {{-1.0, ptmp}, {-1.0, ppsi}});
  if ((rc = dot_into(ctx, ppsi, ppsi, S_SCRATCH))) return rc;
  CK(cudaMemcpyAsync(ctx->h_flag, ctx->d_flag, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->st));
  if ((rc = read_scalars(ctx)) || (rc = check_launch(ctx))) return rc;
  if ((rc = flag_error(ctx, ctx->h_flag[0]))) return rc;
  *norm = std::sqrt(ctx->h_scal[S_SCRATCH]);
  return SDME_OK;
}

int sdme_diag(sdme_ctx* ctx, int u, double c_k, double c_m, int d) {
  double* pu = ctx ? vec(ctx, u) : nullptr;
  double* pd = ctx ? vec(ctx, d) : nullptr;
  if ((!pu && c_k != 0.0) || !pd) return SDME_BAD_ARGUMENT;
  int rc = reset_flag(ctx);
  if (rc) return rc;
  CK(cudaMemsetAsync(pd, 0, ctx->nvec * sizeof(double), ctx->st));
  ctx->ops->diag(ctx, pu, pd, c_k, c_m);
  rc = check_launch(ctx);
  if (rc) return rc;
  return c_k != 0.0 ? check_flag(ctx) : SDME_OK;
}

int sdme_pcg(sdme_ctx* ctx, int u_lin, double c_k, double c_m, int b, int x, double tol, int maxit,
             int precond, int* iters, double* relres) {
  if (!ctx) return SDME_BAD_ARGUMENT;
  double* pu = vec(ctx, u_lin);
  double* pb = vec(ctx, b);
  double* px = vec(ctx, x);
  if ((!pu && c_k != 0.0) || !pb || !px || pb == px || maxit < 0)
    return set_err(ctx, SDME_BAD_ARGUMENT, "bad vector id");
  if (!(tol > 0.0 && tol < 1.0)) return set_err(ctx, SDME_BAD_ARGUMENT, "tolerance must lie in (0, 1)");
  int rc;
  if ((rc = ensure(ctx, ctx->v_r)) || (rc = ensure(ctx, ctx->v_p)) || (rc = ensure(ctx, ctx->v_ap)) ||
      (rc = ensure(ctx, ctx->v_dinv)))
    return rc;
  double* r = vec(ctx, ctx->v_r);
  double* p = vec(ctx, ctx->v_p);
  double* ap = vec(ctx, ctx->v_ap);
  double* dinv = vec(ctx, ctx->v_dinv);
  if (iters) *iters = 0;
  if (relres) *relres = 0.0;
  if (precond != 0 && precond != 1)
    return set_err(ctx, SDME_BAD_ARGUMENT, "unknown preconditioner (out of scope: sgs)");
  // Everything up to the end of the iterations is queued without a host
  // wait; the outcomes (element inversion in the diagonal, non-positive
  // diagonal, ||b|| = 0, converged / indefinite / maxit) are read back once
  // and reported in the reference's order (solver.py:102-170).
  if ((rc = reset_flag(ctx))) return rc;
  CK(cudaMemsetAsync(ctx->d_dflag, 0xFF, sizeof(kNoFlag), ctx->st));  // = kNoFlag
  // K(u) is fixed during the solve: store K = F^-T and ln J at the quadrature
  // points once (MODE_SETUP, flags inverted elements) and iterate with MODE_PA
  const bool pa = c_k != 0.0 && ctx->pa && ensure_qpd(ctx);
  const bool withc = c_k != 0.0 && ctx->pcg_contact && ctx->c_ready;
  if (pa) ctx->ops->element(ctx, MODE_SETUP, pu, nullptr, nullptr, 1.0, 0.0);
  // SDME_PCG_START=0: the start of the solve as separate launches (A/B, bit-identical)
  const bool fused_start = ctx->pcg_start;
  if (precond == 1) {
    CK(cudaMemsetAsync(ap, 0, ctx->nvec * sizeof(double), ctx->st));
    ctx->ops->diag(ctx, pu, ap, c_k, c_m);
    if (withc) contact_op(ctx, CONTACT_DIAG, nullptr, ap, nullptr);
  }
  if (fused_start) {
    // dinv, ||b||, x = 0, r = b, p = z = dinv r, rz = r.z, scalar state and status: two launches
    k_pcg_start<<<kRedBlocks, kRedThreads, 0, ctx->st>>>(dinv, precond == 1 ? ap : nullptr, ctx->d_free, pb, px, r,
                                                         p, ctx->nvec, ctx->d_partial, ctx->d_dflag);
    k_pcg_start_finish<<<1, kRedThreads, 0, ctx->st>>>(ctx->d_partial, ctx->d_scal, tol, (double)maxit,
                                                       ctx->d_status, ctx->d_flag);
    ctx->launches += 2;
    if ((rc = check_launch(ctx))) return rc;
  } else {
    if (precond == 1)
      k_invert_diag<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(dinv, ap, ctx->d_free, ctx->nvec, ctx->d_dflag);
    else
      k_fill_masked<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(dinv, ctx->d_free, 1.0, ctx->nvec);
    ++ctx->launches;
    // ||b||, scalar state and status word on the device; r = b ; p = z = dinv r ; rz = r.z
    if ((rc = dot_into(ctx, pb, pb, S_SCRATCH))) return rc;
    k_pcg_init<<<1, 32, 0, ctx->st>>>(ctx->d_scal, tol, (double)maxit, ctx->d_status, ctx->d_flag);
    ++ctx->launches;
    CK(cudaMemsetAsync(px, 0, ctx->nvec * sizeof(double), ctx->st));
    CK(cudaMemcpyAsync(r, pb, ctx->nvec * sizeof(double), cudaMemcpyDeviceToDevice, ctx->st));
    k_mul<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(p, dinv, r, ctx->nvec);
    ++ctx->launches;
    if ((rc = dot_into(ctx, r, p, S_RZ0))) return rc;
  }
  if (maxit > 0) {
    // warm the operator's one-time launch setup (function attributes,
    // occupancy queries) outside the capture, once per operator kind
    const int kind = (c_k != 0.0 ? 1 : 0) | (c_m != 0.0 ? 2 : 0) | (pa ? 4 : 0);
    if (!(ctx->pcg_warm & (1 << kind))) {
      CK(cudaMemsetAsync(ap, 0, ctx->nvec * sizeof(double), ctx->st));
      if (c_k != 0.0)
        ctx->ops->element(ctx, pa ? MODE_PA : MODE_APPLY, pu, p, ap, c_k, c_m);
      else
        ctx->ops->element(ctx, MODE_MASS, nullptr, p, ap, 0.0, c_m);
      if ((rc = check_launch(ctx))) return rc;
      ctx->pcg_warm |= 1 << kind;
    }
    // large-mesh sequence with k_pcg_p2 zeroing A p for the next iteration:
    // the first iteration's zero (after the warm-up pass above may have used ap)
    if (ctx->pdl && (chain_mode_of(ctx) & 9) == 9) CK(cudaMemsetAsync(ap, 0, ctx->nvec * sizeof(double), ctx->st));
    // one graph launch per solve (build_pcg_graph); the instantiated graph is
    // reused while the operands are the same (every Newton step of a run)
    const sdme_ctx::PcgKey key{pu, px, c_k, c_m, pa, withc, withc ? ctx->c_ca.eps : 0.0,
                               withc ? ctx->c_gen : 0ull};
    if (ctx->pcg_direct) {
      // profiling aid (SDME_PCG_DIRECT=1): plain launches, one host check per
      // iteration, so per-kernel tools see every launch
      for (int it = 0; it <= maxit; ++it) {
        enqueue_pcg_iteration(ctx, pu, px, r, p, ap, dinv, c_k, c_m, pa, withc, 0, 0);
        CK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
        CK(cudaStreamSynchronize(ctx->st));
        if (*ctx->h_status != PCG_RUNNING) break;
      }
      ctx->pcg_per_iter = 0;
    } else if (!ctx->pcg_exec || !(key == ctx->pcg_key)) {
      if (ctx->pcg_exec) cudaGraphExecDestroy(ctx->pcg_exec);
      if (ctx->pcg_graph) cudaGraphDestroy(ctx->pcg_graph);
      ctx->pcg_exec = nullptr;
      ctx->pcg_graph = nullptr;
      if ((rc = build_pcg_graph(ctx, pu, px, r, p, ap, dinv, c_k, c_m, pa, withc))) return rc;
      ctx->pcg_key = key;
    }
    if (!ctx->pcg_direct) CK(cudaGraphLaunch(ctx->pcg_exec, ctx->st));
  }
  CK(cudaMemcpyAsync(ctx->h_flag, ctx->d_flag, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->st));
  CK(cudaMemcpyAsync(ctx->h_status, ctx->d_status, sizeof(int), cudaMemcpyDeviceToHost, ctx->st));
  if ((rc = read_scalars(ctx)) || (rc = check_launch(ctx))) return rc;
  if (c_k != 0.0 && (rc = flag_error(ctx, ctx->h_flag[0]))) return rc;
  if (precond == 1 && ctx->h_flag[1] != kNoFlag)
    return set_err(ctx, SDME_BAD_DIAGONAL, "diagonal preconditioner needs positive diagonal entries",
                   (int64_t)ctx->h_flag[1], -1);
  const double nb = ctx->h_scal[S_NB];
  if (nb == 0.0) return SDME_OK;
  int status = PCG_MAXIT;
  if (maxit > 0) {
    status = *ctx->h_status;
    const int it = (int)ctx->h_scal[S_ITER];
    ctx->launches += ctx->pcg_per_iter * it;
    if (status == PCG_CONVERGED) {
      if (iters) *iters = it;
      if (relres) *relres = ctx->h_scal[S_STOPREL];
      return SDME_OK;
    }
    if (status == PCG_INDEFINITE) {
      if (iters) *iters = it;
      if (relres) *relres = ctx->h_scal[S_STOPREL];
      char buf[128];
      snprintf(buf, sizeof buf, "indefinite operator detected at iteration %d (p^T A p = %.3e)", it,
               ctx->h_scal[S_PAP]);
      return set_err(ctx, SDME_INDEFINITE, buf);
    }
  }
  // maxit: true residual ||b - A x|| / ||b||  (solver.py:166)
  if ((rc = apply_raw(ctx, pu, px, ap, c_k, c_m))) return rc;
  {
    LinComb lc{};
    lc.nt = 2;
    lc.x[0] = pb;
    lc.x[1] = ap;
    lc.c[0] = 1.0;
    lc.c[1] = -1.0;
    k_lincomb<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(lc, r, ctx->nvec);
    ++ctx->launches;
  }
  if ((rc = dot_into(ctx, r, r, S_SCRATCH)) || (rc = read_scalars(ctx))) return rc;
  const double rel = std::sqrt(ctx->h_scal[S_SCRATCH]) / nb;
  if (iters) *iters = maxit;
  if (relres) *relres = rel;
  char buf[128];
  snprintf(buf, sizeof buf, "PCG did not converge in %d iterations (relative residual %.3e)", maxit, rel);
  return set_err(ctx, SDME_MAXIT, buf);
}

int sdme_explicit_step(sdme_ctx* ctx, int u, int u_prev, int v, int load, double s_load, int fc,
                       int inv_ml, double dt, int scratch) {
  if (!ctx) return SDME_BAD_ARGUMENT;
  double *pu = vec(ctx, u), *pup = vec(ctx, u_prev), *pv = vec(ctx, v), *pm = vec(ctx, inv_ml),
         *ps = vec(ctx, scratch);
  const double* pl = load >= 0 ? vec(ctx, load) : nullptr;
  const double* pf = fc >= 0 ? vec(ctx, fc) : nullptr;
  if (!pu || !pup || !pv || !pm || !ps || (load >= 0 && !pl) || (fc >= 0 && !pf) || !(dt > 0.0))
    return set_err(ctx, SDME_BAD_ARGUMENT, "bad explicit-step argument");
  int rc = sdme_fint(ctx, u, scratch);
  if (rc) return rc;
  k_explicit_step<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(pu, pup, pv, pl, s_load, ps, pf, pm, dt, ctx->nvec);
  ++ctx->launches;
  return check_launch(ctx);
}

// n central-difference steps back to back on the context stream (no host
// round trip per step): per step the contact force at u with the parameters
// of the last sdme_contact call (if fc >= 0), f_int, and the update with load
// scale s_load[k] (load >= 0).  The inversion flag is read once at the end;
// it carries the smallest (element, point) over all n steps, so a caller that
// needs the first inverted step replays the chunk step by step.
int sdme_explicit_steps(sdme_ctx* ctx, int n, int u, int u_prev, int v, int load, const double* s_load, int fc,
                        int inv_ml, double dt, int scratch) {
  if (!ctx || n < 0) return SDME_BAD_ARGUMENT;
  double *pu = vec(ctx, u), *pup = vec(ctx, u_prev), *pv = vec(ctx, v), *pm = vec(ctx, inv_ml),
         *ps = vec(ctx, scratch);
  const double* pl = load >= 0 ? vec(ctx, load) : nullptr;
  double* pf = fc >= 0 ? vec(ctx, fc) : nullptr;
  if (!pu || !pup || !pv || !pm || !ps || (load >= 0 && (!pl || !s_load)) || (fc >= 0 && (!pf || !ctx->c_ready)) ||
      !(dt > 0.0))
    return set_err(ctx, SDME_BAD_ARGUMENT, "bad explicit-steps argument");
  int rc = reset_flag(ctx);
  if (rc) return rc;
  // The contact force (4 small face-colour launches, ~8 us each) and f_int
  // (8 colour passes) of a step both read u and write different vectors:
  // the contact runs on a side stream beside the passes and joins before the
  // update (config 4: 0.123 -> 0.10 ms per step).  SDME_CONTACT_SIDE=0: in line.
  static const bool side_on = [] {
    const char* e = getenv("SDME_CONTACT_SIDE");
    return !(e && e[0] == '0');
  }();
  const bool side = pf && side_on;
  if (side && !ctx->st_side) {
    CK(cudaStreamCreateWithFlags(&ctx->st_side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  }
  for (int k = 0; k < n; ++k) {
    if (pf) {
      ContactArgs ca = ctx->c_ca;
      ca.mode = CONTACT_FORCE;
      ca.u = pu;
      ca.fc = pf;
      cudaStream_t main = ctx->st;
      if (side) {
        CK(cudaEventRecord(ctx->ev_fork, main));
        CK(cudaStreamWaitEvent(ctx->st_side, ctx->ev_fork, 0));
        ctx->st = ctx->st_side;  // launch_contact launches on ctx->st
      }
      const cudaError_t me = cudaMemsetAsync(pf, 0, ctx->nvec * sizeof(double), ctx->st);
      launch_contact(ctx, ca);
      ctx->st = main;
      if (me != cudaSuccess) return set_err(ctx, SDME_CUDA_ERROR, cudaGetErrorString(me));
      if (side) CK(cudaEventRecord(ctx->ev_join, ctx->st_side));
    }
    if ((rc = zero_output(ctx, ps))) return rc;  // PDL primary of the first colour pass
    ctx->ops->element(ctx, MODE_FINT, pu, nullptr, ps, 1.0, 0.0);
    ctx->pdl_first = false;
    if (side) CK(cudaStreamWaitEvent(ctx->st, ctx->ev_join, 0));
    k_explicit_step<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(pu, pup, pv, pl, pl ? s_load[k] : 0.0, ps, pf, pm,
                                                             dt, ctx->nvec);
    ++ctx->launches;
  }
  rc = check_launch(ctx);
  if (rc) return rc;
  return check_flag(ctx);
}

int sdme_contact_points(const sdme_ctx* ctx, int side, int qf, int64_t* n) {
  if (!ctx || ctx->gen || side < 0 || side > 5 || qf < 1 || !n) return SDME_BAD_ARGUMENT;
  const int axis = side / 2;
  const int ne[3] = {ctx->geo.nx, ctx->geo.ny, ctx->geo.nz};
  const int d1 = axis == 0 ? 1 : 0, d2 = axis == 2 ? 1 : 2;
  *n = (int64_t)ne[d1] * ne[d2] * qf * qf;
  return SDME_OK;
}

int sdme_contact(sdme_ctx* ctx, int u, int side, int qf, const double* Bf, const double* xf, const double* wf,
                 const double* point, const double* normal, double eps, int fc, double* gaps_host,
                 double* stats) {
  if (!ctx) return SDME_BAD_ARGUMENT;
  if (ctx->gen) return set_err(ctx, SDME_BAD_ARGUMENT, "contact needs a box-mesh context");
  double* pu = vec(ctx, u);
  double* pf = vec(ctx, fc);
  if (!pu || !pf || side < 0 || side > 5 || qf < 1 || qf > kMaxQF || ctx->n > kMaxN || !Bf || !xf || !wf ||
      !point || !normal)
    return set_err(ctx, SDME_BAD_ARGUMENT, "bad contact argument");
  int64_t npts = 0;
  sdme_contact_points(ctx, side, qf, &npts);
  if (npts > ctx->gaps_cap) {
    // a cached PCG graph may hold the old gaps pointer: invalidate it first
    CK(cudaStreamSynchronize(ctx->st));
    cudaFree(ctx->d_gaps);
    if (ctx->h_gaps) cudaFreeHost(ctx->h_gaps);
    ctx->d_gaps = nullptr;
    ctx->h_gaps = nullptr;
    ctx->gaps_cap = 0;
    ++ctx->c_gen;
    CK(cudaMalloc(&ctx->d_gaps, npts * sizeof(double)));
    CK(cudaMallocHost(&ctx->h_gaps, npts * sizeof(double)));
    ctx->gaps_cap = npts;
  }
  FaceTab ft{};
  ft.n = ctx->n;
  ft.qf = qf;
  const int P = ctx->P;
  auto func_of = [&](int l) { return l == 0 ? 0 : (l == P ? 1 : l + 1); };
  for (int a = 0; a < qf; ++a) {
    for (int l = 0; l < ctx->n; ++l) ft.B[a][l] = Bf[a * ctx->n + func_of(l)];
    ft.W[a] = wf[a];
    ft.X[a] = xf[a];
  }
  ContactArgs ca{};
  ca.axis = side / 2;
  ca.side = side % 2;
  const double nrm = std::sqrt(normal[0] * normal[0] + normal[1] * normal[1] + normal[2] * normal[2]);
  for (int c = 0; c < 3; ++c) {
    ca.origin[c] = ctx->origin[c];
    ca.h[c] = ctx->h[c];
    ca.point[c] = point[c];
    ca.normal[c] = std::fabs(nrm - 1.0) > 1e-12 ? normal[c] / nrm : normal[c];
  }
  ca.eps = eps;
  ca.u = pu;
  ca.fc = pf;
  ca.gaps = ctx->d_gaps;
  ca.mode = CONTACT_FORCE;
  {
    // what a captured contact node depends on: face tables and the plane /
    // penalty arguments (u and fc are replaced per launch by contact_op)
    ContactArgs a0 = ctx->c_ca, a1 = ca;
    a0.u = a1.u = nullptr;
    a0.fc = a1.fc = nullptr;
    if (!ctx->c_ready || memcmp(&ctx->c_ft, &ft, sizeof(ft)) != 0 || memcmp(&a0, &a1, sizeof(a0)) != 0)
      ++ctx->c_gen;
  }
  ctx->c_ft = ft;
  ctx->c_ca = ca;
  ctx->c_ready = true;
  CK(cudaMemsetAsync(pf, 0, ctx->nvec * sizeof(double), ctx->st));
  const int ne[3] = {ctx->geo.nx, ctx->geo.ny, ctx->geo.nz};
  const int d1 = ca.axis == 0 ? 1 : 0, d2 = ca.axis == 2 ? 1 : 2;
  launch_contact(ctx, ca);
  int rc = check_launch(ctx);
  if (rc) return rc;
  if (gaps_host || stats) {
    CK(cudaMemcpyAsync(ctx->h_gaps, ctx->d_gaps, npts * sizeof(double), cudaMemcpyDeviceToHost, ctx->st));
    CK(cudaStreamSynchronize(ctx->st));
    if (gaps_host) memcpy(gaps_host, ctx->h_gaps, npts * sizeof(double));
    if (stats) {
      double pen = 0.0, tmin = 0.0;
      long long act = 0;
      bool any = false;
      for (int64_t i = 0; i < npts; ++i) {
        const double gp = ctx->h_gaps[i];
        pen = std::max(pen, -gp);
        if (gp < 0.0) {
          const double tn = -eps * gp;
          tmin = any ? std::min(tmin, tn) : tn;
          any = true;
          ++act;
        }
      }
      stats[0] = std::max(pen, 0.0);
      stats[1] = any ? tmin : 0.0;
      stats[2] = (double)act;
    }
  }
  return SDME_OK;
}

int sdme_lattice_address(const sdme_ctx* ctx, int c, int x, int y, int z, int64_t* addr) {
  if (!ctx || !addr || ctx->gen || c < 0 || c > 2) return SDME_BAD_ARGUMENT;
  const Geo& g = ctx->geo;
  if (x < 0 || x >= g.Lx || y < 0 || y >= g.Ly || z < 0 || z >= g.Lz) return SDME_BAD_ARGUMENT;
  *addr = c * g.Ns + ((int64_t)z * g.Ly + y) * g.Px + x;
  return SDME_OK;
}

int sdme_strain_energy(sdme_ctx* ctx, int u, double* out) {
  double* pu = ctx ? vec(ctx, u) : nullptr;
  if (!pu || !out) return SDME_BAD_ARGUMENT;
  if (ctx->gen) return set_err(ctx, SDME_BAD_ARGUMENT, "strain energy needs a box-mesh context");
  const long long ne = (long long)ctx->geo.nx * ctx->geo.ny * ctx->geo.nz;
  if (!ctx->d_energy) {
    // per-element energies, then the m rule weights (read by the kernel through p)
    CK(cudaMalloc(&ctx->d_energy, (ne + ctx->m) * sizeof(double)));
    CK(cudaMemcpy(ctx->d_energy + ne, ctx->w.data(), ctx->m * sizeof(double), cudaMemcpyHostToDevice));
  }
  int rc = reset_flag(ctx);
  if (rc) return rc;
  ctx->ops->element(ctx, MODE_ENERGY, pu, ctx->d_energy + ne, ctx->d_energy, 1.0, 0.0);
  k_sum<<<kRedBlocks, kRedThreads, 0, ctx->st>>>(ctx->d_energy, ne, ctx->d_partial);
  k_finish<1><<<1, kRedThreads, 0, ctx->st>>>(ctx->d_partial, ctx->d_scal + S_SCRATCH);
  ctx->launches += 2;
  if ((rc = check_flag(ctx)) || (rc = read_scalars(ctx))) return rc;
  *out = ctx->h_scal[S_SCRATCH];
  return check_launch(ctx);
}

int sdme_contact_apply(sdme_ctx* ctx, int p, int y) {
  double* pp = ctx ? vec(ctx, p) : nullptr;
  double* py = ctx ? vec(ctx, y) : nullptr;
  if (!pp || !py || pp == py) return SDME_BAD_ARGUMENT;
  if (!ctx->c_ready) return set_err(ctx, SDME_BAD_ARGUMENT, "no contact evaluation yet (sdme_contact)");
  contact_op(ctx, CONTACT_APPLY, pp, py, nullptr);
  return check_launch(ctx);
}

int sdme_contact_diag(sdme_ctx* ctx, int d) {
  double* pd = ctx ? vec(ctx, d) : nullptr;
  if (!pd) return SDME_BAD_ARGUMENT;
  if (!ctx->c_ready) return set_err(ctx, SDME_BAD_ARGUMENT, "no contact evaluation yet (sdme_contact)");
  contact_op(ctx, CONTACT_DIAG, nullptr, pd, nullptr);
  return check_launch(ctx);
}

int sdme_pcg_contact(sdme_ctx* ctx, int on) {
  if (!ctx) return SDME_BAD_ARGUMENT;
  ctx->pcg_contact = on != 0;
  return SDME_OK;
}

int sdme_time_op(sdme_ctx* ctx, int op, int u, int p, int y, double c_m, int reps, double* ms) {
  if (!ctx || reps < 1 || !ms) return SDME_BAD_ARGUMENT;
  double *pu = vec(ctx, u), *pp = vec(ctx, p), *py = vec(ctx, y);
  if (!pu || !pp || !py) return SDME_BAD_ARGUMENT;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaStreamSynchronize(ctx->st));
  CK(cudaEventRecord(e0, ctx->st));
  for (int r = 0; r < reps; ++r) {
    switch (op) {
      case 0: apply_raw(ctx, pu, pp, py, 1.0, c_m); break;
      case 1:
        zero_output(ctx, py);
        ctx->ops->element(ctx, MODE_FINT, pu, nullptr, py, 1.0, 0.0);
        break;
      case 2: apply_raw(ctx, nullptr, pp, py, 0.0, 1.0); break;
      case 3:
        cudaMemsetAsync(py, 0, ctx->nvec * sizeof(double), ctx->st);
        ctx->ops->diag(ctx, pu, py, 1.0, c_m);
        break;
      case 4:  // quadrature-data setup at u
        if (!ensure_qpd(ctx)) return SDME_CUDA_ERROR;
        ctx->ops->element(ctx, MODE_SETUP, pu, nullptr, nullptr, 1.0, 0.0);
        break;
      case 5:  // K.p (+ c_m M p) from the stored quadrature data (PCG operator)
        if (!ctx->d_qpd) return SDME_BAD_ARGUMENT;
        zero_output(ctx, py);
        ctx->ops->element(ctx, MODE_PA, pu, pp, py, 1.0, c_m);
        break;
      default: return SDME_BAD_ARGUMENT;
    }
  }
  CK(cudaEventRecord(e1, ctx->st));
  CK(cudaEventSynchronize(e1));
  float t = 0.f;
  CK(cudaEventElapsedTime(&t, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms = (double)t / reps;
  return check_launch(ctx);
}

void batch_free(sdme_ctx* ctx);

// Pipelined batch K.p with host buffers (the e2e path of many operator
// applications): pair k's H2D copies (copy stream 1) and result k-1's D2H copy
// (copy stream 2) overlap the permutations and operator of pair k on the
// context stream.  Free-order staging is double-buffered; events order reuse.
int batch_setup(sdme_ctx* ctx) {
  if (ctx->batch) return SDME_OK;
  auto* b = new sdme_ctx::Batch();
  ctx->batch = b;
  bool ok = cudaStreamCreateWithFlags(&b->h2d, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&b->h2d2, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&b->d2h, cudaStreamNonBlocking) == cudaSuccess;
  for (int i = 0; ok && i < 2; ++i) {
    ok = cudaMalloc(&b->su[i], ctx->n_free * sizeof(double)) == cudaSuccess &&
         cudaMalloc(&b->sp[i], ctx->n_free * sizeof(double)) == cudaSuccess &&
         cudaMalloc(&b->sy[i], ctx->n_free * sizeof(double)) == cudaSuccess;
    for (cudaEvent_t* e : {&b->ev_h2d[i], &b->ev_h2d2[i], &b->ev_in_free[i], &b->ev_comp[i], &b->ev_out_free[i]})
      ok = ok && cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess;
  }
  int rc = ok ? alloc_vec(ctx, &b->u) : SDME_CUDA_ERROR;
  if (!rc) rc = alloc_vec(ctx, &b->p);
  if (!rc) rc = alloc_vec(ctx, &b->y);
  if (rc) {  // leave no half-built pipeline behind
    batch_free(ctx);
    cudaGetLastError();
    return set_err(ctx, SDME_CUDA_ERROR, "batch apply: allocation failed");
  }
  return SDME_OK;
}

void batch_free(sdme_ctx* ctx) {
  auto* b = ctx->batch;
  if (!b) return;
  for (int id : {b->u, b->p, b->y})
    if (id >= 0 && vec(ctx, id)) {
      cudaFree(ctx->vecs[id]);
      ctx->vecs[id] = nullptr;
      if (ctx->vec_tmaps[id]) cudaFree(ctx->vec_tmaps[id]);
      ctx->vec_tmaps[id] = nullptr;
    }
  for (int i = 0; i < 2; ++i) {
    cudaFree(b->su[i]);
    cudaFree(b->sp[i]);
    cudaFree(b->sy[i]);
    for (cudaEvent_t e : {b->ev_h2d[i], b->ev_h2d2[i], b->ev_in_free[i], b->ev_comp[i], b->ev_out_free[i]})
      if (e) cudaEventDestroy(e);
  }
  if (b->h2d) cudaStreamDestroy(b->h2d);
  if (b->h2d2) cudaStreamDestroy(b->h2d2);
  if (b->d2h) cudaStreamDestroy(b->d2h);
  delete b;
  ctx->batch = nullptr;
}

int sdme_apply_batch(sdme_ctx* ctx, int n, const double* const* u, const double* const* p, double* const* y,
                     double c_k, double c_m) {
  if (!ctx || n < 0 || (!u && c_k != 0.0) || !p || !y) return SDME_BAD_ARGUMENT;
  if (!ctx->d_perm) return set_err(ctx, SDME_BAD_ARGUMENT, "batch apply needs a box context with a permutation");
  int rc = batch_setup(ctx);
  if (rc) return rc;
  if ((rc = reset_flag(ctx))) return rc;
  auto* b = ctx->batch;
  double* U = vec(ctx, b->u);
  double* Pv = vec(ctx, b->p);
  double* Y = vec(ctx, b->y);
  const size_t bytes = ctx->n_free * sizeof(double);
  for (int k = 0; k < n; ++k) {
    const int s = k & 1;
    // H2D of pair k into staging s (free once the permutations of pair k-2 ran)
    if (k >= 2) {
      CK(cudaStreamWaitEvent(b->h2d, b->ev_in_free[s], 0));
      CK(cudaStreamWaitEvent(b->h2d2, b->ev_in_free[s], 0));
    }
    if (c_k != 0.0) CK(cudaMemcpyAsync(b->su[s], u[k], bytes, cudaMemcpyHostToDevice, b->h2d));
    CK(cudaMemcpyAsync(b->sp[s], p[k], bytes, cudaMemcpyHostToDevice, b->h2d2));
    CK(cudaEventRecord(b->ev_h2d[s], b->h2d));
    CK(cudaEventRecord(b->ev_h2d2[s], b->h2d2));
    // operator on the context stream
    CK(cudaStreamWaitEvent(ctx->st, b->ev_h2d[s], 0));
    CK(cudaStreamWaitEvent(ctx->st, b->ev_h2d2[s], 0));
    if (c_k != 0.0) k_free_to_lattice<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(U, b->su[s], ctx->d_perm, ctx->nvec);
    k_free_to_lattice<<<grid_for(ctx->nvec), 256, 0, ctx->st>>>(Pv, b->sp[s], ctx->d_perm, ctx->nvec);
    ctx->launches += c_k != 0.0 ? 2 : 1;
    CK(cudaEventRecord(b->ev_in_free[s], ctx->st));
    CK(cudaMemsetAsync(Y, 0, ctx->nvec * sizeof(double), ctx->st));
    if (c_k != 0.0)
      ctx->ops->element(ctx, MODE_APPLY, U, Pv, Y, c_k, c_m);
    else
      ctx->ops->element(ctx, MODE_MASS, nullptr, Pv, Y, 0.0, c_m);
    if (k >= 2) CK(cudaStreamWaitEvent(ctx->st, b->ev_out_free[s], 0));
    k_lattice_to_free<<<grid_for(ctx->n_free), 256, 0, ctx->st>>>(b->sy[s], Y, ctx->d_iperm, ctx->n_free);
    ++ctx->launches;
    CK(cudaEventRecord(b->ev_comp[s], ctx->st));
    // D2H of result k
    CK(cudaStreamWaitEvent(b->d2h, b->ev_comp[s], 0));
    CK(cudaMemcpyAsync(y[k], b->sy[s], bytes, cudaMemcpyDeviceToHost, b->d2h));
    CK(cudaEventRecord(b->ev_out_free[s], b->d2h));
  }
  CK(cudaStreamSynchronize(b->d2h));
  CK(cudaStreamSynchronize(ctx->st));
  rc = check_launch(ctx);
  if (rc) return rc;
  return c_k != 0.0 ? check_flag(ctx) : SDME_OK;
}

int sdme_host_alloc(size_t bytes, void** ptr) {
  if (!ptr) return SDME_BAD_ARGUMENT;
  return cudaMallocHost(ptr, bytes) == cudaSuccess ? SDME_OK : SDME_CUDA_ERROR;
}

int sdme_host_free(void* ptr) {
  return cudaFreeHost(ptr) == cudaSuccess ? SDME_OK : SDME_CUDA_ERROR;
}

int sdme_sync(sdme_ctx* ctx) {
  if (!ctx) return SDME_BAD_ARGUMENT;
  CK(cudaStreamSynchronize(ctx->st));
  return SDME_OK;
}

int sdme_launch_count(const sdme_ctx* ctx, int64_t* n) {
  if (!ctx || !n) return SDME_BAD_ARGUMENT;
  *n = ctx->launches;
  return SDME_OK;
}

}  // extern "C"
