/* sdme.h -- C ABI of the B200 matrix-free neo-Hookean path (sm_100a, FP64).
 *
 * Drop-in boundary for the hot path of the reference package `sdmefem`
 * (arXiv 2104.13466).  The reference has no FFI: its seams are duck-typed
 * Python calls.  Each entry point below names the reference
 * interface it replaces; the Python mirror `paper_2104_13466_b200` binds these
 * with ctypes (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - every function returns an sdme_status; details via sdme_last_error().
 *  - all device memory is owned by the context; host buffers are only read or
 *    written during the call (nothing retained).
 *  - one CUDA stream per context; calls are blocking unless named *_async;
 *    a context is not re-entrant.
 *  - vectors are opaque integer ids of device-resident lattice vectors
 *    (3 * Lx*Ly*Lz doubles, component-major, x fastest; Dirichlet points 0).
 *  - "free" vectors are host arrays in the reference free-DOF order
 *    (meshdof.py:345-370), length n_free.
 *  - deterministic: no floating-point atomics; fixed reduction trees; reruns
 *    are bit-identical.
 */
#ifndef SDME_H
#define SDME_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SDME_OK = 0,
  SDME_INVERSION = 1,      /* det F <= 0: ElementInversionError (femcore.py:36-42)     */
  SDME_INDEFINITE = 2,     /* p^T A p <= 0: PCGError (solver.py:151-155)               */
  SDME_MAXIT = 3,          /* PCG iteration cap: PCGError (solver.py:166-170)          */
  SDME_BAD_DIAGONAL = 4,   /* non-positive Jacobi diagonal: ValueError (solver.py:107) */
  SDME_BAD_ARGUMENT = 5,   /* invalid argument / unsupported (P, m)                    */
  SDME_CUDA_ERROR = 6      /* CUDA runtime error (message in sdme_last_error)          */
} sdme_status;

typedef struct sdme_ctx sdme_ctx;

/* Problem descriptor: FemProblem(mesh, element, dmap, mat, rule)
 * (femcore.py:276-295) restricted to axis-aligned gen_box_mesh meshes
 * (meshdof.py:146-193).  B, D are m x (P+1) row-major in the REFERENCE
 * function order [left, right, internal 2..P] (basis1d.py:83); the library
 * permutes them to lattice order. */
typedef struct {
  int P;                 /* polynomial order, 1..8                          */
  int m;                 /* Gauss points per direction (femcore.py:289-292) */
  int nx, ny, nz;        /* elements per axis                               */
  double hx, hy, hz;     /* element edge lengths                            */
  double origin[3];      /* mesh origin                                     */
  const double* B;       /* m x (P+1) values                                */
  const double* D;       /* m x (P+1) derivatives                           */
  const double* w;       /* m weights                                       */
  double mu, lambda_lame, rho0;      /* NeoHookean (material.py:32-46)      */
  int dirichlet_mask[3]; /* per component bits: 1 xmin 2 xmax 4 ymin 8 ymax 16 zmin 32 zmax */
  const int32_t* perm;   /* optional: 3*Lx*Ly*Lz lattice -> free index or -1; NULL = none */
  int64_t n_free;        /* reference free-DOF count (required with perm)   */
} sdme_desc;

/* General hexahedral mesh descriptor: FemProblem(mesh, element,
 * dmap, mat, rule) on any conforming hex mesh (meshdof.py:41-136) with
 * trilinear geometry (meshdof.py:269-296, femcore.py:73-81) and the
 * reference's oriented mode numbering (build_dofmap, meshdof.py:404-472).
 * Vectors of such a context are plain free-DOF arrays (length n_free, the
 * reference order); m must be P + 1 (the reference default rule).  The host
 * builds the tables (paper_2104_13466_b200/mesh.py); kernel point / function
 * order is [comp][z][y][x] over lattice-local 1D offsets (0 = left vertex,
 * P = right vertex, 1..P-1 = internal functions 2..P). */
typedef struct {
  int P;                 /* polynomial order, 2..8                                   */
  int m;                 /* Gauss points per direction: P + 1                        */
  int64_t n_elems;
  const double* B;       /* m x (P+1) values, reference function order               */
  const double* D;       /* m x (P+1) derivatives                                    */
  const double* w;       /* m weights                                                */
  double mu, lambda_lame, rho0;
  int64_t n_free;
  const int32_t* dof;    /* n_elems x 3 x (P+1)^3: 2*free + (sign < 0), or -1        */
  const int64_t* asm_ptr;   /* n_free + 1: CSR of element-vector slots per free DOF  */
  const int32_t* asm_slot;  /* asm_ptr[n_free]: 2*slot + (sign < 0), element order  */
  const double* geom;    /* n_elems x 10 x m^3: J^-1[d][c] (slot 3d + c), w det J    */
  /* optional locality layout (NULL = identity): the element rows of dof / geom
   * and the slots of asm_slot refer to STORAGE positions; elem_id[s] is the
   * reference element id stored at position s (inversion errors report it),
   * asm_rows[r] the free DOF of CSR row r.  Summation order per DOF is still
   * the reference's element order, so results do not depend on the layout. */
  const int32_t* elem_id;
  const int32_t* asm_rows;
} sdme_mesh_desc;

/* lifecycle ------------------------------------------------------------- */
int sdme_create(const sdme_desc* desc, sdme_ctx** out);
/* general mesh context: the same vector / operator / PCG entry points work on
 * it (sdme_contact*, sdme_strain_energy and lattice-order uploads excepted). */
int sdme_create_mesh(const sdme_mesh_desc* desc, sdme_ctx** out);
int sdme_destroy(sdme_ctx* ctx);
/* 3*Lx*Ly*Lz (lattice vector length) */
int sdme_lattice_size(const sdme_ctx* ctx, int64_t* n);
/* Last error: code, element id and quadrature point (inversion), message. */
int sdme_last_error(const sdme_ctx* ctx, int64_t* elem, int* qp, char* msg, size_t n);

/* vectors --------------------------------------------------------------- */
int sdme_vec_alloc(sdme_ctx* ctx, int* id);              /* zero-filled */
int sdme_vec_free(sdme_ctx* ctx, int id);
int sdme_vec_upload(sdme_ctx* ctx, int id, const double* host);     /* lattice order */
int sdme_vec_download(sdme_ctx* ctx, int id, double* host);
int sdme_vec_upload_free(sdme_ctx* ctx, int id, const double* host);    /* reference order */
int sdme_vec_download_free(sdme_ctx* ctx, int id, double* host);
int sdme_vec_fill(sdme_ctx* ctx, int id, double value);  /* Dirichlet points stay 0 */
int sdme_vec_copy(sdme_ctx* ctx, int dst, int src);
/* y = sum_t c[t] * x[t]  (nterms <= 6; y may alias an x) -- the axpys of
 * dynamics.py:219, 246-248 */
int sdme_vec_lincomb(sdme_ctx* ctx, int y, int nterms, const double* c, const int* x);
/* out = a * b elementwise (Jacobi apply, lumped-mass scaling) */
int sdme_vec_mul(sdme_ctx* ctx, int out, int a, int b);
/* deterministic dot product (solver.py:150, 159, 163 `@` / norm) */
int sdme_vec_dot(sdme_ctx* ctx, int a, int b, double* out);
/* dst = 1/src on free points, 0 on Dirichlet points; SDME_BAD_DIAGONAL if a
 * free entry is <= 0 (lumped-mass inverse, Jacobi preconditioner) */
int sdme_vec_reciprocal(sdme_ctx* ctx, int dst, int src);

/* operators (problem-level, femcore.py:346-372) ------------------------- */
/* r = f_int(u)   -- FemProblem.internal_force (femcore.py:346-349)            */
int sdme_fint(sdme_ctx* ctx, int u, int r);
/* y = c_k K_T(u) p + c_m M p -- element_tangent(...)@p + mass (femcore.py:130-156,
 * consumer solver.py:149 `a @ p`, Newmark eff = kt + b1 m, dynamics.py:236-237) */
int sdme_apply(sdme_ctx* ctx, int u, int p, int y, double c_k, double c_m);
/* n operator applications with host buffers (free order; page-locked for full
 * overlap): y[k] = (c_k K(u[k]) + c_m M) p[k].  Pipelined: the H2D copies of
 * pair k+1 and the D2H copy of result k-1 run on two copy streams while pair k
 * is permuted and applied (box contexts with a permutation).  Replaces a loop
 * of element_tangent(...) @ p_e assemblies (femcore.py:130-146) over a batch. */
int sdme_apply_batch(sdme_ctx* ctx, int n, const double* const* u, const double* const* p, double* const* y,
                     double c_k, double c_m);
/* y = M a -- mass_full @ a_trial (dynamics.py:198) */
int sdme_mass(sdme_ctx* ctx, int a, int y);
/* total strain energy sum_e sum_q w det J psi(F) (femcore.py:374-378, material.py:80);
 * fixed-order reduction */
int sdme_strain_energy(sdme_ctx* ctx, int u, double* out);

/* one Newton iterate of newmark_run (dynamics.py:213-226) with one host
 * synchronisation: [uk += du if du >= 0]; atr = b1 (uk - u) - b2 v - b3 a;
 * psi = s_load * load - f_int(uk) - M atr (load may be -1); *norm = ||psi||;
 * tmp is scratch.  SDME_INVERSION as sdme_fint. */
int sdme_newmark_residual(sdme_ctx* ctx, int uk, int du, int u, int v, int a, int load, double s_load, double b1,
                          double b2, double b3, int atr, int tmp, int psi, double* norm);

/* d = diag(c_k K_T(u) + c_m M) on free points -- a.diagonal() (solver.py:106) */
int sdme_diag(sdme_ctx* ctx, int u, double c_k, double c_m, int d);

/* Jacobi-PCG on A = K_T(u_lin) + c_m M (solver.py:129-170 with
 * precond "diagonal" (1) or "none" (0)); x0 = 0.  On SDME_INDEFINITE /
 * SDME_MAXIT, *iters and *relres carry the PCGError stats. */
int sdme_pcg(sdme_ctx* ctx, int u_lin, double c_k, double c_m, int b, int x, double tol,
             int maxit, int precond, int* iters, double* relres);

/* explicit central difference with lumped mass (D6, dynamics.py:152-164):
 * psi = s_load*load - f_int(u) + f_c ; u_next = 2u - u_prev + dt^2 psi / m_L ;
 * v = (u_next - u_prev)/(2 dt).  load / fc may be -1 (absent).  inv_ml is the
 * reciprocal lumped mass vector (0 on Dirichlet points). */
int sdme_explicit_step(sdme_ctx* ctx, int u, int u_prev, int v, int load, double s_load,
                       int fc, int inv_ml, double dt, int scratch);
/* n such steps back to back on the device (no host round trip per step): the
 * contact force (fc >= 0) uses the parameters of the last sdme_contact call,
 * the load scale of step k is s_load[k]; the inversion flag is checked once
 * at the end (smallest element / point over the n steps). */
int sdme_explicit_steps(sdme_ctx* ctx, int n, int u, int u_prev, int v, int load, const double* s_load, int fc,
                        int inv_ml, double dt, int scratch);

/* penalty contact against a rigid plane on a box side (contact.py:87-128):
 * fc = sum_q warea t_N N_f n, gaps (optional, host) = gap per face point in the
 * reference face/point order; side = 0..5 (xmin..zmax); qf = face rule points
 * (default P+1) with Bf (qf x (P+1), reference function order), points xf and
 * weights wf of the 1D face rule; stats[0] = penetration max(-g, 0), stats[1] = min active
 * pressure (0 if none), stats[2] = active point count. */
int sdme_contact(sdme_ctx* ctx, int u, int side, int qf, const double* Bf, const double* xf,
                 const double* wf, const double* point,
                 const double* normal, double eps, int fc, double* gaps_host,
                 double* stats);
/* number of face points of a side for the given qf */
int sdme_contact_points(const sdme_ctx* ctx, int side, int qf, int64_t* n);

/* implicit contact (contact.py:120-140 stiffness, dynamics.py:268-284): with
 * the active set (g < 0) of the last sdme_contact call,
 * y += K_c p,  K_c = eps sum_{q active} warea N_f N_g n n^T  (matrix-free) */
int sdme_contact_apply(sdme_ctx* ctx, int p, int y);
/* d += diag(K_c) */
int sdme_contact_diag(sdme_ctx* ctx, int d);
/* on != 0: sdme_pcg solves with A + K_c (and its diagonal in the Jacobi
 * preconditioner), the operator of newmark_run with contact (dynamics.py:241) */
int sdme_pcg_contact(sdme_ctx* ctx, int on);

/* assembled / Schur-condensed solve (the reference's default solver,
 * SolverConfig(precond="sgs", condense=True), dynamics.py:38-43, 111-127;
 * condense_elements / CondensedSystem / LinearSolver, solver.py:179-322).
 * Box-mesh contexts.  The host describes every element's local DOFs in the
 * reference local order (function-major (p,q,r) r fastest, component fastest,
 * tensorelem.py:97-129): its lattice address (-1 when Dirichlet) and its role,
 * the global boundary index 0..nb-1 (the reference's free index, boundary DOFs
 * first) or -2 for an element-interior DOF (condensed out) or -1
 * (constrained).  With no -2 roles (condense=False) the CSR is the full free
 * operator.  Element matrices use the tabulated physical gradients G (nq x nf
 * x 3), values N (nq x nf) and w det J (nq) of the problem's rule. */
typedef struct sdme_schur sdme_schur;
typedef struct {
  int64_t n_elems;
  int nd;                 /* 3 (P+1)^3 local DOFs                                  */
  int nq;                 /* quadrature points per element                         */
  int64_t nb;             /* size of the (condensed) system                        */
  const int64_t* addr;    /* n_elems x nd lattice addresses, -1 constrained        */
  const int32_t* role;    /* n_elems x nd: boundary index, -1 constrained, -2 interior */
  const int64_t* addr_b;  /* nb lattice addresses of the system's DOFs             */
  const double* G;        /* nq x nf x 3 physical gradients (reference orders)    */
  const double* N;        /* nq x nf values                                        */
  const double* wdet;     /* nq weights x det J                                    */
  double mu, lambda_lame, rho0;
} sdme_schur_desc;
int sdme_schur_create(sdme_ctx* ctx, const sdme_schur_desc* desc, sdme_schur** out);
int sdme_schur_destroy(sdme_schur* s);
/* system size, CSR nonzeros, level counts of the forward / backward SGS sweeps */
int sdme_schur_info(const sdme_schur* s, int64_t* nb, int64_t* nnz, int* fwd_levels, int* bwd_levels);
/* element matrices of c_k K_T(u) + c_m M (femcore.py:130-156; u ignored when
 * c_k = 0), per-element condensation (Cholesky of K_ii; SDME_BAD_ARGUMENT
 * "element interior block is not SPD" as solver.py:284-285 raises ValueError),
 * deterministic CSR assembly in element order */
int sdme_schur_factor(sdme_schur* s, int u, double c_k, double c_m);
/* x = A^-1 b: reduce_rhs, PCG on the (condensed) CSR with precond 0 none,
 * 1 diagonal, 2 symmetric Gauss-Seidel (solver.py:129-170, same order of
 * checks and errors as sdme_pcg), interior recovery; b, x lattice vectors */
int sdme_schur_solve(sdme_schur* s, int b, int x, int precond, double tol, int maxit, int* iters,
                     double* relres);
/* host copies of the assembled CSR (rowptr nb+1, cols nnz, vals nnz) and of
 * element 0's matrix (nd x nd); any pointer may be NULL */
int sdme_schur_matrix(const sdme_schur* s, int64_t* rowptr, int32_t* cols, double* vals,
                      double* element_matrix0);
/* row-major dense lattice -> device address of a lattice point of component c */
int sdme_lattice_address(const sdme_ctx* ctx, int c, int x, int y, int z, int64_t* addr);

/* page-locked host buffers (fast H2D/D2H for the free-order vector calls) */
int sdme_host_alloc(size_t bytes, void** ptr);
int sdme_host_free(void* ptr);

/* timing (CUDA events on the context stream) ----------------------------- */
/* op: 0 = apply (K(u) p + c_m M p from u), 1 = fint, 2 = mass, 3 = diag,
 * 4 = quadrature-data setup at u (K = F^-T, ln J stored per point, as sdme_pcg
 * does once per solve), 5 = apply from the stored data (the PCG operator; needs
 * a prior op 4); returns mean milliseconds per call over `reps` calls. */
int sdme_time_op(sdme_ctx* ctx, int op, int u, int p, int y, double c_m, int reps, double* ms);
int sdme_sync(sdme_ctx* ctx);
/* kernel launches issued by this context since creation (evidence for bench) */
int sdme_launch_count(const sdme_ctx* ctx, int64_t* n);

#ifdef __cplusplus
}
#endif
#endif /* SDME_H */
