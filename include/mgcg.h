/*
 * mgcg.h -- C ABI of the B200-native (sm_100a, fp64) fine-grid solve path of
 * Ferrari & Sigmund, "Towards solving large-scale topology optimization problems
 * with buckling constraints at the cost of linear analyses" (arXiv 1909.13585).
 *
 * What the library computes (PAPER.md line numbers, section / equation):
 *   - K(x) u = f for a batch of right-hand sides: the linear analysis (LA) of
 *     Alg. 1 l.2, the adjoint systems K z_i = phi_i' (grad_u G) phi_i
 *     of Eq. 5 (:133-136) and the fine-scale BVP K Phi = G Psi of Eq. 6 / Alg. 2
 *     l.15 (:161-165, :732).  Solver: conjugate gradients preconditioned by a
 *     geometric multigrid built on the nested discretisations {Omega_j}
 *     (Appendix A; block/multi-RHS use :760-761).
 *   - K_e = E_kappa(x_e) K_e0 and G_e = E_sigma(x_e) G_e0[u_e] (Eq. 2
 *     :101-108); K_e0 is the standard bilinear Q4 (plane stress, thickness 1) /
 *     trilinear H8 unit-element stiffness (SURVEY.md 8(c) reading r1, r2).
 *   - Coarse operators by Galerkin projection K^l = I^1_l K I^l_1 (PAPER.md:155,
 *     Alg. 2 l.5 :705) with bilinear/trilinear interpolation I^j_{j+1} (:146).
 *   - y = G(u) phi, the stress-stiffness product used as RHS in Eq. 6 (:163) and
 *     in the residual Eq. 7 (:181); stress at the element centroid (reading r15).
 *
 * Conventions (all entry points):
 *   - Array arguments are device pointers unless stated otherwise; mgcg_solve and
 *     stress_stiffness_apply also accept host pointers (detected with
 *     cudaPointerGetAttributes) and then copy in/out on the handle's stream.
 *   - Vectors are RHS-major, shape (nrhs, n), fp64; DOF index = d*node + comp;
 *     nodes in C order over (N0+1, N1+1[, N2+1]), axis 0 slowest; comp c is the
 *     displacement along axis c.  Element arrays (E_e, Es_e) in C order over
 *     (N0, N1[, N2]).
 *   - Dirichlet: `fixed[dof] != 0` marks a fixed DOF.  K's fixed rows/columns are
 *     identity, G's are zero; solutions and G-products are 0 at fixed DOFs and
 *     right-hand sides are masked there.
 *   - Ownership: mg_setup copies E_e and fixed; all other arrays are borrowed for
 *     the duration of the call.  The handle owns its device workspace.
 *   - Errors: every call returns mg_status; argument errors have no side
 *     effects (mg_update_modulus validates E before touching the handle);
 *     mg_last_error() gives a one-line description of the last failure on the
 *     calling thread.  On MG_ERR_BREAKDOWN x and the report describe the last
 *     iterate (its true residual is evaluated).
 *   - Handles and threads: several handles (any dim / nu / element) may be alive
 *     and used from several threads.  Calls that launch work are serialised by a
 *     process-wide lock.  The element constants (K0, K^, H, D0) sit in constant
 *     memory shared by all handles: a call on a handle whose (dim, element, nu)
 *     differs from the last one used first waits for all device work
 *     (cudaDeviceSynchronize) and reloads them, so interleaving handles of
 *     different element types is correct but synchronising.
 */
#ifndef MGCG_H
#define MGCG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MG_MAX_RHS 64
#define MG_MAX_LEVELS 12

typedef enum {
    MG_OK = 0,
    MG_ERR_ARG = 1,          /* NULL pointer, bad dim/levels/nrhs/tol            */
    MG_ERR_NONDIVISIBLE = 2, /* N_i not divisible by 2^(levels-1)   */
    MG_ERR_DIM = 3,          /* size mismatch / too large                         */
    MG_ERR_MODULUS = 4,      /* E_e <= 0 or not finite                            */
    MG_ERR_BREAKDOWN = 5,    /* p.Kp <= 0 in CG: operator not SPD                 */
    MG_ERR_MAXITER = 6,      /* max_iter reached; x holds the last iterate        */
    MG_ERR_OOM = 7,
    MG_ERR_CUDA = 8,
    MG_ERR_NCCL = 9,
    MG_ERR_SINGULAR = 10     /* coarsest-level factorisation hit a non-positive pivot */
} mg_status;

/* Element type: MG_ELEM_STD = standard bilinear Q4 / trilinear H8 (SURVEY.md 8(c) reading r1);
 * MG_ELEM_WILSON = incompatible-mode element of the paper:
 * bubble modes 1 - xi_k^2 per component condensed statically on the unit element.  Both use the
 * centroid stress for G (the bubble gradients vanish there). */
#define MG_ELEM_STD 0
#define MG_ELEM_WILSON 1

/* Structured grid: dim = 2 (Q4) or 3 (H8); nel[k] element count along axis k
 * (nel[2] ignored in 2D); nu = Poisson ratio (0.3); element type. Unit elements. */
typedef struct {
    int dim;
    int nel[3];
    double nu;
    int element;
} mg_grid;

/* Multigrid / CG options; pass NULL for defaults {0.6, 1, 1, 1000}.
 * omega: damped-Jacobi factor; nu_pre / nu_post: sweeps per level (symmetric
 * V-cycle requires nu_pre == nu_post >= 1); max_iter: CG iteration cap. */
typedef struct {
    double omega;
    int nu_pre;
    int nu_post;
    int max_iter;
} mg_opts;

/* Per-solve report (host struct). iters[k]: CG iterations of RHS k; relres[k]:
 * recursive ||r_k||/||b_k||; true_relres[k]: ||b_k - K x_k|| / ||b_k|| computed at
 * exit; converged[k] = 1 if true_relres[k] <= tol. Times in milliseconds. */
typedef struct {
    int nrhs;
    int iters[MG_MAX_RHS];
    double relres[MG_MAX_RHS];
    double true_relres[MG_MAX_RHS];
    int converged[MG_MAX_RHS];
    int max_iters;
    int restarts;
    int graph_launches;
    long long kernel_launches;
    double solve_ms;
} mg_report;

typedef struct mg_ctx* mg_handle;

/* Build the hierarchy for one design (Alg. 2 l.1-2, l.5):
 *   grid    element counts, nu.  Requires nel[k] % 2^(levels-1) == 0.
 *   E_e     device, nelem fp64 moduli E_kappa(x_e) > 0 (Eq. 2), copied.
 *   fixed   device, ndof uint8, nonzero = Dirichlet DOF, copied.
 *   levels  1..MG_MAX_LEVELS, counting the finest level (reading r10).
 *   opts    NULL or options.
 *   stream  cudaStream_t (as void*) on which all work of this handle runs;
 *           NULL = the legacy default stream.
 *   out     receives the handle.
 * Work: fine diagonal, Galerkin coarse operators on every level, coarsest
 * dense SPD inverse; all on the device.  Synchronises the stream. */
mg_status mg_setup(const mg_grid* grid, const double* E_e, const uint8_t* fixed,
                   int levels, const mg_opts* opts, void* stream, mg_handle* out);

/* Slab decomposition along axis 0 (BASELINE.json:5 "partitioned into slabs
 * across 1/2/4/8 GPUs ... NCCL halo exchange ... allreduce for CG dot products").
 * The global grid is cut at coarsest-level element boundaries into S = nranks * nslab slabs
 * (mg_partition gives slab k's owned element layers [e_begin, e_end)); rank r (one process
 * per GPU) holds slabs [r*nslab, (r+1)*nslab).  nslab > 1 keeps several slabs in one handle
 * (exchanges by device copies; used to test the decomposition on one GPU).
 *   rank, nranks  this process and the job size (nranks > 1 needs nccl_id)
 *   nslab         slabs held by this rank (>= 1)
 *   nccl_id       NCCL_UNIQUE_ID_BYTES (128) bytes from mg_nccl_unique_id on rank 0,
 *                 broadcast by the caller; NULL when nranks == 1.
 * With a dist, every array argument of every call covers THIS RANK's owned part only:
 * element arrays its element layers [e_begin, e_end) (mg_local_info), vectors and `fixed`
 * its node planes [e_begin, e_end) plus plane N0 on the last rank, same C order. */
typedef struct {
    int rank;
    int nranks;
    int nslab;
    const void* nccl_id;
} mg_dist;

/* mg_setup with a decomposition (dist NULL = one slab = mg_setup).  Requires levels >= 2
 * and S <= N0 / 2^(levels-1).  Collective over the nranks processes. */
mg_status mg_setup_dist(const mg_grid* grid, const double* E_e, const uint8_t* fixed, int levels,
                        const mg_opts* opts, const mg_dist* dist, void* stream, mg_handle* out);
/* Host-only: owned element layers [e_begin, e_end) along axis 0 of slab `part` of `nparts`
 * (coarsest-level layers split as evenly as possible). No device work. */
mg_status mg_partition(const mg_grid* grid, int levels, int nparts, int part, int* e_begin, int* e_end);
/* Host: 128-byte NCCL unique id for mg_dist.nccl_id (loads libnccl.so.2 with dlopen). */
mg_status mg_nccl_unique_id(void* out128);
/* This rank's owned DOF / element counts and its element-layer range. */
mg_status mg_local_info(mg_handle h, long long* ndof_local, long long* nelem_local, int* e_begin, int* e_end);

/* Same grid and BCs, new design: recompute all level operators from E_e.
 * E_e is validated (positive, finite: else MG_ERR_MODULUS, handle unchanged) and copied before the
 * call returns; the call returns once the new operators are enqueued on the handle's stream.  A
 * non-positive pivot of the coarsest SPD inverse (MG_ERR_SINGULAR) is reported by the next call on
 * the handle, which first waits for the operators; mgcg_solve uploads host right-hand sides before
 * that wait, so the upload overlaps the setup. */
mg_status mg_update_modulus(mg_handle h, const double* E_e);

/* Solve K x_k = rhs_k, k < nrhs, by multigrid-preconditioned CG
 * from a zero initial guess, each RHS stopping when ||r_k|| <= tol ||b_k||
 * (reading r12; confirmed by a true residual at exit).
 *   rhs  (nrhs, ndof) fp64, device or host; masked to 0 at fixed DOFs.
 *   x    (nrhs, ndof) fp64 output, device or host.
 *   rep  NULL or a host report.
 * Returns MG_ERR_MAXITER (x = last iterate) or MG_ERR_BREAKDOWN on failure.
 * Synchronous with respect to the handle's stream. 1 <= nrhs <= MG_MAX_RHS. */
mg_status mgcg_solve(mg_handle h, const double* rhs, int nrhs, double tol, double* x, mg_report* rep);

/* NEXT-3: the paper's block variant mgBPCG (Alg. 2 l.15 :732):
 * O'Leary block CG over the nrhs columns with the same V(1,1) preconditioner, sharing one Krylov
 * space; the R x R Gram systems are solved by a pivoted Cholesky whose dropped pivots deflate
 * dependent or converged directions.  Same arguments, report and stopping rule
 * as mgcg_solve (per column ||r_k|| <= tol ||b_k||, true residual at exit); report.iters[k] counts
 * the block iterations until column k converged.  Single slab this round. */
mg_status mgcg_block_solve(mg_handle h, const double* rhs, int nrhs, double tol, double* x, mg_report* rep);

/* NEXT-2: multilevel approximation of the q lowest buckling modes, the four
 * steps of PAPER.md:146-175 (Sec. 2.1):
 *   1. coarse eigenproblem (K^l + lambda^l G^l) psi^l = 0 (Eq. 6) with K^l, G^l the Galerkin
 *      projections on the coarsest level (G^l by the same element agglomeration as K^l);
 *      solved on the device by subspace iteration with the coarsest K^-1 and a host
 *      Rayleigh-Ritz on the (q+8)-dimensional subspace;
 *   2. Psi = I^1_2 ... I^{l-1}_l Psi^l (prolongation to the fine level);
 *   3. K Phi~ = G Psi (Eq. 7) by block PCG (mgcg_block_solve, mgBPCG) to tol;
 *   4. lambda~_i = -phi~_i^T K phi~_i / phi~_i^T G phi~_i (Eq. 8); the returned modes are
 *      K-normalised, phi~_i^T K phi~_i = 1, and the residual of the first pair,
 *      y = (K + lambda~_1 G) phi~_1 (Eq. 7), is formed on request.
 *   Es_e (nelem), u (ndof): device; Phi (q, ndof) device output; lam_tilde (q) host output;
 *   lam_coarse (q) host output or NULL; y1 (ndof) device output or NULL; yres (2) host output or
 *   NULL: ||y||_2 and ||y||_2 / ||K phi~_1||_2.  1 <= q <= 32, levels >= 2, single slab.
 *   Synchronous. */
mg_status mg_multilevel_modes(mg_handle h, const double* Es_e, const double* u, int q, double tol, double* Phi,
                              double* lam_tilde, double* lam_coarse, double* y1, double* yres);

/* y_k = G(u) phi_k for k < nphi (PAPER.md:99 G_e = E_sigma G_e0[u_e]; Eq. 6 :163):
 *   Es_e  device, nelem fp64 stress moduli E_sigma(x_e) = x_e^p E_1 (Eq. 2 :106).
 *   u     device, ndof fp64 displacement (taken as given, incl. fixed DOFs).
 *   phi   (nphi, ndof) fp64; y (nphi, ndof) fp64 output; fixed rows/cols zero.
 * Stress sigma_e = Es_e D0 B(centroid) u_e; G_e = (sum_ij sigma_ij H_ij) kron I_d.
 * Device or host pointers. Asynchronous for device pointers. */
mg_status stress_stiffness_apply(mg_handle h, const double* Es_e, const double* u,
                                 const double* phi, int nphi, double* y);

/* NEXT-1: adjoint right-hand sides of Eq. 5,
 *   b_i = phi_i^T (grad_u G) phi_i,  i < nphi,
 * i.e. b_i[k] = d(phi_i^T G(u) phi_i)/du_k; G is linear in u so b does not depend on u.
 *   Es_e  device, nelem fp64 stress moduli (Eq. 2 :106);  phi (nphi, ndof) device;
 *   b     (nphi, ndof) device output, zero on fixed DOFs (ready for mgcg_solve).
 * Any decomposition (arrays cover the calling rank's owned part, as for mgcg_solve).
 * Asynchronous (single slab) / synchronous (slabs). */
mg_status mg_adjoint_rhs(mg_handle h, const double* Es_e, const double* phi, int nphi, double* b);
/* NEXT-1: element sensitivities of simple buckling load factors, Eq. 4:
 *   out[i][e] = dEk_e (phi_ie^T K_e0 phi_ie - lambda_i z_ie^T K_e0 u_e)
 *             + lambda_i dEs_e phi_ie^T G_e0[u_e] phi_ie
 * with dEk = dE_kappa/dx, dEs = dE_sigma/dx (Eq. 2, caller-supplied), u the state, phi_i the
 * modes, z_i the adjoint solutions (K z_i = mg_adjoint_rhs(phi_i)).  phi, z (and u in the K
 * term) are taken on the free DOFs.  Reading: this is d lambda_i / d x_e for modes
 * normalised by phi^T (-G) phi = 1; for phi^T K phi = 1 multiply by lambda_i.
 *   dEk, dEs (nelem), u (ndof), phi, z (nphi, ndof): device;  lambda: nphi values, host or
 *   device;  out (nphi, nelem) device.  1 <= nphi <= MG_MAX_RHS.  Any decomposition (owned
 *   elements / nodes of the calling rank).  Synchronous. */
mg_status mg_eigen_sensitivity(mg_handle h, const double* dEk, const double* dEs, const double* u, const double* phi,
                               const double* z, const double* lambda, int nphi, double* out);

/* Diagnostics (used by the parity tests; all device pointers, asynchronous):
 * y = A_level x for nrhs vectors (level 0 = fine matrix-free K; level >= 1 =
 * Galerkin operator incl. identity rows at fixed DOFs). */
mg_status mg_matvec(mg_handle h, int level, const double* x, int nrhs, double* y);
/* z = B r : one symmetric V-cycle of the preconditioner on nrhs vectors. */
mg_status mg_vcycle(mg_handle h, const double* r, int nrhs, double* z);
/* coarse = P^T fine (restriction from `level` to level+1), masked (reading r11). */
mg_status mg_restrict(mg_handle h, int level, const double* fine, int nrhs, double* coarse);
/* fine = P coarse (prolongation from level+1 to `level`), masked. */
mg_status mg_prolong(mg_handle h, int level, const double* coarse, int nrhs, double* fine);
/* Element counts and DOF count of a level; nlevels if level < 0. */
mg_status mg_level_info(mg_handle h, int level, int* nel3, long long* ndof, int* nlevels);
/* diag(A_level) (ndof doubles, device). */
mg_status mg_get_diagonal(mg_handle h, int level, double* d);
/* Dense inverse of the coarsest operator (ndof_L x ndof_L, row-major, device). */
mg_status mg_get_coarse_inverse(mg_handle h, double* Ainv);
/* Time the fine-level kernels of one CG iteration standalone (same kernels and launch
 * configuration as inside the solve graph) on nrhs internal vectors, reps launches each,
 * with CUDA events on the handle's stream.  ms[0..3] = average ms per launch of:
 * CG direction + matvec (a2/a7), residual + restriction block (a3/a4), prolongation +
 * post-smoothing block (a3/a4), plain matvec K x (a2).  Synchronous. */
mg_status mg_profile_kernels(mg_handle h, int nrhs, int reps, double* ms);
/* Number of CUDA kernels this handle has launched (graph nodes counted once per launch). */
long long mg_kernel_launches(mg_handle h);

mg_status mg_destroy(mg_handle h);
const char* mg_strerror(mg_status s);
const char* mg_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* MGCG_H */
