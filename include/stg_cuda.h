/*
 * stg_cuda.h -- C ABI of the B200-native space-time DG-SEM slab operator.
 *
 * Drop-in boundary for the hot path of the reference `stdgsem` library
 * (/root/reference/proj/include/stdgsem).  Every entry point names the
 * reference interface it replaces.  Plain pointers and sizes only; no C++,
 * CUDA or torch types cross this boundary.  Status codes instead of
 * exceptions (mapped back to the reference's exception types by the C++ host
 * wrapper paper_2201_05800_b200/csrc/stdgsem_gpu.hpp and the Python mirror
 * paper_2201_05800_b200/api.py):
 *
 *   STG_OK                 0
 *   STG_ERR_INVALID        1  std::invalid_argument   (stdg.hpp:59-61, mesh.hpp:39)
 *   STG_ERR_RUNTIME        2  std::runtime_error      (newton.hpp:74-76)
 *   STG_ERR_NONCONVERGENCE 3  NonconvergenceError     (newton.hpp:40-48, 116-120)
 *   STG_ERR_CUDA           4  CUDA runtime failure (no CPU fallback exists)
 *   STG_ERR_ADMISSIBILITY  5  AdmissibilityError     (models.hpp:15-20, stdg.hpp:41-50)
 *
 * Layout of every vector (unchanged from the reference, stdg.hpp:18-20,
 * mesh.hpp:22-25, mesh.hpp:70-81): temporal-node (stage) blocks outermost,
 * then cell index (x fastest: cell = (cz*ny + cy)*nx + cx), then node index
 * within the cell (x fastest: node = (iz*n + iy)*n + ix), component innermost
 * (r = 4 conservative components for Euler, r = 1 otherwise).  A spatial
 * vector has n_sdof = cells * n^d * r entries, a slab/stage vector
 * n_tau * n_sdof.
 *
 * Memory: unless a function name ends in `_host`, every double* is a DEVICE
 * pointer owned by the caller.  `_host` variants take host pointers and do
 * the host<->device copies inside the call (the reference-facing path that
 * the bench times end to end).
 *
 * Threading: one handle per CUDA stream; a handle is not thread-safe;
 * distinct handles may be used concurrently.
 */
#ifndef STG_CUDA_H
#define STG_CUDA_H

#ifdef __cplusplus
extern "C" {
#endif

#define STG_ABI_VERSION 3

#define STG_OK 0
#define STG_ERR_INVALID 1
#define STG_ERR_RUNTIME 2
#define STG_ERR_NONCONVERGENCE 3
#define STG_ERR_CUDA 4
#define STG_ERR_ADMISSIBILITY 5

/* models: advection_model (models.hpp:40-66) with constant velocity;
 * Burgers (EXTENSION, not in the reference; d = 1 only);
 * advdiff_model (models.hpp:68-76): advection with a constant or rotating
 * (models.hpp:79-85) velocity field plus interior-penalty diffusion eps
 * (spatial.hpp:27-52, 209-261), d in {1, 2};
 * euler_model(gamma) (models.hpp:118-159): 2-D compressible Euler, r = 4. */
#define STG_MODEL_ADVECTION 0
#define STG_MODEL_BURGERS 1
#define STG_MODEL_ADVDIFF 2
#define STG_MODEL_EULER 3

/* velocity fields of STG_MODEL_ADVDIFF */
#define STG_FIELD_CONSTANT 0  /* b = velocity[] */
#define STG_FIELD_ROTATING 1  /* rotating_field(): b = (-4(y-1/2), 4(x-1/2)) */

/* JacobianForm (lodg.hpp:20) */
#define STG_FORM_A 0
#define STG_FORM_A_INV 1

/* LinearMethod (newton.hpp:28).  Only GMRES runs on the device; AUTO maps to
 * GMRES (the direct branches are CPU-only in the reference and infeasible at
 * the configured sizes). */
#define STG_LINEAR_AUTO 0
#define STG_LINEAR_GMRES 3

/* Right preconditioner of the device GMRES.  The reference's Eigen::GMRES
 * defaults to a diagonal preconditioner (newton.hpp:69); point Jacobi stalls
 * on these Jacobians, so the block versions are provided:
 *   TBLOCK  temporal-block Jacobi (n_tau x n_tau per spatial node, advection)
 *   EBLOCK  element-block Jacobi (exact inverse of the element-local block:
 *           d = 1 dense; d = 2 advection with n_tau * (N+1)^2 <= 128 one
 *           shared dense block; d = 3 advection, degree 3, n_tau = 4,
 *           cells % 8 == 0 by fast diagonalisation; advdiff (linear general
 *           model) with n_tau * (N+1)^d <= 32 by coloured probing)
 *   AUTO    EBLOCK where supported, else TBLOCK (advection) / none. */
#define STG_PRECOND_NONE 0
#define STG_PRECOND_TBLOCK 1
#define STG_PRECOND_EBLOCK 2
#define STG_PRECOND_AUTO 3
/* ABI v3: Eigen's default DiagonalPreconditioner -- P = diag(J), with 1 in
 * place of a zero diagonal entry (Eigen's documented rule).  The slab
 * Jacobian's diagonal is exactly zero at interior nodes
 * (test_experiments.cpp:109-111), so this is mostly the identity there;
 * provided so the device solve can run the reference's own algorithm.
 * Advection only. */
#define STG_PRECOND_JACOBI 4
/* Upwind block sweep (d = 1 Burgers, n_tau = 4, degree 1 or 3; the AUTO
 * choice there): block Gauss-Seidel in +x, the element blocks plus each
 * element's inflow coupling to its left neighbour, solved exactly around the
 * periodic ring by a parallel scan (the paper's GMRES + SOR, PAPER.md
 * 1319-1321, as one exact sweep).  Reduces to element-block Jacobi where the
 * flow runs in -x. */
#define STG_PRECOND_SWEEP 5
/* Polynomial (Neumann) preconditioner over the element-block Jacobi P0 = the
 * EBLOCK (or, d = 1 Burgers, SWEEP) choice:
 *   P^-1 = sum_{i=0..m} (I - P0^-1 J)^i P0^-1,  m = 7 (env STG_POLY_TERMS)
 * applied as y_0 = z = P0^-1 r, y_{i+1} = z + y_i - P0^-1 J y_i: m Jacobian
 * actions and m + 1 block applies per GMRES step, in exchange for fewer
 * GMRES steps (c4: 7 -> 1) and their quadratically growing Gram-Schmidt
 * passes.  Any model whose EBLOCK exists. */
#define STG_PRECOND_POLY 6

/* Kernel selection (for tests / benchmarking; AUTO picks the fastest valid). */
#define STG_KERNEL_AUTO 0
#define STG_KERNEL_GENERIC 1
#define STG_KERNEL_FAST 2

typedef struct stg_handle stg_handle;

/* Problem description: uniform_mesh (mesh.hpp:37-55, EXTENDED to d = 3),
 * dg_space (mesh.hpp:93-110) with degree p = `degree`, the temporal SBP
 * operators sbp_operators(n_tau) (operators.hpp:33-44) and the model. */
typedef struct stg_desc {
  int dim;          /* 1, 2 or 3 */
  int degree;       /* spatial polynomial degree N >= 1 (n = N+1 LGL nodes) */
  int n_tau;        /* temporal LGL nodes = stages (2..6) */
  int model;        /* STG_MODEL_* */
  int cells[3];     /* cells per axis (unused axes ignored) */
  double lower[3];  /* domain lower corner */
  double upper[3];  /* domain upper corner */
  double velocity[3]; /* advection velocity b (constant fields) */
  /* ABI v2 (general models; zero-initialise for the defaults): */
  int velocity_field; /* STG_FIELD_* (STG_MODEL_ADVDIFF) */
  double eps;         /* diffusion coefficient >= 0 (STG_MODEL_ADVDIFF) */
  double eta;         /* interior-penalty parameter; <= 0: 10 p^2 (spatial.hpp:366) */
  double gamma;       /* ratio of specific heats; <= 0: 1.4 (STG_MODEL_EULER) */
} stg_desc;

/* NewtonConfig (newton.hpp:30-38) plus the finite-difference step for
 * nonlinear Jacobian actions (fd_eps <= 0: exact linearisation). */
typedef struct stg_newton_config {
  double abs_tol;     /* default 1e-12 */
  double rel_tol;     /* default 1e-12 */
  int max_iter;       /* default 50 */
  int linear;         /* STG_LINEAR_* */
  int gmres_restart;  /* default 30 */
  double gmres_tol;   /* default 1e-12, ||r||_2 <= tol ||b||_2 */
  int gmres_max_it;   /* default 1000 */
  double fd_eps;      /* FD Jacobian-vector step; <= 0: exact (Burgers) or
                         1e-5 (Euler, which has no exact linearisation here) */
  int precond;        /* STG_PRECOND_*; default AUTO */
} stg_newton_config;

#define STG_MAX_HISTORY 64
/* NewtonResult (newton.hpp:93-98) plus Krylov statistics.
 * On STG_ERR_NONCONVERGENCE (NonconvergenceError, newton.hpp:40-48) the
 * record describes the failed solve: the Newton / GMRES iterations done, the
 * last residual norm and the residual history; the solver's last iterate is
 * left in the caller's U (the step's U, or the failing step's slot of
 * U_slabs / U_stages in the integrators -- `failed_step` names it). */
typedef struct stg_solve_info {
  int newton_iterations;
  int linear_iterations;   /* total GMRES iterations over all Newton steps */
  double final_residual;   /* ||res||_inf */
  int n_history;
  double residual_history[STG_MAX_HISTORY];
  int failed_step;         /* ABI v3: integrators, index of the step that did not
                              converge; -1 otherwise */
} stg_solve_info;

/* Defaults of NewtonConfig (newton.hpp:30-38). */
void stg_newton_config_default(stg_newton_config* cfg);

/* Last error message of a handle (NULL: the thread's last create error). */
const char* stg_last_error(const stg_handle* h);

/* assemble_semidiscrete (spatial.hpp:352-385) + the temporal operators:
 * builds the constants (LGL D and w from the host restatement of
 * quadrature.hpp:66-144, mass, Lobatto IIIC tableau operators.hpp:76-112) and
 * device workspace.  Fails with STG_ERR_INVALID on bad descriptors and
 * STG_ERR_CUDA when no device is usable. */
int stg_create(const stg_desc* desc, stg_handle** out);
void stg_destroy(stg_handle* h);

/* Bind a cudaStream_t (NULL = default stream). */
int stg_set_stream(stg_handle* h, void* cuda_stream);
/* Force a kernel family (STG_KERNEL_*), e.g. to test both paths. */
int stg_set_kernel(stg_handle* h, int kernel);
/* Number of spatial (n_sdof) and slab (n_dof = n_tau * n_sdof) unknowns. */
int stg_sizes(const stg_handle* h, long long* n_sdof, long long* n_dof);
/* Copy the handle's LGL nodes/weights (n = degree+1) and temporal D (n_tau^2,
 * row-major D(j,i) at [j*n_tau+i]) to host arrays (any may be NULL). */
int stg_constants(const stg_handle* h, double* nodes, double* weights, double* d_tau);

/* ---- operator applies (device pointers) -------------------------------- */

/* SemiDiscreteSystem::rhs (system.hpp:21) -> SpatialOperator::rhs
 * (spatial.hpp:107-266): F = M^{-1} L_h(u).  u, F: n_sdof. */
int stg_spatial_rhs(stg_handle* h, double t, const double* u, double* F);

/* Spatial Jacobian action J_F(u) v (replaces the assembled spatial_jacobian,
 * spatial.hpp:273-350, applied to v).  Exact for advection; Burgers uses the
 * exact linearisation. */
int stg_spatial_jvp(stg_handle* h, double t, const double* u, const double* v, double* Jv);

/* st_residual (stdg.hpp:56-76): R(U) of one time slab [t_n, t_n+dt] with
 * temporal upwind coupling to u_n.  U, R: n_dof; u_n: n_sdof. */
int stg_st_residual(stg_handle* h, double t_n, double dt, const double* u_n,
                    const double* U, double* R);

/* st_jacobian (stdg.hpp:79-110) applied matrix-free: Jv = dR/dU(U) v.
 * fd_eps > 0 (nonlinear models): central difference [R(U+h v)-R(U-h v)]/2h
 * with h = fd_eps * sqrt(1 + ||U||_2) / ||v||_2 (Walker-Pernice parameter). */
int stg_st_jvp(stg_handle* h, double t_n, double dt, const double* U, const double* v,
               double* Jv, double fd_eps);

/* rk_step stage residual (lodg.hpp:104-122), s = n_tau Lobatto IIIC stages
 * (operators.hpp:76-112): A-form R_i = U_i - u - dt sum_j A_ij F_j,
 * A^{-1}-form R_i = sum_j (A^{-1})_ij/dt (U_j - u) - F_i. */
int stg_stage_residual(stg_handle* h, int form, double t, double dt, const double* u,
                       const double* U, double* R);

/* stage_jacobian (lodg.hpp:43-85) applied matrix-free. */
int stg_stage_jvp(stg_handle* h, int form, double t, double dt, const double* U,
                  const double* v, double* Jv, double fd_eps);

/* ---- solvers (device pointers) ------------------------------------------ */

/* linear_solve GMRES branch (newton.hpp:68-77) on the slab Jacobian at U:
 * solves J(U) x = b, x holds the initial guess on entry; precond = STG_PRECOND_*. */
int stg_gmres_st(stg_handle* h, double t_n, double dt, const double* U, const double* b,
                 double* x, int restart, double tol, int max_it, int precond, int* iterations,
                 double* rel_residual);

/* The right preconditioner gmres_st would use, applied once: out = P^-1 in
 * (P = block-Jacobi part of the slab Jacobian at U; n_dof vectors). */
int stg_st_precond_apply(stg_handle* h, double dt, const double* U, int precond,
                         const double* in, double* out);

/* stdg_step (stdg.hpp:120-143): Newton from 1 (x) u_n; U (n_dof) receives the
 * slab solution, u_next (n_sdof) its last temporal block. */
int stg_stdg_step(stg_handle* h, double t_n, double dt, const double* u_n,
                  const stg_newton_config* cfg, double* U, double* u_next,
                  stg_solve_info* info);

/* stdg_integrate (stdg.hpp:152-173), device-resident: n_steps sequential slabs
 * from u0 over [t0, t_end] (t_k = t0 + (t_end - t0) k / n_steps, as the
 * reference), no host round trip between slabs.  u_final (n_sdof) receives the
 * last state; states (optional, (n_steps + 1) * n_sdof) every state incl. u0;
 * U_slabs (optional, n_steps * n_dof) every slab solution.  info: Newton and
 * GMRES iterations summed over the slabs (total_newton_iterations,
 * stdg.hpp:150), the last slab's residual and history. */
int stg_stdg_integrate(stg_handle* h, double t0, const double* u0, double t_end, int n_steps,
                       const stg_newton_config* cfg, double* u_final, double* states,
                       double* U_slabs, stg_solve_info* info);

/* integrate (lodg.hpp:158-181), device-resident: n_steps rk_steps of the
 * n_tau-stage Lobatto IIIC scheme; U_stages (optional, n_steps * n_dof). */
int stg_rk_integrate(stg_handle* h, int form, double t0, const double* u0, double t_end,
                     int n_steps, const stg_newton_config* cfg, double* u_final, double* states,
                     double* U_stages, stg_solve_info* info);

/* rk_step (lodg.hpp:89-149): Newton on the stage system from 1 (x) u, then
 * u_next = u + dt sum_j b_j F(t + c_j dt, U_j).  U: s*n_sdof stages. */
int stg_rk_step(stg_handle* h, int form, double t, double dt, const double* u,
                const stg_newton_config* cfg, double* U, double* u_next,
                stg_solve_info* info);

/* ---- host-buffer variants (H2D / D2H inside the call) -------------------- */
int stg_st_residual_host(stg_handle* h, double t_n, double dt, const double* u_n,
                         const double* U, double* R);
int stg_stdg_step_host(stg_handle* h, double t_n, double dt, const double* u_n,
                       const stg_newton_config* cfg, double* U, double* u_next,
                       stg_solve_info* info);
int stg_rk_step_host(stg_handle* h, int form, double t, double dt, const double* u,
                     const stg_newton_config* cfg, double* U, double* u_next,
                     stg_solve_info* info);

/* ---- device memory helpers (so FFI callers need no CUDA runtime of their own) */
int stg_device_alloc(long long n_doubles, double** out);
int stg_device_free(double* p);
/* dir: 0 = host -> device, 1 = device -> host, 2 = device -> device */
int stg_memcpy(double* dst, const double* src, long long n_doubles, int dir);
int stg_device_synchronize(void);
/* Page-locked host memory for the *_host entry points: buffers from here are
 * copied by DMA straight from / to the caller's memory (pageable buffers go
 * through the library's own pinned staging).  Fails with
 * STG_ERR_CUDA when no device is present. */
int stg_host_alloc(long long n_doubles, double** out);
int stg_host_free(double* p);

/* ---- host-only constants (no device needed) -------------------------------- */
/* lgl_rule (quadrature.hpp:66-105): n nodes and weights. */
int stg_lgl_rule(int n, double* nodes, double* weights);
/* diff_matrix (quadrature.hpp:128-144): D[j*n+i] = psi_i'(x_j). */
int stg_diff_matrix(int n, double* D);
/* lobatto_tableau (operators.hpp:76-112; s > 4 via to_butcher 55-72). */
int stg_lobatto_tableau(int s, double* A, double* b, double* c);

/* Launch counter (kernels launched through this handle since creation). */
long long stg_kernel_launches(const stg_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* STG_CUDA_H */
