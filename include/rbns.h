/*
 * rbns.h — C ABI of the B200-native batched online solver for the velocity-only reduced Navier–Stokes
 * method (arXiv 1807.11866).  Plain pointers and sizes only; no torch or CUDA C++ types in signatures.
 *
 * The reference ships no code for this path; its interface exists as the SPEC `online`
 * module.  Each entry point names the SPEC operation it replaces:
 *
 *   rbns_model_create        <- ReducedModel hand-off to the online stage
 *   rbns_model_create2       <- same, per-form term families (a/c0 linear, c quadratic, d0/f loads, B
 *                               coupling) with their own descriptors (SPEC.md:339-346 AffineFormSet,
 *                               SPEC.md:449-457 build_reduced_model)
 *   rbns_solve               <- online.solve_block, batched ("batch sweep API")
 *   rbns_solve_host          <- same, host buffers in/out (the query API a CPU caller binds)
 *   rbns_reduced_operator    <- online.reduced_operator (residual + Jacobian)
 *   rbns_solve_ex            <- same as rbns_solve with this call's statistics returned through an out-parameter
 *                               (per-query phase timings, "timing instrumentation is
 *                               per-query and contention-free")
 *   rbns_recover_pressure    <- solve_block step 2, B_sp p = f_s - A_sv u
 *   rbns_reconstruct_pressure<- online.reconstruct_pressure, combined scheme: p = P_att u with the model's
 *                               attached pressure modes
 *   rbns_project_convection  <- build_reduced_model's c-term contraction C_jkl = c(ψ_j, ψ_k, ψ_l) (offline,
 *                               SPEC.md:449-457; reference assemble.py:86-101 convection_matrices)
 *   rbns_error_string        <- errors.RbflowError messages (reference errors.py:4-21)
 *
 * All arrays are IEEE fp64 (or the stated integer type), row-major, C-contiguous.  "dev" pointers are CUDA
 * device pointers on the model's device; "host" pointers are ordinary (pinned or pageable) host memory.
 * Per-sample outcomes are status codes, not errors (NON_CONVERGED is "a reportable outcome,
 * not a crash").  Every function returns RBNS_OK (0) or a nonzero rbns_error; rbns_last_error_message()
 * gives the detail for the calling thread.
 */
#ifndef RBNS_H_
#define RBNS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RBNS_ABI_VERSION 3
#define RBNS_MAX_TERMS 256 /* per term family */
#define RBNS_MAX_GROUPS 4  /* distinct mu1 powers tying linear terms to the quadratic blocks (see create2) */

/* θ_q(μ) descriptor kinds; μ = (mu0, mu1) = (alpha [rad], Re) for the BASELINE configs, (φ [rad], u∞) for the
 * paper's models.  value = scale * base. */
enum rbns_theta_kind {
  RBNS_THETA_CONST = 0,       /* 1                           */
  RBNS_THETA_COS_K = 1,       /* cos(k alpha)                */
  RBNS_THETA_SIN_K = 2,       /* sin(k alpha)                */
  RBNS_THETA_COS_SIN_POW = 3, /* cos(alpha)^k * sin(alpha)^m */
  RBNS_THETA_MONOMIAL = 4     /* mu0^k * mu1^m  (the paper's scale*phi^k*u_inf^m) */
};

/* per-sample outcome (int8) */
enum rbns_status {
  RBNS_CONVERGED = 0,         /* ||delta||_2 <= tol * ||u||_2                         */
  RBNS_NON_CONVERGED = 1,     /* hit max_iter                           */
  RBNS_SINGULAR_SYSTEM = 2,   /* zero / non-finite pivot in the Newton system         */
  RBNS_SINGULAR_RECOVERY = 3, /* pressure Gramian B_sp not SPD          */
  RBNS_NONFINITE = 4          /* Newton update produced inf/nan; u keeps last iterate */
};

enum rbns_error {
  RBNS_OK = 0,
  RBNS_ERR_INVALID_ARGUMENT = 1,
  RBNS_ERR_CUDA = 2,
  RBNS_ERR_OUT_OF_MEMORY = 3,
  RBNS_ERR_UNSUPPORTED = 4,
  RBNS_ERR_NO_PRESSURE = 5,
  RBNS_ERR_NO_ATTACHED = 6     /* reconstruct_pressure on a model without attached pressure modes */
};

typedef struct rbns_theta_term {
  int32_t kind;
  int32_t k;
  int32_t m;
  int32_t reserved;
  double scale;
} rbns_theta_term;

typedef struct rbns_model_desc {
  int32_t n;                    /* reduced velocity dimension N (paper M_V)              */
  int32_t q;                    /* affine terms Q, 1..RBNS_MAX_TERMS                      */
  int32_t n_p;                  /* pressure dimension Np (0 = no recovery operators)      */
  int32_t reserved;
  const double* A;              /* host Q x N x N      projected a-terms (times nu online)  */
  const double* C;              /* host Q x N x N x N  C[q][j][k][l] = c_q(u_j, u_k, u_l)   */
  const double* f;              /* host Q x N          projected loads                      */
  const double* Mp;             /* host Np x Np SPD pressure Gramian (B_sp) or NULL         */
  const double* Bq;             /* host Q x Np x N coupling terms or NULL                   */
  const rbns_theta_term* theta; /* host, Q descriptors                                      */
} rbns_model_desc;

/* One affine family: count terms, each an operator of the family's shape with its own descriptor. */
typedef struct rbns_term_family {
  int32_t count;                /* 0..RBNS_MAX_TERMS                                        */
  int32_t reserved;
  const double* data;           /* host, count x (family shape), row-major                 */
  const rbns_theta_term* theta; /* host, count descriptors                                  */
} rbns_term_family;

enum rbns_model_flags {
  RBNS_NU_LINEAR = 1,   /* multiply the linear family by nu = 1/mu1 (BASELINE configs); clear for the paper's
                           models, whose a-term descriptors carry nu in their scale */
  RBNS_STOP_ABSOLUTE = 2 /* stop when ||delta_stop||_2 <= tol (the coupled solvers' rule) instead
                            of ||delta_stop||_2 <= tol * ||u_stop||_2 (block rule) */
};

/* Reduced model with per-form families.  Residual and Jacobian:
 *   R(u) = L(mu) u + sum_c theta_c(mu) C_c(u, u) - sum_f theta_f(mu) f_f
 *   J(u) = L(mu)   + sum_c theta_c(mu) sum_k (C_c[m,k,l] + C_c[k,m,l]) u_k
 *   L(mu) = [nu] sum_a theta_a(mu) A_a        (a-terms and the lift's c0-terms: everything linear in u)
 * Pressure recovery (cfg-4 form): Mp p = sum_b theta_b(mu) B_b u.
 * Each linear term's h-row contribution (L u, needed by the residual) rides on the quadratic block whose
 * descriptor equals its own up to a constant factor and a power of mu1 (RBNS_MAX_GROUPS distinct powers);
 * linear terms without such a block get an extra (velocity-free) block of the contraction. */
typedef struct rbns_model_desc2 {
  int32_t n;                   /* reduced velocity dimension N                           */
  int32_t n_p;                 /* pressure dimension Np (0 = no recovery)                */
  int32_t flags;               /* rbns_model_flags                                       */
  int32_t n_stop;              /* leading unknowns in the stop norm, 0 = all N (coupled saddle systems:
                                  the velocity block)                        */
  rbns_term_family linear;     /* count x N x N         (>= 1 term)                      */
  rbns_term_family quadratic;  /* count x N x N x N     C[j][k][l] = c(u_j, u_k, u_l)    */
  rbns_term_family load;       /* count x N                                              */
  rbns_term_family coupling;   /* count x Np x N        (Np > 0)                         */
  const double* Mp;            /* host Np x Np SPD, or NULL when Np = 0                  */
  /* ABI 3: optional attached pressure modes of the combined scheme ("optional attached pressure
   * modes for the combined scheme"): column j holds the pressure data attached to velocity mode j, so the
   * reconstructed pressure is p = P_att u.  n_att = 0 / P_att = NULL: none. */
  int32_t n_att;               /* rows of P_att (pressure coefficients)                 */
  int32_t reserved2;
  const double* P_att;         /* host n_att x N                                         */
} rbns_model_desc2;

typedef struct rbns_model rbns_model;

/* Statistics of one solve: returned per call by rbns_solve_ex / rbns_solve_host_ex; rbns_get_stats reads the
 * most recent call's copy kept on the model (a convenience for single-threaded callers). */
typedef struct rbns_stats {
  int64_t sample_iterations;      /* sum over samples of Newton iterations performed               */
  int64_t contraction_iterations; /* sample-iterations that ran the convective GEMM (iter >= 2)    */
  int32_t newton_rounds;          /* outer iterations executed (max over samples)                  */
  int32_t kernel_launches;        /* CUDA kernels launched by the call                             */
  int32_t gemm_launches;          /* launches of the DMMA contraction kernel (incl. the u = 0 step) */
  int32_t lu_launches;            /* launches of the Newton-update (Gauss-Jordan) kernel           */
  double ms_gemm;                 /* device time (CUDA events) in the contraction kernel          */
  double ms_lu;                   /* device time in the Newton-update kernel                      */
  double ms_recovery;             /* device time in pressure recovery                             */
  double ms_total;                /* device time of the whole call (excluding host copies)        */
  double ms_assembly;             /* device time of the u = 0 step's affine assembly (J = nu A(mu)) */
  int64_t pivot_fallbacks;        /* sample-iterations whose pivot-order hint failed verification and
                                     ran the full-search factorization                               */
} rbns_stats;

/* Copy operators to `device`, build the symmetrised GEMM operand S_q = C_q + C_q^(12),
 * and factor Mp once.  The handle is immutable afterwards and may be shared by concurrent solves. */
int rbns_model_create(const rbns_model_desc* desc, int device, rbns_model** out);
/* Per-family form; rbns_model_create(d) == rbns_model_create2 with every family on d->theta and
 * RBNS_NU_LINEAR. */
int rbns_model_create2(const rbns_model_desc2* desc, int device, rbns_model** out);
/* term counts: linear, quadratic, load, coupling, contraction blocks (quadratic + extra), h groups */
int rbns_model_terms(const rbns_model* model, int32_t counts[6]);
int rbns_model_destroy(rbns_model* model);
int rbns_model_info(const rbns_model* model, int32_t* n, int32_t* q, int32_t* n_p, int32_t* device);
/* bytes of device memory the handle owns */
int64_t rbns_model_device_bytes(const rbns_model* model);
/* Contraction path of the handle's velocity operand: 0 = FP64 DMMA kernel (rbns_contract.cuh); s > 0 = the
 * tcgen05 INT8 kernel over s error-free slices per operand entry (rbns_oz.cuh; the default, RBNS_CONTRACT=dmma
 * at model create selects the DMMA kernel).  Both evaluate the same sums to binary64 round-off. */
int rbns_model_contraction_slices(const rbns_model* model);

/* Batched velocity-only Newton solve + optional pressure recovery, device buffers.
 *   mu          dev  B x 2   (alpha [rad], Re)
 *   u           dev  B x N   out: velocity coefficients (last iterate)
 *   p           dev  B x Np  out: recovered pressure, or NULL to skip recovery
 *   iters       dev  B int32 out: Newton linear solves performed, incl. the accepted one
 *   status      dev  B int8  out: rbns_status
 *   last_update dev  B       out: ||delta||_2 of the last accepted update (NaN if none)
 *   stream      cudaStream_t (NULL = legacy default stream)
 * Blocks the host until the results are complete on `stream`.  Newton: u0 = 0, stop when
 * ||delta||_2 <= tol * ||u_new||_2, at most max_iter solves. */
int rbns_solve(rbns_model* model, const double* mu, int64_t batch, double tol, int32_t max_iter,
               double* u, double* p, int32_t* iters, int8_t* status, double* last_update, void* stream);

/* rbns_solve with this call's statistics written to *stats (may be NULL): concurrent solves on different
 * streams each get their own numbers. */
int rbns_solve_ex(rbns_model* model, const double* mu, int64_t batch, double tol, int32_t max_iter, double* u,
                  double* p, int32_t* iters, int8_t* status, double* last_update, rbns_stats* stats, void* stream);

/* Same as rbns_solve with HOST buffers: the call copies mu in and results out (the end-to-end path a
 * CPU-side caller binds; host<->device copies are part of the call). */
int rbns_solve_host(rbns_model* model, const double* mu, int64_t batch, double tol, int32_t max_iter,
                    double* u, double* p, int32_t* iters, int8_t* status, double* last_update,
                    void* stream);

/* rbns_solve_host with per-call statistics (see rbns_solve_ex). */
int rbns_solve_host_ex(rbns_model* model, const double* mu, int64_t batch, double tol, int32_t max_iter, double* u,
                       double* p, int32_t* iters, int8_t* status, double* last_update, rbns_stats* stats,
                       void* stream);

/* Residual and Jacobian of the reduced system at states eta, batched (debug / FD tests).
 *   mu dev B x 2, eta dev B x N, residual dev B x N, jacobian dev B x N x N (row l, column m = dR_l/du_m) */
int rbns_reduced_operator(rbns_model* model, const double* mu, const double* eta, int64_t batch,
                          double* residual, double* jacobian, void* stream);

/* Pressure recovery alone for given velocities: p = Mp^{-1} sum_q theta_q(mu) B_q u (device buffers).
 * status (dev, may be NULL) receives RBNS_SINGULAR_RECOVERY where Mp could not be factored. */
int rbns_recover_pressure(rbns_model* model, const double* mu, const double* u, int64_t batch,
                          double* p, int8_t* status, void* stream);

/* Combined-scheme pressure reconstruction: p = P_att u for every sample, device buffers.
 *   u dev B x N, p dev B x n_att.  RBNS_ERR_NO_ATTACHED when the model carries no attached modes. */
int rbns_reconstruct_pressure(rbns_model* model, const double* u, int64_t batch, double* p, void* stream);
/* rows of P_att (0: none) */
int rbns_model_attached(const rbns_model* model, int32_t* n_att);

int rbns_get_stats(const rbns_model* model, rbns_stats* out);

/* Offline projection of one convective term onto a reduced basis tabulated at P quadrature points (device
 * buffers on the current device, stream-ordered; no model handle):
 *   C[j][k][l] = sum_p w[p] sum_{c,d} val_u[p][d][j] * grad[p][c][d][k] * val_w[p][c][l]
 *   val_u dev P x 2 x N (advecting functions), grad dev P x 2 x 2 x N (grad[p][c][d][k] = d_d psi_{k,c}),
 *   val_w dev P x 2 x N (test functions), w dev P (quadrature weight x |det|), C dev N x N x N.
 * splits: split-K slices over the points (0: automatic); the slices are summed in a fixed order (deterministic). */
int rbns_project_convection(const double* val_u, const double* grad, const double* val_w, const double* w,
                            int64_t points, int32_t n, double* C, int32_t splits, void* stream);

const char* rbns_error_string(int code);
const char* rbns_last_error_message(void);
int rbns_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RBNS_H_ */
