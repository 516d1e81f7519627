/*
 * amgf.h -- C ABI of libamgf.so: B200 (sm_100a) AMGF-PCG for S = K + J^T D J.
 *
 * Method: arxiv 2505.18576 "AMG with Filtering".
 *   S = K + J^T D J ............................. eq:linsystem1
 *   I_c, P (natural embedding), A_w = P^T S P ..... Def. Discrete Operators
 *   M: I - M S = (I - B S)(I - P A_w^{-1} P^T S)(I - B S)   Def. AMGF
 *   B = one AMG V-cycle with l1 smoothing ......... PAPER.md:368, 587-595
 *   PCG, relative preconditioned residual ......... PAPER.md:368
 * The arithmetic follows DESIGN.md section 3 ("contract"), under which results are bitwise
 * identical to the CPU oracle in oracle/.
 *
 * Conventions for every function:
 *   - All array arguments are DEVICE pointers owned by the caller and only read during the call,
 *     unless the function name ends in _host (host pointers) or the comment says otherwise.
 *   - Index arrays are int32, values are IEEE binary64; matrices are block-CSR with column indices
 *     sorted ascending inside each row and 3x3 blocks stored row-major.
 *   - Dof numbering: dof = 3*node + component.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Every call is stream-ordered.
 *     Calls that return host-visible data (setup, pcg_solve, level_info/get, *_host) synchronise it.
 *   - No exception crosses the ABI.  A negative amgf_status is an error; amgf_last_error() returns
 *     a thread-local description.  On error the handle is left unchanged and usable (setup leaves
 *     *out = NULL).  A handle is used by one host thread / one stream at a time.
 */
#ifndef AMGF_H
#define AMGF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  AMGF_OK = 0,
  AMGF_NOT_CONVERGED = 1,      /* PCG reached max_it (not an error)              */
  AMGF_ERR_ARG = -1,           /* null pointer, bad size, Z not a permutation of I_c            */
  AMGF_ERR_NONFINITE = -2,     /* NaN/Inf in K, J or D                             */
  AMGF_ERR_DOMAIN = -3,        /* some D_k <= 0                                    */
  AMGF_ERR_NOT_SPD = -4,       /* non-positive Cholesky pivot in A_w or the coarsest operator   */
  AMGF_ERR_RANK = -5,          /* rank-deficient tentative prolongator block      */
  AMGF_ERR_BREAKDOWN = -6,     /* PCG: p.Sp <= 0 or r.Mr < 0                      */
  AMGF_ERR_CUDA = -7,          /* CUDA runtime error                                            */
  AMGF_ERR_OOM = -8,           /* device allocation failed                                      */
  AMGF_ERR_LIMIT = -9,         /* an internal capacity limit was exceeded (message says which)  */
  AMGF_ERR_FORMAT = -10        /* amgf_import: missing / truncated / inconsistent hierarchy file  */
} amgf_status;

typedef struct {
  int32_t pre_sweeps;      /* smoother sweeps before restriction, >= 1 (default 1); a sweep is one
                              Chebyshev polynomial or one l1-Jacobi step (see `smoother`)     */
  int32_t post_sweeps;     /* smoother sweeps after prolongation, >= 1 (default 1)           */
  int32_t coarsest_size;   /* stop coarsening at <= this many dofs (default 64) */
  int32_t max_levels;      /* default 25                                                     */
  int32_t power_iters;     /* power steps for lambda_max(D^-1 A) (default 6, DESIGN R19)      */
  int32_t nd_levels;       /* nested-dissection depth of A_w's elimination order (default 3, DESIGN R16) */
  int32_t smoother;        /* 1 = Chebyshev in D_l1^-1 A on [1/cheb_ratio, 1] (default, DESIGN R18 /
                              contract C23): each sweep is one polynomial of degree cheb_degree;
                              0 = l1-Jacobi (contract C4);
                              2 = nodal-block l1-Jacobi: x += B^-1 (b - A x), B = blockdiag(A_ii + diag of the
                              off-block l1 row sums) (variant f4, DESIGN R22, contracts C24/C25)            */
  int32_t cheb_degree;     /* 1..32 (default 2)                                               */
  uint64_t agg_seed;       /* aggregation priority seed (default 0x5EED)                     */
  double cheb_ratio;       /* > 1 (default 20)                                                */
  int32_t filter_basis;    /* 0 (default): P = the identity columns at I_c (the natural embedding,
                              PAPER.md:391), A_w = S[Z, Z];  1: P = J^T (the generality remark, PAPER.md:583-585:
                              any full-column-rank P), A_w = J S J^T (m x m) -- DESIGN.md R21 */
  int32_t pad_;
} amgf_config;

#define AMGF_MAX_LEVELS 32

typedef struct {
  int32_t iterations;      /* number of S*p products                                         */
  int32_t converged;       /* 1 if sqrt(r.Mr / r0.Mr0) < rtol                                */
  double rel_pres_norm;    /* final sqrt(r.Mr / r0.Mr0)                                      */
  double solve_ms;         /* device time of the solve (CUDA events)                         */
  double setup_ms;         /* the handle's last setup: amgf_setup / amgf_import wall time, or the device
                              time of the last amgf_update_D (numeric re-setup)                */
  int32_t n_levels;        /* levels of the AMG hierarchy (1 = the coarsest solve only)       */
  int32_t pad_;
  int64_t level_dofs[AMGF_MAX_LEVELS];  /* scalar unknowns per level (0 beyond n_levels)       */
  int64_t level_nnzb[AMGF_MAX_LEVELS];  /* stored blocks of each level operator (3x3 at level 0,
                                           6x6 below)                                        */
} amgf_report;

typedef struct amgf_ctx *amgf_handle;

/* Fill *cfg with the defaults above. */
void amgf_default_config(amgf_config *cfg);

/* Build the AMGF preconditioner for S = K + J^T D J on the GPU.
 *   nodes            number of 3-dof nodes; n = 3*nodes
 *   K_ptr[nodes+1], K_col[nnzb], K_val[9*nnzb]   K in 3x3 BSR (symmetric positive semidefinite
 *                    blocks per body, Dirichlet rows = identity)
 *   m, J_ptr[m+1], J_col[nnz], J_val[nnz]        gap Jacobian, scalar CSR over dofs
 *   D[m]             log-barrier Hessian diagonal, > 0
 *   Z[nc]            contact dofs I_c in the column order of P: duplicate-free and
 *                    containing every structurally nonzero column of J (e.g. exactly those columns, or
 *                    all components of the interface nodes).  NULL: J's columns in ascending order.
 *   B_nns[n*6]       near-null space (rigid-body modes), row-major n x 6
 *   cfg              NULL for defaults
 * Synchronises `stream`.  The handle deep-copies everything it needs. */
amgf_status amgf_setup(int32_t nodes, const int32_t *K_ptr, const int32_t *K_col, const double *K_val,
                       int32_t m, const int32_t *J_ptr, const int32_t *J_col, const double *J_val,
                       const double *D, const int32_t *Z, int32_t nc, const double *B_nns,
                       const amgf_config *cfg, void *stream, amgf_handle *out);

/* Numeric re-setup for a new D (same K, J, Z): re-forms S, A_w and its factor and all Galerkin
 * values; aggregation and all sparsity patterns are reused (they do not depend on D, reading R5). */
amgf_status amgf_update_D(amgf_handle h, const double *D, void *stream);

/* Numeric re-setup for the bound-constrained system (Remark boundconstr):
 *   A~ = K + J~^T D~ J~,  J~ = [J; I; -I],  D~ = diag(D, D_lo, D_up),
 * i.e. S = K + J^T D J + diag(D_lo) + diag(D_up); in the entry chain of contract C1 the rows of I and -I
 * follow J's rows, so a diagonal entry continues with fma(1*D_lo[p], 1, acc) then fma(-1*D_up[p], -1, acc).
 *   D_lo[n], D_up[n]   device arrays, finite and >= 0 (0: no bound on that dof); either may be NULL (zeros);
 *                      both NULL is amgf_update_D.  The bounds do not change I_c (Z stays J's contact dofs).
 * Errors as amgf_update_D (AMGF_ERR_DOMAIN for a negative bound diagonal). */
amgf_status amgf_update_D_box(amgf_handle h, const double *D, const double *D_lo, const double *D_up, void *stream);

/* z = M r, one AMGF application (Def. AMGF, three stages SPEC.md:245).  r, z: n doubles. */
amgf_status amgf_apply(amgf_handle h, const double *r, double *z, void *stream);

/* x = B b, one V-cycle of the AMG hierarchy.  b, x: n doubles. */
amgf_status amgf_vcycle(amgf_handle h, const double *b, double *x, void *stream);

/* y = A_level x (level 0: S).  Sizes: 3*nodes at level 0, 6*n_agg below. */
amgf_status amgf_spmv(amgf_handle h, int32_t level, const double *x, double *y, void *stream);

/* y = K x with the stiffness matrix the handle was set up with (contract C2 chains: per scalar row an fma chain
 * from +0 over K's blocks in ascending column, components ascending).  For the interior-point driver's residual
 * r_u = K u - f + J^T lambda (PAPER.md eq:optConditionsPrimalDual).  x, y: n doubles.  AMGF_ERR_ARG on an
 * imported handle. */
amgf_status amgf_spmv_K(amgf_handle h, const double *x, double *y, void *stream);

/* PCG on S x = b with AMGF (precond = 0) or AMG-only (precond = 1), x0 = 0, stops when
 * sqrt(r.Mr / r0.Mr0) < rtol or after max_it iterations.  Synchronises `stream`. */
amgf_status amgf_pcg_solve(amgf_handle h, const double *b, double *x, double rtol, int32_t max_it,
                           int32_t precond, amgf_report *rep, void *stream);

/* Same with HOST b and x: copies b host->device, solves, copies x device->host (e2e timing). */
amgf_status amgf_pcg_solve_host(amgf_handle h, const double *b_host, double *x_host, double rtol,
                                int32_t max_it, int32_t precond, amgf_report *rep, void *stream);

/* Write the handle's preconditioner to the existing directory `dir` (the exchange format
 * with the oracle, oracle/__init__.py Oracle.export): raw little-endian binary files plus a text manifest.
 *   amgf_hierarchy.txt   "amgf_hierarchy 1", then "key value" lines: nodes nlev nc bw nco and the solver
 *                        configuration (pre_sweeps post_sweeps smoother cheb_degree cheb_ratio nd_levels
 *                        coarsest_size max_levels power_iters agg_seed), then per level
 *                        "level l nodes b nnzb nnzb_P n_agg"
 *   L<l>_A_{ptr,col}.i32, L<l>_A_val.f64   level operator A_l (BSR, b x b row-major blocks; A_0 = S)
 *   L<l>_l1.f64                            l1 row sums d_l1 of A_l (smoother diagonal)
 *   L<l>_{P,R}_{ptr,col}.i32, _val.f64     prolongator P_l (b x 6 blocks) and R_l = P_l^T (6 x b), l < nlev-1
 *   Z.i32 [nc]                             contact dofs in P's column order
 *   pi.i32 [nc]                            elimination order of A_w as Z positions (DESIGN R16)
 *   Lw.f64 [nc*nc]                         dense lower Cholesky factor of A_w[pi,pi], row-major
 *   Lc.f64 [nco*nco]                       dense lower Cholesky factor of the coarsest operator
 * Dense factors are written in full (n_c^2 doubles: 571 MB at cfg 3).  Synchronises the handle's stream. */
amgf_status amgf_export(amgf_handle h, const char *dir);

/* Build a handle from a directory in the amgf_export format (written by amgf_export or by the oracle) so
 * that amgf_apply / amgf_vcycle / amgf_spmv / amgf_pcg_solve run on exactly that hierarchy (north star:
 * "single preconditioner applies on an identical exported hierarchy").  Nothing is recomputed: operators,
 * l1 diagonals, transfer operators and both factors are taken as stored; the solver configuration comes
 * from the manifest.  The A_w factor must vanish outside the structure of the nested-dissection order the
 * manifest's (nc, bw, nd_levels) define, pi must be that order and bw must be the structural band width
 * of S[Z, Z] (AMGF_ERR_FORMAT otherwise).  The handle has no K, J or D: amgf_update_D returns
 * AMGF_ERR_ARG.  Synchronises `stream`; *out = NULL on error. */
amgf_status amgf_import(const char *dir, void *stream, amgf_handle *out);

/* Hierarchy introspection (tests, bench).  info[0] = levels, info[1] = nc, info[2] = coarsest dofs,
 * info[3] = band width of A_w's factor, then per level l: info[4+6l .. 9+6l] =
 * {nodes, block size, nnzb(A), nnzb(P), n_agg, SELL slots of A}; info[196] = size of the separator
 * off-block factor, info[197] = number of nested-dissection blocks, info[198] = first level of the fused
 * coarse-tail kernel (-1: none), info[199] = its cluster size in CTAs, info[200] = the filter-space dimension nf
 * (n_c, or m with filter_basis 1; the size of arrays 22 and 25 below).  info needs 4 + 6*32 + 5 entries. */
amgf_status amgf_level_info(amgf_handle h, int64_t *info);

/* Copy one hierarchy array to the HOST buffer dst.  which: 0 A.ptr 1 A.col 2 A.val 3 P.ptr 4 P.col
 * 5 P.val 6 R.ptr 7 R.col 8 R.val 9 l1 diagonal 10 aggregate ids 11 near-null space 12 {lambda,
 * omega} 14 root flags 15 component labels 20 Z 22 in-block band of the factor of A_w[pi,pi] (nc x W
 * row-major over pi positions, W = band stride, L_ik at column bw-(i-k), diagonal at column bw)
 * 23 separator-vs-subtree factor entries 24 coarsest factor band (nco x Wc row-major, Wc =
 * band_stride(nco-1), L_ik at column nco-1-(i-k)) 25 pi (elimination order as Z positions) 27 block table
 * {int p0, len, kind, t0; int64 off; int level, pad}.  Sizes follow amgf_level_info.  Synchronises the handle's last stream. */
amgf_status amgf_level_get(amgf_handle h, int32_t which, int32_t level, void *dst);

/* PCG coefficients of the last amgf_pcg_solve: alpha_k = rho_k / (p_k . S p_k) and beta_k = rho_{k+1} / rho_k
 * of iterations k = 1..n (n <= iterations of that solve), into HOST arrays of n doubles.  They define the
 * Lanczos matrix of M S whose eigenvalues (Ritz values) estimate its spectrum (paper remark
 * upper_bound_estimate, section 4: beta = condition number of the AMG-preconditioned contact-free
 * operator).  AMGF_ERR_ARG if n exceeds the iterations of the last solve. */
amgf_status amgf_pcg_history(amgf_handle h, int32_t n, double *alpha, double *beta);

/* Device times (CUDA events, ms) of the last amgf_update_D into HOST ms[5]: {total, S = K + J^T D J,
 * hierarchy (power iterations, prolongators, Galerkin products, SELL refresh), coarsest Cholesky, A_w
 * factorization (side stream, concurrent with the hierarchy)}.  Zeros before the first update. */
amgf_status amgf_setup_times(amgf_handle h, double *ms);

/* Debug bounds check (no compute-sanitizer on the target pool): with AMGF_GUARD=1 in the environment every
 * internal allocation of a handle is followed by a 4 KB guard zone of a fixed byte pattern; this returns the
 * number of guard zones that were overwritten (out-of-bounds writes) since creation, -2 when AMGF_GUARD is not
 * set, -1 on a null handle or CUDA error.  Synchronises the device. */
int64_t amgf_debug_guard_check(amgf_handle h);

/* Number of kernel launches issued by this handle since creation (bench accounting). */
int64_t amgf_launch_count(amgf_handle h);

const char *amgf_last_error(void);
void amgf_destroy(amgf_handle h);

#ifdef __cplusplus
}
#endif
#endif
