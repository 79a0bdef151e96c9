/*
 * rdd.h — C ABI of the B200 solve pipeline for the RaNN + overlapping-Schwarz method
 * (arXiv 2412.19207). The reference library `rannddm` is header-only C++ with Eigen value
 * types (proj/include/rannddm, *.hpp); it exports no symbols, so this ABI is
 * the drop-in boundary a reference maintainer binds. Every entry point
 * names the reference function it replaces.
 *
 * Conventions
 *   - One context per host thread; one CUDA stream per context; calls are synchronous.
 *   - All pointer arguments are HOST pointers, caller-owned, copied in/out.
 *   - Dense matrices are column-major (Eigen's default storage order).
 *   - Return value: RDD_OK or an error class mirroring the reference's exception types;
 *     rdd_last_error() carries the reference's message text.
 */
#ifndef RDD_H
#define RDD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: the reference's exception classes */
#define RDD_OK 0
#define RDD_INVALID_ARGUMENT 1 /* std::invalid_argument */
#define RDD_RUNTIME_ERROR 2    /* std::runtime_error    */
#define RDD_DOMAIN_ERROR 3     /* std::domain_error     */
#define RDD_CUDA_ERROR 4       /* device failure (no reference analogue) */

/* problems (problems.hpp:43-173 built-ins, plus the BASELINE.json configs) */
#define RDD_PROBLEM_EXAMPLE1 1   /* problems.hpp:43  -Δu=f, multiscale sines, tanh-ramp L   */
#define RDD_PROBLEM_EXAMPLE2 2   /* problems.hpp:91  advection-diffusion space-time (no exact) */
#define RDD_PROBLEM_EXAMPLE3 3   /* problems.hpp:110 3-component -Δu+u=f on the cube          */
#define RDD_PROBLEM_POISSON 10   /* C1/C5: -Δu=f, u=Π sin(πx_a) on [0,1]^d                   */
#define RDD_PROBLEM_MULTISCALE 11/* C2: u=sin2πx sin2πy + 0.1 sin50πx sin50πy                 */
#define RDD_PROBLEM_HEAT 12      /* C3: u_t = 0.1Δu, space-time (x,y,t)                       */
#define RDD_PROBLEM_ADVECTION 13 /* C4: u_t + 2u_x = 0 on [0,2]x[0,1]                          */

/* decomposition kinds */
#define RDD_DECOMP_REFERENCE 0 /* geometry.hpp:109 build_decomposition(domain, counts, delta)      */
#define RDD_DECOMP_CELL 1      /* cell-centred boxes extended by `delta` x width per side (§8d)   */

/* tau modes (reduction.hpp:89 truncate; relative mode = BASELINE's σ/σmax > τ) */
#define RDD_TAU_OFF 0
#define RDD_TAU_ABSOLUTE 1
#define RDD_TAU_RELATIVE 2

#define RDD_PCA_PSI 0        /* reduction.hpp:30 build_sample_matrix           */
#define RDD_PCA_OP_APPLIED 1 /* reduction.hpp:53 build_operator_sample_matrix  */

/* krylov.hpp:16 SolverKind */
#define RDD_SOLVER_QR 0
#define RDD_SOLVER_CG 1
#define RDD_SOLVER_CGS 2
#define RDD_SOLVER_BICG 3
#define RDD_SOLVER_GMRES 4

/* schwarz.hpp:18 SchwarzKind; -1 = none */
#define RDD_PRECOND_NONE (-1)
#define RDD_PRECOND_AS 0
#define RDD_PRECOND_SAS 1
#define RDD_PRECOND_RAS 2

/* normal-operator formulation used by the Krylov loop */
#define RDD_OPERATOR_TWO_PASS 0 /* Hᵀ(H·w), runner.hpp:232-234 (reference semantics) */
#define RDD_OPERATOR_NORMAL 1   /* block-sparse HᵀH from the normal blocks           */

/* Mirrors rannddm::RunConfig (config.hpp:23-68) plus the BASELINE extensions. */
typedef struct rdd_config {
  int problem;      /* RDD_PROBLEM_*                                   */
  int n;            /* example1 complexity (config.hpp:27)             */
  int dim;          /* filled from the problem when 0                  */
  int counts[4];    /* subdomains per axis                             */
  int decomposition;/* RDD_DECOMP_*                                    */
  double delta;     /* overlap ratio (REFERENCE) or extension (CELL)   */
  int m;            /* hidden width                                    */
  int activation;   /* 0 tanh, 1 sin (basis.hpp:14)                    */
  uint64_t seed;
  int colloc[4];    /* collocation grid per axis                       */
  int boundary_per_edge; /* extra cell-centred points per domain edge (2-D, C1) */
  int test[4];      /* test grid per axis                              */
  int tau_mode;     /* RDD_TAU_*                                       */
  double tau;
  int pca_matrix;   /* RDD_PCA_*                                       */
  int solver;       /* RDD_SOLVER_*                                    */
  int precond;      /* RDD_PRECOND_*                                   */
  double rel_tol;
  int max_iter;     /* 0 = 10 * DoF (krylov.hpp:78-81)                 */
  int gmres_restart;/* 0 = full                                        */
  int op_form;      /* RDD_OPERATOR_* (product only; oracle ignores)   */
  int true_residual;/* GMRES: diagnostic true residual each step (krylov.hpp:360-367); 1 = as reference */
  int ref_resolution;/* example2 Crank-Nicolson reference grid (config.hpp:28); 0 = 2001    */
} rdd_config;

/* Mirrors rannddm::RunSummary (runner.hpp:147-156) + device phase split. */
typedef struct rdd_summary {
  uint64_t seed;
  int J, DoF, N, p;
  int iterations;
  int converged;
  int breakdown;
  double e_l2, e_l1n;
  double t_assemble, t_precond, t_solve, t_evaluate; /* seconds */
  double t_pca;        /* part of t_assemble (instance build incl. PCA) */
  double final_residual;
} rdd_summary;

typedef struct rdd_ctx rdd_ctx;

/* ---- lifecycle ---------------------------------------------------------------------- */
int rdd_create(rdd_ctx** out, int device);
void rdd_destroy(rdd_ctx* ctx);
const char* rdd_last_error(const rdd_ctx* ctx);
const char* rdd_version(void);
/* ABI self-check: sizeof(rdd_config), sizeof(rdd_summary) as compiled into the library */
int rdd_abi_sizes(int32_t* config_size, int32_t* summary_size);

/* ---- pipeline (runner.hpp) ---------------------------------------------------------- */
/* runner.hpp:40-70 build_instance(cfg, seed): decomposition, collocation grid, random bases
 * (host SplitMix64, bit-exact), then per-subdomain PCA on the device. */
int rdd_build_instance(rdd_ctx* ctx, const rdd_config* cfg, uint64_t seed);
/* runner.hpp:89-101 assemble_equilibrated → assembly.hpp:41-108 assemble, :186-204 column_norms/scale_columns */
int rdd_assemble(rdd_ctx* ctx, int equilibrate);
/* assembly.hpp:148-183 normal_blocks + schwarz.hpp:39-61 build_index_sets + :93-148 build_preconditioner */
int rdd_build_preconditioner(rdd_ctx* ctx, int kind);
/* runner.hpp:232-251: b = Hᵀ F_c, solve_with (krylov.hpp:391: cg, cgs, bicg, gmres), W ./= scales;
 * solver = RDD_SOLVER_QR: runner.hpp:217-222 densify + column-pivoted QR (krylov.hpp:97-101) */
int rdd_solve(rdd_ctx* ctx, int solver, double rel_tol, int max_iter, int gmres_restart);
/* runner.hpp:253-256 evaluate_solution + exact_values + compute_errors (problems.hpp:294) */
int rdd_evaluate(rdd_ctx* ctx, const int* test_res);
/* runner.hpp:202-275 run_single */
int rdd_run_single(rdd_ctx* ctx, const rdd_config* cfg, uint64_t seed, rdd_summary* out);
int rdd_get_summary(rdd_ctx* ctx, rdd_summary* out);
/* run_single again on the inputs already resident in HBM (bench: inputs resident when timing) */
int rdd_rerun_resident(rdd_ctx* ctx, rdd_summary* out);
/* number of library kernel launches issued by the calling thread so far */
int64_t rdd_launch_count(void);
/* cumulative host->device / device->host bytes copied by the calling thread */
int rdd_io_bytes(int64_t* h2d, int64_t* d2h);
/* CUDA events on the context's stream (slots 0..7) and the elapsed device time between two */
int rdd_event_record(rdd_ctx* ctx, int slot);
int rdd_event_elapsed(rdd_ctx* ctx, int slot_a, int slot_b, double* ms);

/* ---- caller inputs: the reference's objects instead of a RunConfig ------------------
 * The phase API above then runs on them: rdd_build_custom (instead of rdd_build_instance),
 * rdd_assemble, rdd_build_preconditioner, rdd_solve, rdd_evaluate_at. */
/* geometry.hpp:84-97 CartesianDecomposition as build_decomposition made it: dim, subdomains per
 * axis, the domain box, per subdomain (axis 0 slowest, geometry.hpp:146-167) the box lo/hi, centre
 * and half width (J x dim each, subdomain after subdomain) and its neighbour set (CSR over J,
 * ascending, self included, geometry.hpp:169-174). The boxes must form a tensor product. */
int rdd_set_decomposition(rdd_ctx* ctx, int dim, const int32_t* counts, const double* domain_lo,
                          const double* domain_hi, const double* box_lo, const double* box_hi,
                          const double* center, const double* half, const int32_t* nbr_ptr,
                          const int32_t* nbr_idx);
/* geometry.hpp:189-197 PointSet (the collocation points): N points, dim coordinates each, point
 * after point. */
int rdd_set_points(rdd_ctx* ctx, int64_t N, const double* pts);
/* basis.hpp:24-48 RandomBasis of every subdomain: R (m x dim, neuron after neuron) and b (m),
 * subdomain after subdomain; activation 0 = tanh, 1 = sin (basis.hpp:14). */
int rdd_set_bases(rdd_ctx* ctx, int J, int m, const double* R, const double* b, int activation);
/* problems.hpp:28-37 ProblemSpec evaluated by the caller at the collocation points:
 *   op_coef  the linear operator's coefficients on the jet (value, gradient[dim], Hessian upper
 *            triangle row by row; jet_len = 1 + dim + dim(dim+1)/2): LinearOperator::apply on unit
 *            jets (constant-coefficient operators, as every reference operator is);
 *   L_jets   the jet of the constraining factor L at every point (N x jet_len, point after point);
 *   F        f_c − A[G_c] at every point (N x C, column-major; assembly.hpp:97-106). */
int rdd_set_problem(rdd_ctx* ctx, int C, const double* op_coef, const double* L_jets, const double* F);
/* runner.hpp:40-70 build_instance on the caller inputs (index + PCA). From cfg only the PCA
 * settings (tau_mode, tau, pca_matrix) and op_form are read. */
int rdd_build_custom(rdd_ctx* ctx, const rdd_config* cfg);
/* runner.hpp:105-127 evaluate_solution(inst, W, pts) at M caller points (point after point) with
 * the caller's unscaled W (p x C, column-major) or, W = NULL, the last solve's; L_vals = L at the
 * points (M), G_vals = G_c at the points (M x C, column-major; NULL = 0); u_out M x C column-major. */
int rdd_evaluate_at(rdd_ctx* ctx, int64_t M, const double* pts, const double* W, const double* L_vals,
                    const double* G_vals, double* u_out);

/* ---- operators (pluggable into the reference's LinearMap, krylov.hpp:42-52) ---------- */
/* Vector lengths are checked like the reference's (RDD_INVALID_ARGUMENT, "... wrong length"). */
int rdd_matvec(rdd_ctx* ctx, const double* w, int64_t nw, double* y, int64_t ny);             /* assembly.hpp:110 */
int rdd_matvec_transpose(rdd_ctx* ctx, const double* r, int64_t nr, double* out, int64_t nout); /* :123 */
int rdd_normal_apply(rdd_ctx* ctx, const double* w, int64_t nw, double* out, int64_t nout);   /* runner.hpp:233 */
int rdd_precond_apply(rdd_ctx* ctx, const double* v, int64_t nv, double* z, int64_t nz,
                      int transpose);                                          /* schwarz.hpp:153/189 */

/* ---- dense diagnostics (krylov.hpp:403-440; runner.hpp:344-400) ----------------------- */
/* cap: the dense size limit (krylov.hpp:404 kDenseSpectrumCap = 4000 when <= 0; the reference's
 * override_caps passes 1<<20). Larger matrices fail with RDD_INVALID_ARGUMENT and the reference's
 * "matrix of size N exceeds the dense diagnostics cap (C)". */
/* spectrum_cmd / sweep_tau (runner.hpp:344-362, 381-393) on the assembled, equilibrated system:
 * eigenvalues of the dense HᵀH (ascending, imag 0) and of M⁻¹HᵀH (sorted by real part, then imag,
 * as write_spectrum_csv orders them) for the built preconditioner, and the condition numbers of
 * both (σmax / smallest positive σ). Each output may be NULL; arrays hold p entries. The
 * preconditioned outputs need rdd_build_preconditioner first. */
int rdd_spectra(rdd_ctx* ctx, int cap, double* normal_re, double* normal_im, double* precond_re, double* precond_im,
                double* cond_normal, double* cond_precond);
/* krylov.hpp:413 spectrum: all eigenvalues of a square column-major host matrix, sorted by
 * (real, imag); Householder Hessenberg reduction + Francis double-shift QR on the device. */
int rdd_dense_spectrum(rdd_ctx* ctx, int64_t rows, int64_t cols, const double* A, int cap, double* wr, double* wi);
/* krylov.hpp:423 singular_values: min(rows, cols) values, non-increasing (bidiagonalisation +
 * Golub–Kahan bisection on the device). */
int rdd_dense_singular_values(rdd_ctx* ctx, int64_t rows, int64_t cols, const double* A, int cap, double* s);
/* krylov.hpp:430 condition_number; RDD_DOMAIN_ERROR when every singular value is zero. */
int rdd_dense_condition_number(rdd_ctx* ctx, int64_t rows, int64_t cols, const double* A, int cap, double* cond);

/* ---- exports (parity tooling; assembly.hpp:206-256 densify/export analogues) --------- */
/* Returns the element count (or <0 on error). With out == NULL only the count is returned.
 * Names (e.g.): int "rows" j, "row_ptr", "p_j", "col_off", "nbr" i, "nb_pairs", "local_rank",
 * "local_n", "set" i, "owner", "mult", "iterations", "converged", "n_fallback", "qr_rank";
 * double "points", "box_lo"/"box_hi", "R" j, "b" j, "S" j, "sigma" j, "V" j, "H" j, "F",
 * "scales", "nb" k, "nb_dense", "H_dense", "local_cond", "W" c, "hist" c, "true_hist" c,
 * "approx", "exact". */
int64_t rdd_get_i(rdd_ctx* ctx, const char* what, int index, int32_t* out, int64_t cap);
int64_t rdd_get_d(rdd_ctx* ctx, const char* what, int index, double* out, int64_t cap);

/* ---- timing / instrumentation -------------------------------------------------------- */
/* Device time (ms) of the last call of a named kernel family and its launch count since reset. */
int rdd_kernel_stats(rdd_ctx* ctx, const char* family, double* ms_total, int64_t* launches);
int rdd_reset_stats(rdd_ctx* ctx);
int rdd_set_timing(rdd_ctx* ctx, int on);  /* per-family CUDA-event timing (adds syncs) */
int rdd_set_verbose(rdd_ctx* ctx, int on);  /* phase times and solver diagnostics on stderr */
/* Numeric switches of the device path (no reference counterpart; the reference always takes the
   eigen pseudo-inverse of schwarz.hpp:131-146):
     "full_rank_cond"  local blocks A_i whose condition estimate is below this take the Cholesky
                       path, the rest the eigen pseudo-inverse with the reference cutoff
                       (default in DESIGN.md §4 K8; 0 routes every block to the eigen path).
     "pca_refine"      subspace-refinement steps Y = Sᵀ(S·V) of the PCA (DESIGN §4 K4a;
                       0 = automatic).
     "pca_stop"        stop of the PCA's pivoted Cholesky relative to its first pivot (1e-17).
     "inv_max"         largest local order n_i kept as an explicit packed inverse (default 1024;
                       0 = every block through the envelope-packed Cholesky factor).
   Takes effect at the next rdd_build_preconditioner. RDD_INVALID_ARGUMENT for unknown names. */
int rdd_set_param(rdd_ctx* ctx, const char* name, double value);
/* Time `reps` calls of the normal operator on device-resident vectors (CUDA events). */
int rdd_bench_operator(rdd_ctx* ctx, int op_form, int reps, double* ms_per_call, double* bytes_per_call);
/* Time `reps` applications of the built Schwarz preconditioner (schwarz.hpp:153-215) on a
   device-resident vector (CUDA events on the context stream). bytes_per_call = algorithmic HBM
   bytes: the local operators (factor read twice, explicit inverse or dense pseudo-inverse read
   once), the gathered/scattered local vectors and the reduction. */
int rdd_bench_precond(rdd_ctx* ctx, int transpose, int reps, double* ms_per_call, double* bytes_per_call);
/* Batched Jacobi eigensolver probe (no reference counterpart; tuning aid): `batch` random
   symmetric matrices of order n, exactly `sweeps` sweeps, eigenvectors included; ms via events. */
int rdd_bench_jacobi(rdd_ctx* ctx, int n, int batch, int sweeps, double* ms);
/* Batched DMMA GEMM probe (no reference counterpart; tuning aid): `batch` independent products
   C = op(A)·op(B) of shape M x N x K, mode 0 = NN, 1 = TN (Aᵀ), 2 = NT (Bᵀ); ms per launch
   over `reps` launches (CUDA events). Algorithmic flops = 2·M·N·K·batch. */
int rdd_bench_gemm(rdd_ctx* ctx, int mode, int M, int N, int K, int batch, int reps, double* ms);

#ifdef __cplusplus
}
#endif
#endif /* RDD_H */
