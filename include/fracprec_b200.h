/*
 * fracprec_b200 — C ABI of the B200-native solve phase (GMRES + block-AMG
 * preconditioners t-p-u / t-u-p / t-u-p* for the 3x3 contact/fracture-flow
 * Jacobian of arXiv 2112.12397).
 *
 * Every entry point replaces one call of the reference's C++ API
 * (/root/reference/proj/core/include/fracprec/ headers); the mapping is noted per
 * function.  Conventions:
 *   - return value: FP_OK (0) or an error code; fp_last_error() gives the
 *     message (thread-local).  Codes mirror the reference's exception classes:
 *     std::invalid_argument -> FP_INVALID_ARGUMENT, fracprec::numerical_error ->
 *     FP_NUMERICAL_ERROR (errors.hpp:15-18); CUDA failures -> FP_CUDA_ERROR.
 *   - matrices cross the boundary as CSR views in the reference's layout
 *     (csr.hpp:16-22: 0-based, columns sorted and unique per row).  Row offsets
 *     may be 32-bit (row_offsets32, the reference's std::vector<int>) or 64-bit
 *     (row_offsets64); exactly one must be non-null.
 *   - handles own all device memory; host arrays are borrowed for the call.
 *   - `mem` selects where vector arguments live: FP_MEM_HOST or FP_MEM_DEVICE.
 *   - one CUDA stream per system handle (non-blocking); calls on one handle are
 *     serialized.  Ordering contract for FP_MEM_DEVICE vectors: the call does
 *     not wait on any other stream, so the caller must complete the producers
 *     of its inputs first (the Python mirror synchronizes torch's current
 *     stream); every call returns only after its outputs are written, so they
 *     may be consumed on any stream afterwards.
 */
#ifndef FRACPREC_B200_H
#define FRACPREC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FP_OK 0
#define FP_INVALID_ARGUMENT 1
#define FP_NUMERICAL_ERROR 2
#define FP_CUDA_ERROR 3
#define FP_INTERNAL_ERROR 4

#define FP_MEM_HOST 0
#define FP_MEM_DEVICE 1

/* PrecondConfig::Variant (precond.hpp:20) */
#define FP_TPU 0
#define FP_TUP 1
#define FP_TUP_STAR 2

/* AmgConfig::Smoother (amg.hpp:24) */
#define FP_SMOOTHER_JACOBI 0
#define FP_SMOOTHER_SGS 1
#define FP_SMOOTHER_CHEBYSHEV 2 /* extension: degree-k Chebyshev in D^-1 A (not in the reference) */
#define FP_SMOOTHER_MCGS 3      /* extension: multicolour symmetric Gauss-Seidel (greedy colouring) */

typedef struct fp_csr {
  int32_t n_rows, n_cols;
  const int32_t* row_offsets32; /* n_rows + 1, or NULL */
  const int64_t* row_offsets64; /* n_rows + 1, or NULL */
  const int32_t* col_indices;
  const double* values;
} fp_csr;

/* BlockSystem (block.hpp:36-45): J = [A C1 Q1; C2 -H 0; Q2 0 T] */
typedef struct fp_block_system {
  int32_t n_u, n_t, n_p;
  fp_csr A, C1, Q1, C2, H, Q2, T, F_u; /* F_u may be empty (n_rows = 0) */
} fp_block_system;

/* AmgConfig (amg.hpp:19-31) */
typedef struct fp_amg_config {
  double strength_threshold;
  int32_t max_coarse, pre_sweeps, post_sweeps;
  int32_t smoother; /* the GPU path runs FP_SMOOTHER_JACOBI, _CHEBYSHEV or _MCGS */
  int32_t prolongation_smoothing;
  int32_t cycles_per_apply;
  double jacobi_omega, stall_ratio;
  int32_t max_levels;
  /* FP_SMOOTHER_CHEBYSHEV: polynomial degree per sweep, lambda_max / lambda_min, power iterations */
  int32_t chebyshev_degree;
  double chebyshev_ratio;
  int32_t power_iterations;
  int32_t row_sum; /* FP_ROW_SUM_* (0 = ordered, the reference's summation order) */
} fp_amg_config;

/* Row-sum order of the V-cycle's coarse operators (A_l for l >= 1, R_l = P_l^T):
 * FP_ROW_SUM_ORDERED - left to right, the reference's spmv / spmv_transpose order;
 * FP_ROW_SUM_STRIDED - extension: 32 lane-strided partials (entry k of a row into
 *                      partial k mod 32, in order) combined by an xor tree; one warp
 *                      per row.  Restated in the oracle (spmv_strided32). */
enum { FP_ROW_SUM_ORDERED = 0, FP_ROW_SUM_STRIDED = 1 };

/* How the fracture-block factor (T or S~2, SparseFactor) is applied:
 * FP_FACTOR_SWEEP   - forward/backward column sweeps on the banded factor;
 * FP_FACTOR_INVERSE - the explicit inverse of every fracture block (columns =
 *                     sweep solves of unit vectors), streamed as a block GEMV;
 * FP_FACTOR_PANEL   - the factor cut into panels of one bandwidth, so L and U are
 *                     block bidiagonal; per panel the dense L_qq^-1, L_qq^-1 L_q,q-1
 *                     (and U's) are streamed by two chains of cluster steps (needs a
 *                     factor without row interchanges);
 * FP_FACTOR_AUTO    - panels when available, else the faster of the other two that
 *                     fits device memory. */
enum { FP_FACTOR_AUTO = 0, FP_FACTOR_SWEEP = 1, FP_FACTOR_INVERSE = 2, FP_FACTOR_PANEL = 3 };

/* PrecondConfig (precond.hpp:19-30); inner is always AMG on this path */
typedef struct fp_precond_config {
  int32_t variant;
  fp_amg_config amg;
  int32_t factor_solve; /* FP_FACTOR_* (0 = auto) */
} fp_precond_config;

/* Arnoldi orthogonalization.  Both use the reference's DGKS second-pass test
 * (gmres.cpp:96-102: repeat the pass when ||w|| < ||w_pre|| / sqrt 2).
 * FP_ORTH_MGS - modified Gram-Schmidt, the reference's own loop (default);
 *               one grid-wide reduction per basis vector.
 * FP_ORTH_CGS - classical Gram-Schmidt: all coefficients of a pass from one
 *               reduction (2 per step, 4 with the second pass); same iterates in
 *               exact arithmetic, held to the reference's GMRES bars. */
enum { FP_ORTH_MGS = 0, FP_ORTH_CGS = 1 };

typedef struct fp_gmres_options {
  double tol;       /* relative, on ||b - op x|| (gmres.hpp:29-33) */
  int32_t restart;  /* GMRES(m) restart length; >= max_iter gives full GMRES */
  int32_t max_iter;
  int32_t scaled;   /* 1: solve the driver's D J D system (driver.cpp:229-255) */
  int32_t orthogonalization; /* FP_ORTH_* (0 = MGS, the reference's) */
  int32_t probe;             /* 1: time the finest-level Jacobi sweep of every 8th Arnoldi step
                                (CUDA events inside the graph) into fp_solve_stats.probe_* */
} fp_gmres_options;

/* SolveStats (gmres.hpp:15-22) + bookkeeping */
typedef struct fp_solve_stats {
  int32_t iterations, converged, breakdown, restarts, precond_applies;
  double final_rel_residual;
  double device_seconds;       /* CUDA-event time of the solve on the handle's stream */
  int64_t kernel_launches;     /* kernels of this library launched by the solve (graph nodes included) */
  double* residual_history;    /* optional caller buffer */
  int32_t history_capacity;
  int32_t history_len;
  double probe_ms;             /* with fp_gmres_options.probe: summed time of the probed launches */
  int32_t probe_launches;
  int32_t reorth_steps;        /* Arnoldi steps that ran the second (DGKS) orthogonalization pass */
} fp_solve_stats;

typedef struct fp_system fp_system;           /* device-resident J (BlockSystem) */
typedef struct fp_precond fp_precond;         /* device-resident M^-1 */
typedef struct fp_host_precond fp_host_precond; /* host-built preconditioner data */

/* Reference-built hierarchy upload (TpuPreconditioner / TupPreconditioner,
 * precond.hpp:53-74, AmgHierarchy amg.hpp:35-50).  levels[0].A is S~ (t-p-u)
 * or S1 (t-u-p); levels[l>0].P maps level l to level l-1; diag = smoother_diag.
 * factor_matrix is T (t-p-u, factored LDL^T) or S~2 (t-u-p, factored LU);
 * h_blocks are the n_p regularized 3x3 blocks of H~ (BlockDiagonal3, row-major). */
typedef struct fp_amg_level_desc {
  fp_csr A;
  fp_csr P;
  const double* smoother_diag;
} fp_amg_level_desc;

typedef struct fp_precond_desc {
  int32_t variant;
  const double* h_blocks;
  fp_csr factor_matrix;
  int32_t n_levels;
  const fp_amg_level_desc* levels;
  fp_amg_config amg;
  int32_t factor_solve; /* FP_FACTOR_* (0 = auto) */
} fp_precond_desc;

const char* fp_last_error(void);
const char* fp_version(void);
void fp_amg_config_default(fp_amg_config* cfg); /* reference defaults, smoother = Jacobi */

/* ---- system: BlockSystem upload and BlockSystemOperator::apply (block.cpp:55-74) */
int fp_system_create(const fp_block_system* J, fp_system** out);
void fp_system_destroy(fp_system* s);
int fp_system_dims(const fp_system* s, int32_t* n_u, int32_t* n_t, int32_t* n_p);
/* y = J x */
int fp_system_apply(fp_system* s, const double* x, double* y, int32_t mem);
/* BlockScaling::from (driver.cpp:114-125) */
int fp_block_scaling(const fp_system* s, double* st, double* sp);

/* ---- preconditioner build: build_tpu / build_tup (precond.cpp:119-202) on the host */
int fp_host_precond_build(const fp_block_system* J, const fp_precond_config* cfg, const double* node_coords,
                          int32_t n_nodes, fp_host_precond** out);
void fp_host_precond_destroy(fp_host_precond* p);
/* number of AMG levels and the row count of each (levels[] may be NULL) */
int fp_host_precond_levels(const fp_host_precond* p, int32_t* n_levels, int32_t* level_rows);
/* copy out a host-built matrix: what 0 = A_l (level), 1 = P_l (level >= 1), 2 = T or S~2.
 * Call with row_offsets == NULL first to get dims / nnz. */
int fp_host_precond_matrix(const fp_host_precond* p, int32_t what, int32_t level, int32_t* n_rows, int32_t* n_cols,
                           int64_t* nnz, int64_t* row_offsets, int32_t* col_indices, double* values);
/* what 0 = H~ blocks (9 n_p), 1 = T_diag (t-p-u) or S_K (t-u-p), 2 = smoother diag of level `level`,
 * 3 = {lambda_max} of level `level` (Chebyshev smoother, extension) */
int fp_host_precond_vector(const fp_host_precond* p, int32_t what, int32_t level, double* out, int64_t* len);

/* build_tpu / build_tup (precond.cpp:119-202) on a generated workload (libfp_workload.so,
 * include/fracprec_workload.h) and its node coordinates in place — fp_host_precond_build
 * without copying the blocks (the large configs' fine operator is tens of GB on the host) */
typedef struct fp_workload fp_workload;
int fp_workload_host_precond_build(const fp_workload* w, const fp_precond_config* cfg, fp_host_precond** out);

/* Upload-time choices of a host-built preconditioner (they change no host data): the coarse
 * row-sum order (FP_ROW_SUM_*) and the factor application (FP_FACTOR_*) the next
 * fp_precond_create uses.  One host setup can so be uploaded in every mode. */
int fp_host_precond_set_upload(fp_host_precond* p, int32_t row_sum, int32_t factor_solve);

/* ---- Jacobian assembly of the fracture blocks on the device:
 * assemble_fracture_blocks (assembly.cpp:229-406) — C2, H, T, F_u and Q2 for a fracture state, the
 * part of the Jacobian the Newton loop rebuilds every step (A, C1, Q1 stay).  create uploads the
 * workload's fracture model (faces, TPFA edges, Dirichlet flags, constants); run assembles the blocks
 * for a state (include/fracprec_workload.h fp_fracture_state) and, when s is not NULL, installs them
 * into the device system (layouts and block scaling rebuilt on the device; build the preconditioner
 * afterwards, as driver.cpp:229-230 does every Newton step).  matrix copies a block out
 * (what 0 = C2, 1 = H, 2 = T, 3 = F_u, 4 = Q2; call with row_offsets == NULL for the sizes). */
typedef struct fp_fracture_state fp_fracture_state;
typedef struct fp_fracture_assembly fp_fracture_assembly;
int fp_fracture_assembly_create(const fp_workload* w, fp_fracture_assembly** out);
void fp_fracture_assembly_destroy(fp_fracture_assembly* a);
int fp_fracture_assembly_run(fp_fracture_assembly* a, const fp_fracture_state* st, fp_system* s);
int fp_fracture_assembly_matrix(const fp_fracture_assembly* a, int32_t what, int32_t* n_rows, int32_t* n_cols,
                                int64_t* nnz, int64_t* row_offsets, int32_t* col_indices, double* values);

/* ---- upload to the device */
int fp_precond_create(fp_system* s, const fp_host_precond* hp, fp_precond** out);
int fp_precond_upload(fp_system* s, const fp_precond_desc* desc, fp_precond** out);
void fp_precond_destroy(fp_precond* p);

/* ---- applies: TpuOperator / TupOperator::apply (precond.cpp:285-296), amg_apply (amg.cpp:293-305) */
int fp_precond_apply(fp_precond* p, const double* x, double* y, int32_t mem);
int fp_amg_apply(fp_precond* p, const double* r, double* x, int32_t mem);
/* InnerSolver::call_count / reset_count (precond.hpp:34-42) */
int64_t fp_precond_inner_calls(fp_precond* p, int32_t reset);
/* Where build_tpu / build_tup run (fp_host_precond_build, fp_workload_host_precond_build):
 * 1 = on the device (the default when a CUDA device is present): the Schur core, the strength graph,
 *     the prolongation smoothing and the Galerkin products in HBM, the BFS aggregation and the
 *     per-aggregate QR on the host; the AMG levels stay device-resident for fp_precond_create
 *     (fp_host_precond_matrix downloads them on request);
 * 0 = on the host (OpenMP; FRACPREC_B200_SETUP=host selects it at start-up).
 * Both build the oracle's hierarchy bit for bit.  Applies to builds started afterwards. */
int fp_set_setup_backend(int32_t device);
int fp_setup_backend(int32_t* device);
/* The factor application the preconditioner resolved to: FP_FACTOR_SWEEP or FP_FACTOR_INVERSE */
int fp_precond_factor_solve(const fp_precond* p, int32_t* mode);
/* algorithmic HBM bytes and kernel launches of one fp_precond_apply / fp_system_apply */
int fp_precond_traffic(fp_precond* p, double* apply_bytes, int32_t* apply_launches, double* japply_bytes);

/* Kernel timing for the roofline: each phase is launched `reps` times back to
 * back on the handle's stream between CUDA events (ms = average per launch);
 * bytes are the algorithmic HBM bytes of one launch. */
typedef struct fp_profile {
  double apply_ms, apply_bytes;     /* one full preconditioner application (CUDA graph) */
  int32_t apply_launches;
  double japply_ms, japply_bytes;   /* one J application */
  double fine_resid_ms, fine_resid_bytes; /* finest level: fused first Jacobi sweep + residual (BSR3) */
  double fine_post_ms, fine_post_bytes;   /* finest level: Jacobi post-smoothing sweep (BSR3) */
  double band_ms, band_bytes;       /* banded T / S~2 solve */
  double coarse_ms;                 /* dense coarse-level solve */
  int32_t n_levels;
  int32_t level_rows[32];
  int64_t level_nnz[32];
  double vcycle_ms[32];             /* V-cycle from level l down (CUDA graph); level l alone = [l] - [l+1] */
  double apply_wasted_bytes;        /* bytes one apply streams beyond apply_bytes (explicit block inverses) */
} fp_profile;
int fp_precond_profile(fp_precond* p, int32_t reps, fp_profile* out);

/* ---- solve: gmres(op, precond, b, tol, max_iter) (gmres.hpp:29-33) + GMRES(m) restart */
int fp_gmres(fp_system* s, fp_precond* p, const double* b, double* x, int32_t mem, const fp_gmres_options* opt,
             fp_solve_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* FRACPREC_B200_H */
