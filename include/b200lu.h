/* b200lu — C ABI of the B200-native (sm_100a, FP64) refactorize + solve path.
 *
 * This is the drop-in boundary for ONE path of the reference library `rlu`
 * (arXiv 2306.14337 restatement): value scatter -> pivot-free numeric
 * (re)factorization -> L/U triangular solves -> SpMV + FGMRES refinement, on a
 * fixed sparsity pattern whose symbolic analysis (AMD ordering, optional MC64
 * matching/scaling, fill pattern, scatter map) was produced by the reference's
 * own host code and is consumed here bit-exact.
 *
 * Each entry point names the reference interface it replaces. Reference paths
 * are relative to the reference tree's proj/ directory.
 *
 * Conventions
 *   - plain pointers and sizes only; int64 indices and float64 values, exactly
 *     the reference's index_t / double (include/rlu/sparse.hpp:10-11);
 *   - `on_device` != 0 means the vector/value pointers are device pointers on
 *     the handle's device (no copy); 0 means host pointers (copied on the
 *     handle's stream, the call returns after the result is on the host);
 *   - every call on one handle must be serialised by the caller (the reference
 *     contract, include/rlu/numeric.hpp:19-21); distinct handles are
 *     independent;
 *   - no device allocation happens after b200lu_create (the reference's
 *     no-allocation-after-warm-up contract, include/rlu/trisolve.hpp:31-33);
 *   - there is NO CPU fallback: without a CUDA device every compute entry
 *     point returns B200LU_NO_DEVICE.
 */
#ifndef B200LU_H
#define B200LU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct b200lu_handle b200lu_handle;

/* Mirrors the reference's exception types (include/rlu/errors.hpp:11-54). */
typedef enum {
  B200LU_OK = 0,
  B200LU_ZERO_PIVOT = 1,       /* rlu::ZeroPivotError{row}; see failed_row */
  B200LU_PATTERN_MISMATCH = 2, /* rlu::PatternMismatchError */
  B200LU_DIMENSION = 3,        /* rlu::DimensionError */
  B200LU_INVALID_FACTORS = 4,  /* rlu::Error("...: factors are not valid"), src/trisolve.cpp:20 */
  B200LU_CUDA_ERROR = 5,
  B200LU_INVALID_ARGUMENT = 6,
  B200LU_NO_DEVICE = 7,
  B200LU_ZERO_DIAGONAL = 8,         /* rlu::ZeroDiagonalError{row}, host analysis (src/symbolic.cpp:121-123) */
  B200LU_STRUCTURALLY_SINGULAR = 9  /* rlu::StructurallySingularError{deficient_rows}, host analysis (src/matching.cpp:27-31,49-52,132-143) */
} b200lu_status;

/* Borrowed, read-only image of rlu::SymbolicFactors
 * (include/rlu/symbolic.hpp:48-59). Only read during b200lu_create. */
typedef struct {
  int64_t n;
  int64_t nnz_factors;              /* combined_pattern.nnz() */
  int64_t nnz_source;               /* scatter_map.size() == nnz(A) */
  const int64_t* row_offsets;       /* combined_pattern.row_offsets, n+1 */
  const int64_t* col_indices;       /* combined_pattern.col_indices, nnz_factors */
  const int64_t* diag_pos;          /* n */
  const int64_t* scatter_map;       /* nnz_source */
  const double* scatter_scale;      /* nnz_source */
  const int64_t* amd_forward;       /* amd.forward, n */
  const int64_t* col_perm_forward;  /* match->col_perm.forward, n; NULL when match is absent */
  const double* row_scale;          /* match->scaling.row_scale, n; NULL when match is absent */
  const double* col_scale;          /* match->scaling.col_scale, n; NULL when match is absent */
  const int64_t* source_row_offsets; /* source_pattern.row_offsets, n+1 */
  const int64_t* source_col_indices; /* source_pattern.col_indices, nnz_source */
} b200lu_symbolic_view;

/* rlu::FactorOptions (include/rlu/numeric.hpp:12-15); ExecPolicy is CPU-specific and has no
 * device counterpart. */
typedef struct {
  double pivot_floor; /* |u_ii| at or below this fails the row; reference default 1e-30 */
  int device;         /* CUDA device ordinal */
  void* stream;       /* cudaStream_t to run on; NULL = the handle creates its own */
  int refine_capacity; /* largest RefineConfig.max_iterations this handle will see (Krylov storage); 0 = 20 */
  int flags;           /* B200LU_FLAG_* */
  int concurrency;     /* handles expected to run at the same time on this device (scenario batches:
                          one handle + stream per in-flight system). 0 or 1 = the handle may fill the
                          GPU. With c > 1 every persistent grid is sized to 1/c of the device and all
                          claim orders are dynamic, so kernels of different handles can share the SMs
                          in any interleaving without waiting on each other's residency. */
} b200lu_options;

/* Summation order of the triangular sweeps (lower_core / upper_core, src/trisolve.cpp:28-68).
 * The L/U values and SpMV always reproduce the reference bit for bit. By default the sweeps sum
 * each row's terms in an order chosen for the device: U rows are folded from the last column to
 * the first (the order in which their dependencies are produced), and the narrow end of the
 * dependency DAG runs inside one CTA with per-lane partial sums and a shuffle tree. That order is
 * fixed — results are deterministic — but it rounds differently from the reference's serial sum.
 * With this flag both sweeps run entirely in the sync-free kernel and fold in the reference's
 * ascending column order: lower_solve / upper_solve / solve_system are then bit-identical to the
 * CPU result, at a longer critical path. */
#define B200LU_FLAG_STRICT_ORDER 1

/* rlu::RefineConfig (include/rlu/refine.hpp:13-17) */
typedef struct {
  int max_iterations; /* default 20 */
  double tolerance;   /* default 1e-14 */
} b200lu_refine_config;

/* rlu::RefineOutcome (include/rlu/refine.hpp:19-24); x is returned through the call. */
typedef struct {
  int iterations;
  int converged;
  int history_len;
  double residual_history[66]; /* [true initial, estimates...]; capacity max_iterations+1 <= 65 */
} b200lu_refine_outcome;

/* Derived-schedule facts, for reports and the roofline arithmetic. */
typedef struct {
  int64_t n, nnz_factors, nnz_source;
  int64_t nnz_lower;        /* strict-lower slots == number of (row, pivot) pairs */
  int64_t update_pairs;     /* sum over pivots of the pivot row's upper length */
  int64_t lower_levels;     /* dependency levels of L (== levels of the factorization) */
  int64_t upper_levels;
  int64_t max_row_len;
  int64_t big_rows;         /* rows handled by the per-CTA wide slot */
  int64_t device_bytes;     /* total device memory owned by the handle */
  int64_t alloc_events;     /* device allocations performed so far (constant after create) */
  int64_t lower_tail_rows;  /* rows / levels of the L sweep handled inside one CTA (0: no split) */
  int64_t lower_tail_levels;
  int64_t upper_tail_rows;  /* same for the U sweep */
  int64_t upper_tail_levels;
} b200lu_stats;

void b200lu_default_options(b200lu_options* opt);
const char* b200lu_status_string(b200lu_status s);
const char* b200lu_last_error(const b200lu_handle* h); /* "" when none */
int b200lu_device_count(void);

/* NumericFactors::NumericFactors (src/numeric.cpp:8-12): uploads the int32 pattern, diag_pos,
 * scatter map/scale, permutations and scalings; derives the level schedules and the update
 * destination table; allocates value, solve and refinement workspaces once. */
b200lu_status b200lu_create(const b200lu_symbolic_view* sym, const b200lu_options* opt,
                            b200lu_handle** out);
void b200lu_destroy(b200lu_handle* h);

/* pattern_equal(A, sym.source_pattern) guard of scatter_values (src/numeric.cpp:15-17,
 * src/sparse.cpp pattern_equal). Host-side; returns B200LU_PATTERN_MISMATCH on any difference. */
b200lu_status b200lu_check_pattern(const b200lu_handle* h, int64_t n, const int64_t* row_offsets,
                                   const int64_t* col_indices);

/* reset_values (src/numeric.cpp:75-77) == scatter_values (14-23) without the pattern guard:
 * a_values is nnz_source doubles in source-CSR order. Also keeps A's values on the device
 * as the operator for SpMV / refinement. Leaves the factors invalid until factorized. */
b200lu_status b200lu_reset_values(b200lu_handle* h, const double* a_values, int on_device);

/* factorize_scattered (src/numeric.cpp:79 -> eliminate 27-58). On a pivot with
 * |u_ii| <= pivot_floor returns B200LU_ZERO_PIVOT and *failed_row = the lowest failing
 * row of the permuted matrix; the factors stay invalid. failed_row may be NULL. */
b200lu_status b200lu_factorize_scattered(b200lu_handle* h, int64_t* failed_row);

/* refactorize (src/numeric.cpp:70-73) == reset_values + factorize_scattered. Also serves
 * factorize (62-68) on a fresh handle. */
b200lu_status b200lu_refactorize(b200lu_handle* h, const double* a_values, int on_device,
                                 int64_t* failed_row);

/* NumericFactors::valid / generation (include/rlu/numeric.hpp:25-26). */
int b200lu_valid(const b200lu_handle* h);
uint64_t b200lu_generation(const b200lu_handle* h);

/* NumericFactors::values (include/rlu/numeric.hpp:24): nnz_factors doubles aligned to the
 * combined pattern. After reset_values and before factorization this is the scattered
 * matrix, exactly as in the reference. set_values mirrors tests that craft a factor
 * object by hand (tests/test_trisolve.cpp:171-184). */
b200lu_status b200lu_get_values(b200lu_handle* h, double* host_out);
b200lu_status b200lu_set_values(b200lu_handle* h, const double* host_in, int valid);
/* Device pointer to the factor values (borrowed; valid while the handle lives). */
const double* b200lu_values_device(const b200lu_handle* h);

/* lower_solve / upper_solve (src/trisolve.cpp:72-88 -> lower_core 28-42, upper_core 46-68),
 * in the permuted space. `len` is checked against n (DimensionError). upper_solve reports an
 * exactly zero diagonal as B200LU_ZERO_PIVOT with *failed_row = that row. */
b200lu_status b200lu_lower_solve(b200lu_handle* h, int64_t len, const double* y, double* x,
                                 int on_device);
b200lu_status b200lu_upper_solve(b200lu_handle* h, int64_t len, const double* y, double* x,
                                 int on_device, int64_t* failed_row);

/* solve_system (src/trisolve.cpp:90-119): x = D_c Q P^T U^-1 L^-1 P D_r b. */
b200lu_status b200lu_solve(b200lu_handle* h, int64_t len, const double* b, double* x,
                           int on_device, int64_t* failed_row);

/* spmv (src/sparse.cpp:128-143) and relative_residual (283-288) with A = the matrix whose
 * values were last given to reset_values/refactorize. */
b200lu_status b200lu_spmv(b200lu_handle* h, const double* x, double* y, int on_device);
b200lu_status b200lu_relative_residual(b200lu_handle* h, const double* x, const double* b,
                                       int on_device, double* out);

/* fgmres_refine (src/refine.cpp:39-142) with A as above and the preconditioner
 * solve_system(factors, .) — the pairing cli::solve_sequence uses (src/cli.cpp:121-135).
 * use_preconditioner == 0 selects the identity operator (tests/test_refine.cpp:31).
 * x0 and x_out may alias. Never fails for non-convergence (include/rlu/refine.hpp:41-42). */
b200lu_status b200lu_refine_fgmres(b200lu_handle* h, const double* b, const double* x0,
                                   double* x_out, int on_device, int use_preconditioner,
                                   const b200lu_refine_config* cfg, b200lu_refine_outcome* outcome);

/* classic_refine (src/refine.cpp:150-188). */
b200lu_status b200lu_refine_classic(b200lu_handle* h, const double* b, const double* x0,
                                    double* x_out, int on_device, int use_preconditioner,
                                    const b200lu_refine_config* cfg, b200lu_refine_outcome* outcome);

/* cgs2_orthonormalize (include/rlu/refine.hpp:25-35, src/refine.cpp:8-26): two full Gram-Schmidt passes of
 * v against the k orthonormal vectors basis[j] ([k][n], contiguous), then normalisation. coefficients_out[k]
 * (host): the combined projection coefficients; vector_out[n]: the normalised remainder (the unnormalised one
 * on breakdown); *norm_out: the remainder's norm before normalisation; *breakdown_out: 1 when that norm is at
 * most 1e-300. k may not exceed the handle's refine_capacity. basis / v / vector_out are host or device
 * pointers as `on_device` says. */
b200lu_status b200lu_cgs2_orthonormalize(b200lu_handle* h, int64_t k, const double* basis, const double* v,
                                         int on_device, double* coefficients_out, double* vector_out,
                                         double* norm_out, int* breakdown_out);

b200lu_status b200lu_get_stats(const b200lu_handle* h, b200lu_stats* out);
/* Host-only (needs no device): validates a symbolic view and derives the device schedule the
 * way b200lu_create does — the level orders that replace SyncFreeScheduler's ascending claim
 * order (include/rlu/schedule.hpp:49-79) and the per-row update-pair offsets. Any of the three
 * output arrays may be NULL. lower_order / upper_order: n int32; pair_row_ptr: n+1 int64. */
b200lu_status b200lu_schedule_probe(const b200lu_symbolic_view* sym, b200lu_stats* stats,
                                    int32_t* lower_order, int32_t* upper_order,
                                    int64_t* pair_row_ptr, char* error_buf, int error_buf_len);
/* Optional device-side phase timing: CUDA events recorded on the handle's stream around each
 * kernel, the counterpart of the steady_clock phase timers of cli::solve_sequence
 * (src/cli.cpp:105-132; fields scatter_ms / factor_ms / trisolve_ms / refine_ms of
 * SystemRecord, include/rlu/report.hpp:19-22). ms_out / count_out hold B200LU_NUM_PHASES
 * entries: accumulated kernel milliseconds and launch counts per phase since the last reset. */
enum {
  B200LU_PHASE_SCATTER = 0, /* K1 */
  B200LU_PHASE_FACTOR = 1,  /* K2 */
  B200LU_PHASE_LOWER = 2,   /* K3, L sweep */
  B200LU_PHASE_UPPER = 3,   /* K3, U sweep */
  B200LU_PHASE_PERMUTE = 4, /* solve_system prologue / epilogue */
  B200LU_PHASE_SPMV = 5,    /* K4: SpMV / fused residual */
  B200LU_PHASE_VECTOR = 6,  /* K4: dot, projection, axpy, scale */
  B200LU_PHASE_TAIL = 7,    /* K3: the narrow end of either sweep inside one cluster (default mode) */
  B200LU_NUM_PHASES = 8
};
b200lu_status b200lu_set_timing(b200lu_handle* h, int enabled);
b200lu_status b200lu_get_phase_times(b200lu_handle* h, double* ms_out, int64_t* count_out, int reset);
/* Number of kernels this handle has launched since creation (bench.py's gpu_launches). */
uint64_t b200lu_launch_count(const b200lu_handle* h);
/* Blocks until everything queued on the handle's stream has finished. */
b200lu_status b200lu_synchronize(b200lu_handle* h);

/* Device-resident KKT values. assemble_kkt (src/kkt.cpp:53-77) builds
 * K = [[H + D_y + delta_p I, J^T], [J, -delta_d I]]; across a barrier sequence, and under the
 * regularization escalation of cli::solve_sequence (src/cli.cpp:148-154: doubled deltas, same
 * pattern), only K's diagonal changes. After one reset_values / refactorize with the full values,
 * b200lu_kkt_update rewrites the diagonal on the device exactly as the reference sums it —
 * K_ii = H_ii + (D_y[i] + delta_p) for the n_primal primal rows, -delta_d for the dual rows — and
 * scatters, i.e. it replaces reset_values for the next system: 8*n_primal bytes cross the bus
 * instead of 8*nnz(K), none if D_y already lives on the device. Follow with
 * b200lu_factorize_scattered. h_diag: H's own diagonal values (0 where H has none), n_primal
 * doubles; diag_source_pos: position of K_ii in source-CSR order, n entries. */
b200lu_status b200lu_kkt_bind(b200lu_handle* h, int64_t n_primal, const double* h_diag,
                              const int64_t* diag_source_pos);
b200lu_status b200lu_kkt_update(b200lu_handle* h, const double* d_y, int on_device, double delta_p,
                                double delta_d);

/* ------------------------------------------------------------------------------------------
 * Scenario batches (BASELINE config "batch of 256 independent scenario systems"):
 * `batch` independent systems that share ONE symbolic analysis (same pattern, different values
 * and right-hand sides), factorized and solved together. The reference has no batched entry
 * point — cli::solve_sequence (src/cli.cpp:80-135) runs its systems one after another through
 * the same four calls; each b200lu_batch_* function below is the corresponding single-system
 * call applied to every scenario, with every scenario's arithmetic performed entry by entry in
 * the reference's order: per-scenario L/U values, lower/upper/solve_system results and SpMV are
 * bit-identical to the single-system CPU results.
 *
 * Array conventions: value arrays are [batch][nnz_source], vectors are [batch][n], both
 * scenario-major and contiguous (scenario s starts at s * nnz_source resp. s * n); host or
 * device pointers as selected by `on_device`. Per-scenario outputs (failed_rows, residuals,
 * outcomes) hold `batch` entries. Internally every array is stored scenario-interleaved in
 * groups of 32. */
typedef struct b200lu_batch b200lu_batch;

typedef struct {
  int64_t batch, padded_batch;
  int64_t unit_scenarios; /* scenarios a refactorization warp handles at once: 32, one lane per scenario */
  int64_t blocks;         /* row blocks of the trailing part of the refactorization (kBlockRows rows each) */
  int64_t factor_rows;    /* rows with at least one pivot */
  int64_t blocked_rows, blocked_pairs; /* of those, rows (and their update pairs) handled in row blocks */
  int64_t factor_grid, tri_grid;
  int64_t n, nnz_factors, nnz_source, update_pairs, lower_levels, upper_levels;
  int64_t device_bytes, alloc_events, launches;
  /* tiled trailing part (csrc/tile.cuh): rows resident in shared memory, pivot rows streamed by TMA */
  int64_t tiled;                /* 1: the trailing part runs in the tiled kernel (then `blocks` counts tiles) */
  int64_t tile_rows;            /* rows (consumer warps) per tile */
  int64_t tile_smem_bytes, tile_grid;
  int64_t tile_fetched_entries; /* pivot-row entries TMA fetches per 8-scenario unit (x 64 bytes) */
} b200lu_batch_info;

/* NumericFactors::NumericFactors (src/numeric.cpp:8-12) for `batch` systems at once. Only
 * pivot_floor, device, stream and refine_capacity of `opt` are used. */
b200lu_status b200lu_batch_create(const b200lu_symbolic_view* sym, const b200lu_options* opt,
                                  int64_t batch, b200lu_batch** out);
void b200lu_batch_destroy(b200lu_batch* h);
const char* b200lu_batch_last_error(const b200lu_batch* h);
/* pattern_equal guard (src/numeric.cpp:15-17), as b200lu_check_pattern. */
b200lu_status b200lu_batch_check_pattern(const b200lu_batch* h, int64_t n, const int64_t* row_offsets,
                                         const int64_t* col_indices);
/* reset_values / factorize_scattered / refactorize (src/numeric.cpp:70-79) per scenario.
 * failed_rows (may be NULL): per scenario the lowest failing permuted row, -1 when the scenario
 * factorized. Returns B200LU_ZERO_PIVOT when any scenario failed; the others are valid. */
b200lu_status b200lu_batch_reset_values(b200lu_batch* h, const double* a_values, int on_device);
b200lu_status b200lu_batch_factorize_scattered(b200lu_batch* h, int64_t* failed_rows);
b200lu_status b200lu_batch_refactorize(b200lu_batch* h, const double* a_values, int on_device,
                                       int64_t* failed_rows);
int b200lu_batch_valid(const b200lu_batch* h, int64_t scenario);
/* NumericFactors::values of one scenario (nnz_factors doubles, host). */
b200lu_status b200lu_batch_get_values(b200lu_batch* h, int64_t scenario, double* host_out);
/* lower_solve / upper_solve / solve_system (src/trisolve.cpp:72-119) per scenario. Results of
 * scenarios whose factorization failed are unspecified. */
b200lu_status b200lu_batch_lower_solve(b200lu_batch* h, const double* y, double* x, int on_device);
b200lu_status b200lu_batch_upper_solve(b200lu_batch* h, const double* y, double* x, int on_device,
                                       int64_t* failed_rows);
b200lu_status b200lu_batch_solve(b200lu_batch* h, const double* b, double* x, int on_device,
                                 int64_t* failed_rows);
/* relative_residual (src/sparse.cpp:283-288) per scenario; out holds `batch` doubles (host). */
b200lu_status b200lu_batch_relative_residual(b200lu_batch* h, const double* x, const double* b,
                                             int on_device, double* out);
/* fgmres_refine (src/refine.cpp:39-142) per scenario, all scenarios advancing in lockstep;
 * outcomes holds `batch` entries. */
b200lu_status b200lu_batch_refine_fgmres(b200lu_batch* h, const double* b, const double* x0,
                                         double* x_out, int on_device, int use_preconditioner,
                                         const b200lu_refine_config* cfg,
                                         b200lu_refine_outcome* outcomes);
/* classic_refine (src/refine.cpp:150-188) per scenario. */
b200lu_status b200lu_batch_refine_classic(b200lu_batch* h, const double* b, const double* x0,
                                          double* x_out, int on_device, int use_preconditioner,
                                          const b200lu_refine_config* cfg,
                                          b200lu_refine_outcome* outcomes);
/* b200lu_kkt_bind / b200lu_kkt_update for every scenario: d_y is [batch][n_primal]; H, J and the
 * deltas are shared (scenarios of one network differ in their barrier diagonal and right-hand side). */
b200lu_status b200lu_batch_kkt_bind(b200lu_batch* h, int64_t n_primal, const double* h_diag,
                                    const int64_t* diag_source_pos);
b200lu_status b200lu_batch_kkt_update(b200lu_batch* h, const double* d_y, int on_device, double delta_p,
                                      double delta_d);
/* Staged (pipelined) submission for a SEQUENCE of batches, the device-side shape of cli::solve_sequence's
 * loop (src/cli.cpp:80-135): while batch k is factorized and solved, the inputs of batch k + 1 cross the bus
 * on a dedicated copy stream into the staging buffer that is not in use, and the solutions of batch k leave on
 * a third stream. Host buffers should be page-locked (cudaHostRegister / pinned allocation) for the copies
 * to overlap; every buffer of these calls (values, right-hand sides, host_x_out) may also be memory of the handle's
 * device, in which case the copies are device-to-device (a caller that keeps its systems in HBM gets the same
 * submission without a host round trip between the steps). Typical loop:
 *     stage_inputs(v[0], b[0]);
 *     for k: if (k + 1 < K) stage_inputs(v[k+1], b[k+1]); refactorize_staged(); solve_refine_staged(.., x[k], ..);
 *     staged_wait();                  // x[k] may be read only after staged_wait (or after the next-but-one call)
 * Staged inputs are consumed in the order they were staged (two staging sets: at most two batches may be
 * staged and unconsumed; a third stage_inputs is refused).
 * stage_inputs: [batch][nnz_source] values and/or [batch][n] right-hand sides (either may be NULL to keep the
 * previous one); returns at once. refactorize_staged = reset_values + factorize_scattered on the staged values
 * (src/numeric.cpp:70-79). solve_refine_staged = solve_system (src/trisolve.cpp:90-119) on the staged
 * right-hand sides, then fgmres_refine (src/refine.cpp:39-142) from that solution when `refine` != 0; the result
 * is copied to host_x_out asynchronously. The second staging set (one more copy of the values, right-hand
 * sides and solutions on the device) is allocated by the first stage_inputs call. */
b200lu_status b200lu_batch_stage_inputs(b200lu_batch* h, const double* host_values, const double* host_rhs);
b200lu_status b200lu_batch_refactorize_staged(b200lu_batch* h, int64_t* failed_rows);
b200lu_status b200lu_batch_solve_refine_staged(b200lu_batch* h, int refine, const b200lu_refine_config* cfg,
                                               double* host_x_out, b200lu_refine_outcome* outcomes,
                                               int64_t* failed_rows);
b200lu_status b200lu_batch_staged_wait(b200lu_batch* h);
b200lu_status b200lu_batch_get_info(const b200lu_batch* h, b200lu_batch_info* out);

/* Diagnostics — HOST ONLY, needs no device; not on any product path. Builds the tile plan the batched
 * refactorization derives for the trailing rows of the pattern (rows_per_tile rows and tile_entries
 * row entries of shared memory per tile, trailing part = the levels narrower than tail_width rows) and
 * executes that plan for ONE scenario on the host with the index arithmetic of the device kernel:
 * `values` holds the scattered matrix (scatter_values, src/numeric.cpp:14-23) on entry and the factors
 * on return; the arithmetic is eliminate's (src/numeric.cpp:34-49). The CPU tests compare the result
 * with the oracle bit for bit, which pins the plan (tiling, pivot merge, chunking, claim order) without
 * a GPU. Returns B200LU_ZERO_PIVOT with *failed_row as eliminate would. */
typedef struct {
  int64_t tiles, rows, items;
  int64_t pairs;                /* update pairs of the tiled rows */
  int64_t fetched_entries;      /* pivot-row entries fetched per unit (each pivot row once per tile) */
  int64_t consumed_entries;     /* the same entries counted once per consuming row (= no sharing) */
  int64_t largest_tile_entries;
} b200lu_tile_plan_stats;
b200lu_status b200lu_tile_plan_emulate(const b200lu_symbolic_view* sym, int rows_per_tile, int64_t tile_entries,
                                       int64_t tail_width, double pivot_floor, double* values, int64_t* failed_row,
                                       b200lu_tile_plan_stats* stats, char* error_buf, int error_buf_len);
/* Diagnostics: the 16 phase counters (clock cycles summed over warps) of the tiled refactorization kernel;
 * all zero unless the library was built with -DB200LU_TILE_PROF (csrc/tile.cuh lists the phases). */
b200lu_status b200lu_batch_tile_profile(b200lu_batch* h, int64_t* cycles_out, int reset);
b200lu_status b200lu_batch_set_timing(b200lu_batch* h, int enabled);
b200lu_status b200lu_batch_get_phase_times(b200lu_batch* h, double* ms_out, int64_t* count_out, int reset);
b200lu_status b200lu_batch_synchronize(b200lu_batch* h);

/* ---- Host-side symbolic analysis --------------------------------------------------------
 * rlu::symbolic_analyze(A, AnalyzeOptions{use_scaling, use_amd}) (include/rlu/symbolic.hpp:67-75,
 * src/symbolic.cpp:156-203) with mc64_scale (src/matching.cpp:17-189), amd_order (src/ordering.cpp:9-122) and
 * fill1_pattern (src/symbolic.cpp:95-154): the same permutations, scale factors, combined L+U pattern, diag_pos
 * and scatter map BIT FOR BIT, from algorithms whose cost follows the size of the result (csrc/analyze.cpp).
 * Host code only: no device is needed or used. `values` (nnz doubles, source order) is read only when
 * use_scaling != 0. On every return with *out != NULL the object must be destroyed; when the status is not OK
 * it carries the error (b200lu_analysis_status / _message) and no product. RowLookupTable, the CPU
 * elimination's per-row hash/bitmap, is not part of the product: the device path does not use it. */
typedef struct b200lu_analysis b200lu_analysis;
b200lu_status b200lu_analyze(int64_t n, const int64_t* row_offsets, const int64_t* col_indices, const double* values,
                             int use_scaling, int use_amd, b200lu_analysis** out);
/* Status of the analysis; failed_row = ZeroDiagonalError::row (a row of the permuted matrix B, as the
 * reference reports it) or the first deficient row; deficient_rows = StructurallySingularError::deficient_rows
 * (borrowed, sorted). Any out pointer may be NULL. */
b200lu_status b200lu_analysis_status(const b200lu_analysis* a, int64_t* failed_row, const int64_t** deficient_rows,
                                     int64_t* deficient_count);
const char* b200lu_analysis_message(const b200lu_analysis* a);
/* The product as the view b200lu_create / b200lu_batch_create consume; pointers are borrowed from the
 * analysis object. fill_count (may be NULL) = SymbolicFactors::fill_count. */
b200lu_status b200lu_analysis_view(const b200lu_analysis* a, b200lu_symbolic_view* view, int64_t* fill_count);
/* Host milliseconds spent in {matching, ordering, permutation, fill pattern, scatter map, total};
 * matched_product (may be NULL) = MatchingResult::matched_product. */
b200lu_status b200lu_analysis_times(const b200lu_analysis* a, double* ms_out6, double* matched_product);
void b200lu_analysis_destroy(b200lu_analysis* a);

#ifdef __cplusplus
}
#endif
#endif /* B200LU_H */
