/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C CPU restatement of the reference hot path (rlu, arXiv 2306.14337):
 * value scatter -> pivot-free up-looking LU -> unit-L / U triangular solves ->
 * SpMV + flexible-GMRES refinement. Every function cites the reference
 * file:line it restates (paths relative to /root/reference/proj).
 *
 * Parity status: PINNED. tests/test_oracle_vs_reference.py checks every
 * function here bit-for-bit against the unmodified reference
 * (oracle/_ref/librlu_ref.so) on seeded inputs, and tests/test_oracle_golden.py
 * checks it against the reference tests' known answers and the committed
 * fixtures under tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * link or load this library; the CUDA product path never does.
 */
#ifndef RLU_ORACLE_H
#define RLU_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  RLO_OK = 0,
  RLO_ZERO_PIVOT = 1,
  RLO_DIMENSION = 3,
  RLO_ERROR = 4
};

/* Combined L+U pattern of SymbolicFactors (include/rlu/symbolic.hpp:48-59):
 * strict-lower slots of row i are L, diag_pos[i] and beyond are U. */
typedef struct {
  int64_t n;
  const int64_t* row_offsets; /* n+1 */
  const int64_t* col_indices; /* nnzF, strictly increasing per row */
  const int64_t* diag_pos;    /* n, global offset of (i,i) */
} rlo_pattern;

/* The transform stages of solve_system (src/trisolve.cpp:90-119). col_perm,
 * row_scale and col_scale are all NULL when analysis ran without matching. */
typedef struct {
  const int64_t* amd_forward;      /* n */
  const int64_t* col_perm_forward; /* n or NULL */
  const double* row_scale;         /* n or NULL */
  const double* col_scale;         /* n or NULL */
} rlo_transform;

typedef struct {
  int64_t n;
  const int64_t* row_offsets;
  const int64_t* col_indices;
  const double* values;
} rlo_csr;

/* src/numeric.cpp:14-23 (pattern guard excluded: it is host logic of the caller). */
void rlo_scatter_values(int64_t nnz_factors, int64_t nnz_source, const int64_t* scatter_map,
                        const double* scatter_scale, const double* a_values, double* out);

/* src/numeric.cpp:27-58, sequential mode. `colpos` is caller scratch of n int64.
 * Returns RLO_ZERO_PIVOT and the lowest failing row when |u_ii| <= pivot_floor. */
int rlo_eliminate(const rlo_pattern* F, double* values, double pivot_floor, int64_t* colpos,
                  int64_t* failed_row);

/* src/trisolve.cpp:28-42. Safe in place. */
void rlo_lower_solve(const rlo_pattern* F, const double* values, const double* y, double* x);

/* src/trisolve.cpp:46-68. Exact-zero diagonal -> RLO_ZERO_PIVOT + row. */
int rlo_upper_solve(const rlo_pattern* F, const double* values, const double* y, double* x,
                    int64_t* failed_row);

/* src/trisolve.cpp:90-119. w1, w2: caller scratch of n doubles. */
int rlo_solve_system(const rlo_pattern* F, const double* values, const rlo_transform* T,
                     const double* b, double* x, double* w1, double* w2, int64_t* failed_row);

/* src/sparse.cpp:128-143, 271-288. */
void rlo_spmv(const rlo_csr* A, const double* x, double* y);
double rlo_dot(int64_t n, const double* a, const double* b);
double rlo_norm2(int64_t n, const double* a);
void rlo_axpy(int64_t n, double alpha, const double* x, double* y);
double rlo_relative_residual(const rlo_csr* A, const double* x, const double* b);

/* src/refine.cpp:8-26. basis: k row-major n-vectors. coefficients: k. vec: n (in/out). */
void rlo_cgs2(int64_t n, int64_t k, const double* basis, double* vec, double* coefficients,
              double* norm, int* breakdown);

/* Preconditioner = solve_system with the given factors, or the identity when F == NULL. */
typedef struct {
  const rlo_pattern* F;
  const double* values;
  const rlo_transform* T;
} rlo_precond;

/* src/refine.cpp:39-142 (fgmres_refine) / 150-188 (classic_refine).
 * history must hold max(1,max_iterations)+2 doubles. */
int rlo_fgmres(const rlo_csr* A, const double* b, const double* x0, const rlo_precond* M,
               int max_iterations, double tolerance, double* x_out, int* iterations,
               int* converged, double* history, int* history_len);
int rlo_classic_refine(const rlo_csr* A, const double* b, const double* x0, const rlo_precond* M,
                       int max_iterations, double tolerance, double* x_out, int* iterations,
                       int* converged, double* history, int* history_len);

#ifdef __cplusplus
}
#endif
#endif
