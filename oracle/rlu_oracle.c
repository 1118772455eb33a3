/* TEST INFRASTRUCTURE — NOT PRODUCT CODE. See rlu_oracle.h for the contract.
 *
 * Compiled with -ffp-contract=off: the reference's baseline x86-64 build emits
 * separate multiply and subtract, and every comparison against it is bitwise.
 */
#include "rlu_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ scatter */

/* src/numeric.cpp:19-22: out.assign(nnzF, 0); out[map[k]] = A.values[k] * scale[k]. */
void rlo_scatter_values(int64_t nnz_factors, int64_t nnz_source, const int64_t* scatter_map,
                        const double* scatter_scale, const double* a_values, double* out) {
  for (int64_t s = 0; s < nnz_factors; ++s) out[s] = 0.0;
  for (int64_t k = 0; k < nnz_source; ++k) out[scatter_map[k]] = a_values[k] * scatter_scale[k];
}

/* ---------------------------------------------------------------- eliminate */

/* src/numeric.cpp:34-49, one row at a time in ascending order (the sequential
 * branch of SyncFreeScheduler::run, include/rlu/schedule.hpp:54-58).
 *
 * The reference resolves "where does column j live in row i" with a per-row
 * bitmap/hash (src/symbolic.cpp:73-93); here a dense column->offset scratch
 * plays that role. The arithmetic and its order are unchanged: for each
 * strict-lower column d ascending, alpha = a_id / u_dd, then every upper entry
 * of row d is multiplied by alpha and subtracted from row i. */
int rlo_eliminate(const rlo_pattern* F, double* values, double pivot_floor, int64_t* colpos,
                  int64_t* failed_row) {
  const int64_t n = F->n;
  int64_t failed = -1;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lo = F->row_offsets[i], hi = F->row_offsets[i + 1];
    const int64_t diag = F->diag_pos[i];
    for (int64_t k = lo; k < hi; ++k) colpos[F->col_indices[k]] = k;
    for (int64_t k = lo; k < diag; ++k) {
      const int64_t d = F->col_indices[k];
      const double alpha = values[k] / values[F->diag_pos[d]];
      values[k] = alpha;
      for (int64_t t = F->diag_pos[d] + 1; t < F->row_offsets[d + 1]; ++t) {
        const int64_t slot = colpos[F->col_indices[t]];
        const double prod = alpha * values[t];
        values[slot] = values[slot] - prod;
      }
    }
    /* src/numeric.cpp:48 + schedule.hpp:82-87: lowest failing row wins; the row
     * still completes so later rows run on poisoned values. */
    if (fabs(values[diag]) <= pivot_floor && failed < 0) failed = i;
  }
  if (failed_row) *failed_row = failed;
  return failed >= 0 ? RLO_ZERO_PIVOT : RLO_OK;
}

/* ---------------------------------------------------------- triangular solves */

/* src/trisolve.cpp:33-41 */
void rlo_lower_solve(const rlo_pattern* F, const double* values, const double* y, double* x) {
  for (int64_t i = 0; i < F->n; ++i) {
    double acc = y[i];
    for (int64_t k = F->row_offsets[i]; k < F->diag_pos[i]; ++k) {
      const double prod = values[k] * x[F->col_indices[k]];
      acc = acc - prod;
    }
    x[i] = acc;
  }
}

/* src/trisolve.cpp:52-67 */
int rlo_upper_solve(const rlo_pattern* F, const double* values, const double* y, double* x,
                    int64_t* failed_row) {
  const int64_t n = F->n;
  int64_t failed_v = -1; /* virtual index n-1-i; lowest virtual == highest row */
  for (int64_t v = 0; v < n; ++v) {
    const int64_t i = n - 1 - v;
    double acc = y[i];
    for (int64_t k = F->diag_pos[i] + 1; k < F->row_offsets[i + 1]; ++k) {
      const double prod = values[k] * x[F->col_indices[k]];
      acc = acc - prod;
    }
    const double diag = values[F->diag_pos[i]];
    if (diag == 0.0 && failed_v < 0) failed_v = v;
    x[i] = acc / diag;
  }
  if (failed_v >= 0) {
    if (failed_row) *failed_row = n - 1 - failed_v;
    return RLO_ZERO_PIVOT;
  }
  if (failed_row) *failed_row = -1;
  return RLO_OK;
}

/* src/trisolve.cpp:96-118 */
int rlo_solve_system(const rlo_pattern* F, const double* values, const rlo_transform* T,
                     const double* b, double* x, double* w1, double* w2, int64_t* failed_row) {
  const int64_t n = F->n;
  const int64_t* p = T->amd_forward;
  if (T->col_perm_forward) {
    for (int64_t i = 0; i < n; ++i) w1[p[i]] = T->row_scale[i] * b[i];
  } else {
    for (int64_t i = 0; i < n; ++i) w1[p[i]] = b[i];
  }
  rlo_lower_solve(F, values, w1, w2);
  const int st = rlo_upper_solve(F, values, w2, w1, failed_row);
  if (st != RLO_OK) return st;
  if (T->col_perm_forward) {
    const int64_t* q = T->col_perm_forward;
    for (int64_t j = 0; j < n; ++j) x[j] = T->col_scale[j] * w1[p[q[j]]];
  } else {
    for (int64_t j = 0; j < n; ++j) x[j] = w1[p[j]];
  }
  return RLO_OK;
}

/* -------------------------------------------------------------- sparse BLAS */

/* src/sparse.cpp:135-141 */
void rlo_spmv(const rlo_csr* A, const double* x, double* y) {
  for (int64_t i = 0; i < A->n; ++i) {
    double acc = 0.0;
    for (int64_t k = A->row_offsets[i]; k < A->row_offsets[i + 1]; ++k) {
      const double prod = A->values[k] * x[A->col_indices[k]];
      acc = acc + prod;
    }
    y[i] = acc;
  }
}

/* src/sparse.cpp:271-275 */
double rlo_dot(int64_t n, const double* a, const double* b) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double prod = a[i] * b[i];
    acc = acc + prod;
  }
  return acc;
}

/* src/sparse.cpp:277 */
double rlo_norm2(int64_t n, const double* a) { return sqrt(rlo_dot(n, a, a)); }

/* src/sparse.cpp:279-281 */
void rlo_axpy(int64_t n, double alpha, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) {
    const double prod = alpha * x[i];
    y[i] = y[i] + prod;
  }
}

/* src/sparse.cpp:283-288 */
double rlo_relative_residual(const rlo_csr* A, const double* x, const double* b) {
  const int64_t n = A->n;
  double* r = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  rlo_spmv(A, x, r);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  const double bn = rlo_norm2(n, b);
  const double res = rlo_norm2(n, r) / (bn > 0.0 ? bn : 1.0);
  free(r);
  return res;
}

/* --------------------------------------------------------------- refinement */

/* src/refine.cpp:8-26. Two passes; inside a pass each basis vector is
 * projected out immediately after its coefficient is taken (dot, then axpy). */
void rlo_cgs2(int64_t n, int64_t k, const double* basis, double* vec, double* coefficients,
              double* norm, int* breakdown) {
  for (int64_t j = 0; j < k; ++j) coefficients[j] = 0.0;
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t j = 0; j < k; ++j) {
      const double* q = basis + j * n;
      const double h = rlo_dot(n, q, vec);
      coefficients[j] += h;
      rlo_axpy(n, -h, q, vec);
    }
  }
  *norm = rlo_norm2(n, vec);
  if (*norm <= 1e-300) {
    *breakdown = 1;
    return;
  }
  *breakdown = 0;
  for (int64_t i = 0; i < n; ++i) vec[i] /= *norm;
}

static void apply_precond(const rlo_precond* M, int64_t n, const double* in, double* out,
                          double* w1, double* w2) {
  if (M && M->F) {
    int64_t failed;
    rlo_solve_system(M->F, M->values, M->T, in, out, w1, w2, &failed);
  } else {
    memcpy(out, in, sizeof(double) * (size_t)n);
  }
}

/* src/refine.cpp:30-35 */
static double true_relres(const rlo_csr* A, const double* b, const double* x, double bnorm,
                          double* scratch) {
  rlo_spmv(A, x, scratch);
  for (int64_t i = 0; i < A->n; ++i) scratch[i] = b[i] - scratch[i];
  return rlo_norm2(A->n, scratch) / bnorm;
}

/* src/refine.cpp:39-142 */
int rlo_fgmres(const rlo_csr* A, const double* b, const double* x0, const rlo_precond* M,
               int max_iterations, double tolerance, double* x_out, int* iterations,
               int* converged, double* history, int* history_len) {
  const int64_t n = A->n;
  const size_t nb = sizeof(double) * (size_t)(n > 0 ? n : 1);
  const int m = max_iterations > 1 ? max_iterations : 1;
  const double bn = rlo_norm2(n, b);
  const double bnorm = bn > 0.0 ? bn : 1.0;
  int hl = 0;

  *iterations = 0;
  *converged = 0;
  memcpy(x_out, x0, sizeof(double) * (size_t)n);

  double* r = (double*)malloc(nb);
  rlo_spmv(A, x0, r);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  const double beta = rlo_norm2(n, r);
  double best_res = beta / bnorm;
  history[hl++] = best_res;
  if (best_res <= tolerance) {
    *converged = 1;
    *history_len = hl;
    free(r);
    return RLO_OK;
  }

  double* V = (double*)malloc(nb * (size_t)(m + 1)); /* orthonormal basis, row-major */
  double* Z = (double*)malloc(nb * (size_t)m);       /* preconditioned vectors */
  int nV = 0;
  for (int64_t i = 0; i < n; ++i) V[i] = r[i] / beta;
  nV = 1;

  /* Column-major Hessenberg after rotations: H[col] has col+2 entries. */
  double* H = (double*)calloc((size_t)m * (size_t)(m + 2), sizeof(double));
  double* g = (double*)calloc((size_t)m + 1, sizeof(double));
  double* cs = (double*)calloc((size_t)m, sizeof(double));
  double* sn = (double*)calloc((size_t)m, sizeof(double));
  double* hcol = (double*)calloc((size_t)m + 2, sizeof(double));
  double* yv = (double*)calloc((size_t)m, sizeof(double));
  double* w = (double*)malloc(nb);
  double* scratch = (double*)malloc(nb);
  double* candidate = (double*)malloc(nb);
  double* w1 = (double*)malloc(nb);
  double* w2 = (double*)malloc(nb);
  g[0] = beta;
  double accept_below = tolerance * bnorm;

  for (int i = 0; i < m; ++i) {
    double* zi = Z + (size_t)i * (size_t)n;
    apply_precond(M, n, V + (size_t)i * (size_t)n, zi, w1, w2);
    rlo_spmv(A, zi, w);

    double norm;
    int breakdown;
    rlo_cgs2(n, nV, V, w, hcol, &norm, &breakdown);
    const int ncoef = nV; /* == i + 1 unless an earlier breakdown ended the loop */
    hcol[ncoef] = breakdown ? 0.0 : norm;
    if (!breakdown) {
      memcpy(V + (size_t)nV * (size_t)n, w, sizeof(double) * (size_t)n);
      ++nV;
    }

    for (int k = 0; k < i; ++k) {
      const double t = hcol[k];
      hcol[k] = cs[k] * t + sn[k] * hcol[k + 1];
      hcol[k + 1] = -sn[k] * t + cs[k] * hcol[k + 1];
    }
    const double hii = hcol[i], hsub = hcol[i + 1];
    const double gam = hypot(hii, hsub);
    if (gam == 0.0) {
      cs[i] = 1.0;
      sn[i] = 0.0;
    } else {
      cs[i] = hii / gam;
      sn[i] = hsub / gam;
    }
    hcol[i] = gam;
    hcol[i + 1] = 0.0;
    const double gi = g[i];
    g[i] = cs[i] * gi;
    g[i + 1] = -sn[i] * gi;
    memcpy(H + (size_t)i * (size_t)(m + 2), hcol, sizeof(double) * (size_t)(i + 2));

    *iterations = i + 1;
    const double estimate = fabs(g[i + 1]);
    history[hl++] = estimate / bnorm;

    const int last = breakdown || i == m - 1;
    if (estimate <= accept_below || last) {
      const int its = *iterations;
      for (int row = its - 1; row >= 0; --row) {
        double t = g[row];
        for (int col = row + 1; col < its; ++col) t -= H[(size_t)col * (size_t)(m + 2) + row] * yv[col];
        yv[row] = t / H[(size_t)row * (size_t)(m + 2) + row];
      }
      memcpy(candidate, x0, sizeof(double) * (size_t)n);
      for (int col = 0; col < its; ++col) rlo_axpy(n, yv[col], Z + (size_t)col * (size_t)n, candidate);

      const double res = true_relres(A, b, candidate, bnorm, scratch);
      if (res < best_res) {
        best_res = res;
        memcpy(x_out, candidate, sizeof(double) * (size_t)n);
      }
      if (best_res <= tolerance) {
        *converged = 1;
        break;
      }
      if (last) break;
      accept_below = estimate * 0.5;
    }
  }

  *history_len = hl;
  free(r); free(V); free(Z); free(H); free(g); free(cs); free(sn); free(hcol); free(yv);
  free(w); free(scratch); free(candidate); free(w1); free(w2);
  return RLO_OK;
}

/* src/refine.cpp:150-188 */
int rlo_classic_refine(const rlo_csr* A, const double* b, const double* x0, const rlo_precond* M,
                       int max_iterations, double tolerance, double* x_out, int* iterations,
                       int* converged, double* history, int* history_len) {
  const int64_t n = A->n;
  const size_t nb = sizeof(double) * (size_t)(n > 0 ? n : 1);
  const double bn = rlo_norm2(n, b);
  const double bnorm = bn > 0.0 ? bn : 1.0;
  int hl = 0;
  *iterations = 0;
  *converged = 0;
  memcpy(x_out, x0, sizeof(double) * (size_t)n);

  double best_res = rlo_relative_residual(A, x0, b);
  history[hl++] = best_res;
  if (best_res <= tolerance) {
    *converged = 1;
    *history_len = hl;
    return RLO_OK;
  }
  double* x = (double*)malloc(nb);
  double* r = (double*)malloc(nb);
  double* d = (double*)malloc(nb);
  double* w1 = (double*)malloc(nb);
  double* w2 = (double*)malloc(nb);
  memcpy(x, x0, sizeof(double) * (size_t)n);
  for (int it = 0; it < max_iterations; ++it) {
    rlo_spmv(A, x, r);
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    apply_precond(M, n, r, d, w1, w2);
    rlo_axpy(n, 1.0, d, x);
    *iterations = it + 1;

    rlo_spmv(A, x, r);
    for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
    const double res = rlo_norm2(n, r) / bnorm;
    history[hl++] = res;
    if (res < best_res) {
      best_res = res;
      memcpy(x_out, x, sizeof(double) * (size_t)n);
    }
    if (best_res <= tolerance) {
      *converged = 1;
      break;
    }
  }
  *history_len = hl;
  free(x); free(r); free(d); free(w1); free(w2);
  return RLO_OK;
}
