// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// Thin extern "C" bridge over the UNMODIFIED reference library `rlu`
// (/root/reference/proj). The reference sources are compiled where they lie
// (see oracle/Makefile); nothing from them is copied into this repository.
// The resulting oracle/_ref/librlu_ref.so is used ONLY by tests/, by
// __graft_entry__.smoke() and by bench.py (input fixtures + the CPU baseline
// arm). The shipped CUDA path never links or loads it.
//
// What it exposes (all through plain pointers so ctypes can drive it):
//   * the reference's own input generators: gen_sequence (proj/src/kkt.cpp:94)
//     and the test generators random_sparse / random_vector
//     (proj/tests/oracles.hpp:186-218) on a caller-held mt19937_64;
//   * symbolic_analyze (proj/src/symbolic.cpp:156) and getters for every field
//     of SymbolicFactors (proj/include/rlu/symbolic.hpp:48-59);
//   * the hot path itself: reset_values / factorize_scattered / refactorize
//     (proj/src/numeric.cpp:62-79), lower_solve / upper_solve / solve_system
//     (proj/src/trisolve.cpp:72-119), spmv / relative_residual
//     (proj/src/sparse.cpp:128,283), fgmres_refine / classic_refine /
//     cgs2_orthonormalize (proj/src/refine.cpp:8-188);
//   * a phase timer that mirrors cli::solve_sequence's clock placement
//     (proj/src/cli.cpp:105-135).

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include <omp.h>

#include "rlu/kkt.hpp"
#include "rlu/numeric.hpp"
#include "rlu/refine.hpp"
#include "rlu/symbolic.hpp"
#include "rlu/trisolve.hpp"

// proj/tests/oracles.hpp is header-only and depends only on rlu/sparse.hpp.
#include "oracles.hpp"

using namespace rlu;

namespace {

enum Status : int {
  kOk = 0,
  kZeroPivot = 1,
  kPatternMismatch = 2,
  kDimension = 3,
  kError = 4,
  kStructurallySingular = 5,
  kZeroDiagonal = 6,
};

thread_local std::string g_last_error;
thread_local std::int64_t g_last_row = -1;

template <class Fn>
int guarded(Fn&& fn) {
  g_last_row = -1;
  try {
    fn();
    return kOk;
  } catch (const ZeroPivotError& e) {
    g_last_error = e.what();
    g_last_row = e.row;
    return kZeroPivot;
  } catch (const PatternMismatchError& e) {
    g_last_error = e.what();
    return kPatternMismatch;
  } catch (const DimensionError& e) {
    g_last_error = e.what();
    return kDimension;
  } catch (const StructurallySingularError& e) {
    g_last_error = e.what();
    return kStructurallySingular;
  } catch (const ZeroDiagonalError& e) {
    g_last_error = e.what();
    g_last_row = e.row;
    return kZeroDiagonal;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return kError;
  }
}

struct SymHandle {
  std::shared_ptr<const SymbolicFactors> sym;
};

struct NumHandle {
  std::unique_ptr<NumericFactors> nf;
  SolveWorkspace ws;
  ExecPolicy exec;
};

CsrMatrix make_csr(std::int64_t n, const std::int64_t* row_offsets, const std::int64_t* cols,
                   const double* values) {
  CsrMatrix A;
  A.nrows = n;
  A.ncols = n;
  A.row_offsets.assign(row_offsets, row_offsets + n + 1);
  const std::int64_t nnz = row_offsets[n];
  A.col_indices.assign(cols, cols + nnz);
  if (values) A.values.assign(values, values + nnz);
  return A;
}

ExecPolicy make_exec(int parallel, int workers) {
  ExecPolicy e;
  e.mode = parallel ? ExecMode::scheduled_parallel : ExecMode::sequential;
  e.worker_count = workers > 0 ? workers : omp_get_max_threads();
  return e;
}

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

template <class T>
void copy_out(const std::vector<T>& v, T* out) {
  if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(T));
}

}  // namespace

extern "C" {

const char* rluref_last_error() { return g_last_error.c_str(); }
std::int64_t rluref_last_row() { return g_last_row; }
int rluref_max_threads() { return omp_get_max_threads(); }

// ---------------------------------------------------------------- generators

void* rluref_rng_create(std::uint64_t seed) { return new std::mt19937_64(seed); }
void rluref_rng_destroy(void* rng) { delete static_cast<std::mt19937_64*>(rng); }
std::int64_t rluref_rng_uniform_int(void* rng, std::int64_t lo, std::int64_t hi) {
  std::uniform_int_distribution<index_t> d(lo, hi);
  return d(*static_cast<std::mt19937_64*>(rng));
}
double rluref_rng_uniform_real(void* rng, double lo, double hi) {
  std::uniform_real_distribution<double> d(lo, hi);
  return d(*static_cast<std::mt19937_64*>(rng));
}

// oracle::random_sparse (proj/tests/oracles.hpp:186-210); returns a CsrMatrix*.
void* rluref_random_sparse(void* rng, std::int64_t n, std::int64_t extra_per_row, double lo,
                           double hi, int diagonally_dominant) {
  auto* A = new CsrMatrix(oracle::random_sparse(*static_cast<std::mt19937_64*>(rng), n,
                                                extra_per_row, lo, hi, diagonally_dominant != 0));
  return A;
}
// oracle::random_vector (proj/tests/oracles.hpp:212-218)
void rluref_random_vector(void* rng, std::int64_t n, double lo, double hi, double* out) {
  const DenseVector v = oracle::random_vector(*static_cast<std::mt19937_64*>(rng), n, lo, hi);
  copy_out(v, out);
}

void* rluref_csr_create(std::int64_t n, const std::int64_t* row_offsets, const std::int64_t* cols,
                        const double* values) {
  return new CsrMatrix(make_csr(n, row_offsets, cols, values));
}
void rluref_csr_destroy(void* A) { delete static_cast<CsrMatrix*>(A); }
std::int64_t rluref_csr_n(void* A) { return static_cast<CsrMatrix*>(A)->nrows; }
std::int64_t rluref_csr_nnz(void* A) { return static_cast<CsrMatrix*>(A)->nnz(); }
void rluref_csr_get(void* Ap, std::int64_t* row_offsets, std::int64_t* cols, double* values) {
  const auto& A = *static_cast<CsrMatrix*>(Ap);
  copy_out(A.row_offsets, row_offsets);
  copy_out(A.col_indices, cols);
  if (values && A.has_values()) copy_out(A.values, values);
}
void rluref_csr_set_values(void* Ap, const double* values) {
  auto& A = *static_cast<CsrMatrix*>(Ap);
  A.values.assign(values, values + A.col_indices.size());
}

// gen_sequence (proj/src/kkt.cpp:94-207) with every GenConfig field exposed.
void* rluref_gen_sequence(std::int64_t n, std::int64_t m, std::uint64_t topology_seed,
                          std::uint64_t y_seed, std::int64_t num_systems, double mu0,
                          double mu_min, double reduction, double delta_p, double delta_d) {
  KktSequence* seq = nullptr;
  const int st = guarded([&] {
    GenConfig c;
    c.n = n;
    c.m = m;
    c.topology_seed = topology_seed;
    c.y_seed = y_seed;
    c.num_systems = num_systems;
    c.mu0 = mu0;
    c.mu_min = mu_min;
    c.reduction = reduction;
    c.delta_p = delta_p;
    c.delta_d = delta_d;
    seq = new KktSequence(gen_sequence(c));
    // The per-step blocks (H, J copies) are only needed for escalation; drop
    // them so C4-sized sequences stay small.
    seq->blocks.clear();
    seq->blocks.shrink_to_fit();
  });
  return st == kOk ? seq : nullptr;
}
// Same, keeping the per-step KktBlocks (H, J, D_y, deltas: include/rlu/kkt.hpp:14-21) so that the
// diagonal-only value path and the regularization escalation (src/cli.cpp:148-154) can be checked.
void* rluref_gen_sequence_blocks(std::int64_t n, std::int64_t m, std::uint64_t topology_seed,
                                 std::uint64_t y_seed, std::int64_t num_systems, double mu0,
                                 double mu_min, double reduction, double delta_p, double delta_d) {
  KktSequence* seq = nullptr;
  const int st = guarded([&] {
    GenConfig c;
    c.n = n;
    c.m = m;
    c.topology_seed = topology_seed;
    c.y_seed = y_seed;
    c.num_systems = num_systems;
    c.mu0 = mu0;
    c.mu_min = mu_min;
    c.reduction = reduction;
    c.delta_p = delta_p;
    c.delta_d = delta_d;
    seq = new KktSequence(gen_sequence(c));
  });
  return st == kOk ? seq : nullptr;
}
int rluref_seq_has_blocks(void* s) { return static_cast<KktSequence*>(s)->blocks.empty() ? 0 : 1; }
std::int64_t rluref_seq_n_primal(void* s) { return static_cast<KktSequence*>(s)->blocks.at(0).H.nrows; }
// H's own diagonal values (0 where H has no diagonal entry) and D_y / deltas of step k.
void rluref_seq_h_diag(void* s, std::int64_t k, double* out) {
  const auto& H = static_cast<KktSequence*>(s)->blocks.at(k).H;
  for (index_t i = 0; i < H.nrows; ++i) {
    const index_t t = H.find(i, i);
    out[i] = t < 0 ? 0.0 : H.values[t];
  }
}
void rluref_seq_dy(void* s, std::int64_t k, double* out) {
  copy_out(static_cast<KktSequence*>(s)->blocks.at(k).D_y, out);
}
void rluref_seq_deltas(void* s, std::int64_t k, double* delta_p, double* delta_d) {
  const auto& b = static_cast<KktSequence*>(s)->blocks.at(k);
  *delta_p = b.delta_p;
  *delta_d = b.delta_d;
}
// The regularization step of the escalation policy (src/cli.cpp:53, 148-154): doubles both deltas
// of step k and re-assembles K in place (same pattern, stronger diagonal).
int rluref_seq_double_regularization(void* s, std::int64_t k) {
  return guarded([&] {
    auto& seq = *static_cast<KktSequence*>(s);
    KktBlocks& b = seq.blocks.at(k);
    b.delta_p = b.delta_p == 0.0 ? 1e-12 : 2.0 * b.delta_p;
    b.delta_d = b.delta_d == 0.0 ? 1e-12 : 2.0 * b.delta_d;
    KktSystem regged = assemble_kkt(b);
    seq.systems[k].K = std::move(regged.K);
  });
}
void rluref_seq_destroy(void* s) { delete static_cast<KktSequence*>(s); }
std::int64_t rluref_seq_num_systems(void* s) {
  return static_cast<std::int64_t>(static_cast<KktSequence*>(s)->systems.size());
}
std::int64_t rluref_seq_n(void* s) { return static_cast<KktSequence*>(s)->systems[0].K.nrows; }
std::int64_t rluref_seq_nnz(void* s) { return static_cast<KktSequence*>(s)->systems[0].K.nnz(); }
double rluref_seq_mu(void* s, std::int64_t k) { return static_cast<KktSequence*>(s)->systems[k].mu; }
void rluref_seq_pattern(void* s, std::int64_t* row_offsets, std::int64_t* cols) {
  const auto& K = static_cast<KktSequence*>(s)->systems[0].K;
  copy_out(K.row_offsets, row_offsets);
  copy_out(K.col_indices, cols);
}
void rluref_seq_values(void* s, std::int64_t k, double* values) {
  copy_out(static_cast<KktSequence*>(s)->systems[k].K.values, values);
}
void rluref_seq_rhs(void* s, std::int64_t k, double* rhs) {
  copy_out(static_cast<KktSequence*>(s)->systems[k].rhs, rhs);
}
// Borrowed CsrMatrix* of system k (owned by the sequence).
void* rluref_seq_matrix(void* s, std::int64_t k) {
  return &static_cast<KktSequence*>(s)->systems[k].K;
}

// ------------------------------------------------------------------ analysis

void* rluref_analyze(void* Ap, int use_scaling, int use_amd, double* analyze_ms) {
  SymHandle* h = nullptr;
  const int st = guarded([&] {
    const auto t0 = Clock::now();
    AnalyzeOptions o;
    o.use_scaling = use_scaling != 0;
    o.use_amd = use_amd != 0;
    auto sym =
        std::make_shared<const SymbolicFactors>(symbolic_analyze(*static_cast<CsrMatrix*>(Ap), o));
    if (analyze_ms) *analyze_ms = ms_since(t0);
    h = new SymHandle{std::move(sym)};
  });
  return st == kOk ? h : nullptr;
}
void rluref_sym_destroy(void* h) { delete static_cast<SymHandle*>(h); }
std::int64_t rluref_sym_n(void* h) { return static_cast<SymHandle*>(h)->sym->n; }
std::int64_t rluref_sym_nnz_factors(void* h) {
  return static_cast<SymHandle*>(h)->sym->combined_pattern.nnz();
}
std::int64_t rluref_sym_nnz_source(void* h) {
  return static_cast<std::int64_t>(static_cast<SymHandle*>(h)->sym->scatter_map.size());
}
std::int64_t rluref_sym_fill_count(void* h) { return static_cast<SymHandle*>(h)->sym->fill_count; }
int rluref_sym_has_match(void* h) { return static_cast<SymHandle*>(h)->sym->match ? 1 : 0; }
void rluref_sym_pattern(void* h, std::int64_t* row_offsets, std::int64_t* cols,
                        std::int64_t* diag_pos) {
  const auto& s = *static_cast<SymHandle*>(h)->sym;
  copy_out(s.combined_pattern.row_offsets, row_offsets);
  copy_out(s.combined_pattern.col_indices, cols);
  copy_out(s.diag_pos, diag_pos);
}
void rluref_sym_scatter(void* h, std::int64_t* scatter_map, double* scatter_scale) {
  const auto& s = *static_cast<SymHandle*>(h)->sym;
  copy_out(s.scatter_map, scatter_map);
  copy_out(s.scatter_scale, scatter_scale);
}
void rluref_sym_source_pattern(void* h, std::int64_t* row_offsets, std::int64_t* cols) {
  const auto& s = *static_cast<SymHandle*>(h)->sym;
  copy_out(s.source_pattern.row_offsets, row_offsets);
  copy_out(s.source_pattern.col_indices, cols);
}
void rluref_sym_amd(void* h, std::int64_t* forward) {
  copy_out(static_cast<SymHandle*>(h)->sym->amd.forward, forward);
}
void rluref_sym_match(void* h, std::int64_t* col_perm_forward, double* row_scale,
                      double* col_scale) {
  const auto& s = *static_cast<SymHandle*>(h)->sym;
  if (!s.match) return;
  copy_out(s.match->col_perm.forward, col_perm_forward);
  copy_out(s.match->scaling.row_scale, row_scale);
  copy_out(s.match->scaling.col_scale, col_scale);
}
// RowLookupTable::variant census (proj/include/rlu/symbolic.hpp:28): rows using the hash variant.
std::int64_t rluref_sym_hash_rows(void* h) {
  const auto& s = *static_cast<SymHandle*>(h)->sym;
  std::int64_t c = 0;
  for (index_t i = 0; i < s.n; ++i) {
    c += s.row_lookup.variant(i) == RowLookupTable::Variant::hash;
  }
  return c;
}

// ------------------------------------------------------------------- numeric

void* rluref_numeric_create(void* symh, double pivot_floor, int parallel, int workers) {
  auto* h = new NumHandle;
  FactorOptions opt;
  opt.pivot_floor = pivot_floor;
  opt.exec = make_exec(parallel, workers);
  h->exec = opt.exec;
  h->nf = std::make_unique<NumericFactors>(static_cast<SymHandle*>(symh)->sym, opt);
  return h;
}
void rluref_numeric_destroy(void* h) { delete static_cast<NumHandle*>(h); }
void rluref_numeric_set_exec(void* hp, int parallel, int workers) {
  auto* h = static_cast<NumHandle*>(hp);
  h->exec = make_exec(parallel, workers);
  h->nf->options.exec = h->exec;
}
// Execution policy of the solve phases only (solve_system takes its own ExecPolicy,
// include/rlu/trisolve.hpp:36); rluref_numeric_set_exec sets both.
void rluref_numeric_set_solve_exec(void* hp, int parallel, int workers) {
  static_cast<NumHandle*>(hp)->exec = make_exec(parallel, workers);
}
int rluref_reset_values(void* h, void* A) {
  return guarded([&] { reset_values(*static_cast<NumHandle*>(h)->nf, *static_cast<CsrMatrix*>(A)); });
}
int rluref_factorize_scattered(void* h) {
  return guarded([&] { factorize_scattered(*static_cast<NumHandle*>(h)->nf); });
}
int rluref_refactorize(void* h, void* A) {
  return guarded([&] { refactorize(*static_cast<NumHandle*>(h)->nf, *static_cast<CsrMatrix*>(A)); });
}
int rluref_numeric_valid(void* h) { return static_cast<NumHandle*>(h)->nf->valid ? 1 : 0; }
std::uint64_t rluref_numeric_generation(void* h) {
  return static_cast<NumHandle*>(h)->nf->generation;
}
void rluref_numeric_get_values(void* h, double* out) {
  copy_out(static_cast<NumHandle*>(h)->nf->values, out);
}
void rluref_numeric_set_values(void* hp, const double* in, int valid) {
  auto* h = static_cast<NumHandle*>(hp);
  std::memcpy(h->nf->values.data(), in, h->nf->values.size() * sizeof(double));
  h->nf->valid = valid != 0;
}

int rluref_lower_solve(void* hp, std::int64_t len, const double* y, double* x) {
  auto* h = static_cast<NumHandle*>(hp);
  return guarded([&] {
    const DenseVector r = lower_solve(*h->nf, DenseVector(y, y + len), h->exec);
    copy_out(r, x);
  });
}
int rluref_upper_solve(void* hp, std::int64_t len, const double* y, double* x) {
  auto* h = static_cast<NumHandle*>(hp);
  return guarded([&] {
    const DenseVector r = upper_solve(*h->nf, DenseVector(y, y + len), h->exec);
    copy_out(r, x);
  });
}
int rluref_solve_system(void* hp, std::int64_t len, const double* b, double* x) {
  auto* h = static_cast<NumHandle*>(hp);
  return guarded([&] {
    DenseVector xv;
    solve_system(*h->nf, DenseVector(b, b + len), h->ws, xv, h->exec);
    copy_out(xv, x);
  });
}
std::uint64_t rluref_workspace_allocation_events(void* hp) {
  return static_cast<NumHandle*>(hp)->ws.allocation_events;
}

// ---------------------------------------------------------------- sparse ops

int rluref_spmv(void* A, const double* x, double* y) {
  return guarded([&] {
    const auto& M = *static_cast<CsrMatrix*>(A);
    const DenseVector r = spmv(M, DenseVector(x, x + M.ncols));
    copy_out(r, y);
  });
}
double rluref_relative_residual(void* A, const double* x, const double* b) {
  const auto& M = *static_cast<CsrMatrix*>(A);
  return relative_residual(M, DenseVector(x, x + M.ncols), DenseVector(b, b + M.nrows));
}
double rluref_dot(std::int64_t n, const double* a, const double* b) {
  return dot(DenseVector(a, a + n), DenseVector(b, b + n));
}
double rluref_norm2(std::int64_t n, const double* a) { return norm2(DenseVector(a, a + n)); }

// ---------------------------------------------------------------- refinement

// precond_handle == nullptr selects the identity preconditioner.
// method: 0 = fgmres_refine, 1 = classic_refine.
// history must hold max_iterations + 2 doubles.
int rluref_refine(void* Ap, const double* b, const double* x0, void* precond_handle, int method,
                  int max_iterations, double tolerance, double* x_out, int* iterations,
                  int* converged, double* history, int* history_len) {
  return guarded([&] {
    const auto& A = *static_cast<CsrMatrix*>(Ap);
    const std::int64_t n = A.nrows;
    auto* h = static_cast<NumHandle*>(precond_handle);
    const LinearOperator precond = [h](const DenseVector& in, DenseVector& out) {
      if (h) {
        solve_system(*h->nf, in, h->ws, out, h->exec);
      } else {
        out = in;
      }
    };
    RefineConfig cfg;
    cfg.max_iterations = max_iterations;
    cfg.tolerance = tolerance;
    const DenseVector bv(b, b + n), xv(x0, x0 + n);
    const RefineOutcome out = method == 0 ? fgmres_refine(A, bv, xv, precond, cfg)
                                          : classic_refine(A, bv, xv, precond, cfg);
    copy_out(out.x, x_out);
    *iterations = out.iterations;
    *converged = out.converged ? 1 : 0;
    *history_len = static_cast<int>(out.residual_history.size());
    copy_out(out.residual_history, history);
  });
}

// cgs2_orthonormalize (proj/src/refine.cpp:8-26); basis is k row-major n-vectors.
int rluref_cgs2(std::int64_t n, std::int64_t k, const double* basis, const double* v,
                double* coefficients, double* vec_out, double* norm, int* breakdown) {
  return guarded([&] {
    std::vector<DenseVector> B;
    for (std::int64_t j = 0; j < k; ++j) B.emplace_back(basis + j * n, basis + (j + 1) * n);
    const Cgs2Result r = cgs2_orthonormalize(B, DenseVector(v, v + n));
    copy_out(r.coefficients, coefficients);
    copy_out(r.vector, vec_out);
    *norm = r.norm;
    *breakdown = r.breakdown ? 1 : 0;
  });
}

// --------------------------------------------------------------- phase timer

// One pass of the hot path over system k of a generated sequence with the
// clocks placed exactly as cli::solve_sequence places them
// (proj/src/cli.cpp:105-135). times_ms = {scatter, factor, trisolve, refine}.
// refine: 0 none, 1 fgmres. x_out may be null.
int rluref_run_system(void* hp, void* seqp, std::int64_t k, int refine, int max_iterations,
                      double tolerance, double* times_ms, double* relres_direct,
                      double* relres_final, int* refine_iters, double* x_out) {
  auto* h = static_cast<NumHandle*>(hp);
  auto& sys = static_cast<KktSequence*>(seqp)->systems[k];
  return guarded([&] {
    DenseVector x;
    auto t = Clock::now();
    reset_values(*h->nf, sys.K);
    times_ms[0] = ms_since(t);

    t = Clock::now();
    factorize_scattered(*h->nf);
    times_ms[1] = ms_since(t);

    t = Clock::now();
    solve_system(*h->nf, sys.rhs, h->ws, x, h->exec);
    times_ms[2] = ms_since(t);

    *relres_direct = relative_residual(sys.K, x, sys.rhs);
    *relres_final = *relres_direct;
    *refine_iters = 0;
    times_ms[3] = 0.0;
    if (refine == 1) {
      RefineConfig rc;
      rc.max_iterations = max_iterations;
      rc.tolerance = tolerance;
      const LinearOperator precond = [&](const DenseVector& in, DenseVector& out) {
        solve_system(*h->nf, in, h->ws, out, h->exec);
      };
      t = Clock::now();
      RefineOutcome outcome = fgmres_refine(sys.K, sys.rhs, x, precond, rc);
      times_ms[3] = ms_since(t);
      *refine_iters = outcome.iterations;
      x = std::move(outcome.x);
      *relres_final = relative_residual(sys.K, x, sys.rhs);
    }
    if (x_out) copy_out(x, x_out);
  });
}

}  // extern "C"
