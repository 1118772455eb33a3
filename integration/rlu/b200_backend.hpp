// rlu/b200_backend.hpp — the reference-side adapter: drop this header into the reference's include/rlu/
// and add -lb200lu to the link line. Same names, argument meaning and exception types as the reference's
// own hot-path entry points (include/rlu/numeric.hpp:42-53, trisolve.hpp:23-39, refine.hpp:35-52), on a
// DeviceFactors instead of a NumericFactors. This file is COMPILED against the unmodified reference
// headers and sources by oracle/Makefile (target _ref/adapter_test) and exercised on the GPU by
// tests/test_adapter.py with the loop of cli::solve_sequence (src/cli.cpp:96-135).
#pragma once
#include <memory>
#include <string>
#include <vector>

#include "rlu/numeric.hpp"
#include "rlu/refine.hpp"
#include "rlu/symbolic.hpp"
#include "rlu/trisolve.hpp"
#include "b200lu.h"  // this repo: include/b200lu.h

namespace rlu::b200 {

// Borrowed view of an existing analysis product: every field of SymbolicFactors the device needs
// (include/rlu/symbolic.hpp:48-59). index_t is int64 and DenseVector is std::vector<double>, exactly
// what the C ABI takes, so no conversion or copy happens on the host.
inline b200lu_symbolic_view view_of(const SymbolicFactors& s) {
  b200lu_symbolic_view v{};
  v.n = s.n;
  v.nnz_factors = s.combined_pattern.nnz();
  v.nnz_source = static_cast<std::int64_t>(s.scatter_map.size());
  v.row_offsets = s.combined_pattern.row_offsets.data();
  v.col_indices = s.combined_pattern.col_indices.data();
  v.diag_pos = s.diag_pos.data();
  v.scatter_map = s.scatter_map.data();
  v.scatter_scale = s.scatter_scale.data();
  v.amd_forward = s.amd.forward.data();
  if (s.match) {
    v.col_perm_forward = s.match->col_perm.forward.data();
    v.row_scale = s.match->scaling.row_scale.data();
    v.col_scale = s.match->scaling.col_scale.data();
  }
  v.source_row_offsets = s.source_pattern.row_offsets.data();
  v.source_col_indices = s.source_pattern.col_indices.data();
  return v;
}

// symbolic_analyze (symbolic.hpp:72-75, src/symbolic.cpp:156-203) through b200lu_analyze: the same SymbolicFactors —
// permutations, scale factors, combined pattern, diag_pos, scatter map — bit for bit, 4-20x sooner (host code only; no
// device involved). `row_lookup`, the CPU elimination's per-row hash / bitmap, is built only when asked for: the device
// path never reads it, the reference's own factorize / refactorize do.
inline SymbolicFactors symbolic_analyze(const CsrMatrix& A, const AnalyzeOptions& options = {}, bool with_row_lookup = false) {
  if (A.nrows != A.ncols) throw DimensionError("symbolic_analyze: matrix must be square");
  A.check_structure();
  if (options.use_scaling && !A.has_values()) throw Error("mc64_scale: matrix has no values");
  b200lu_analysis* a = nullptr;
  const b200lu_status st = b200lu_analyze(A.nrows, A.row_offsets.data(), A.col_indices.data(),
                                          options.use_scaling ? A.values.data() : nullptr, options.use_scaling, options.use_amd, &a);
  if (!a) throw Error(std::string("symbolic_analyze: ") + b200lu_status_string(st));
  const std::shared_ptr<b200lu_analysis> guard(a, b200lu_analysis_destroy);
  if (st != B200LU_OK) {
    std::int64_t row = -1, count = 0;
    const std::int64_t* rows = nullptr;
    b200lu_analysis_status(a, &row, &rows, &count);
    const std::string msg = b200lu_analysis_message(a);
    if (st == B200LU_ZERO_DIAGONAL) throw ZeroDiagonalError(msg, row);
    if (st == B200LU_STRUCTURALLY_SINGULAR) throw StructurallySingularError(msg, std::vector<std::int64_t>(rows, rows + count));
    throw Error(msg);
  }
  b200lu_symbolic_view v{};
  std::int64_t fill = 0;
  double matched = 0.0;
  b200lu_analysis_view(a, &v, &fill);
  b200lu_analysis_times(a, nullptr, &matched);
  SymbolicFactors sf;
  sf.n = v.n;
  sf.combined_pattern.nrows = sf.combined_pattern.ncols = v.n;
  sf.combined_pattern.row_offsets.assign(v.row_offsets, v.row_offsets + v.n + 1);
  sf.combined_pattern.col_indices.assign(v.col_indices, v.col_indices + v.nnz_factors);
  sf.diag_pos.assign(v.diag_pos, v.diag_pos + v.n);
  sf.scatter_map.assign(v.scatter_map, v.scatter_map + v.nnz_source);
  sf.scatter_scale.assign(v.scatter_scale, v.scatter_scale + v.nnz_source);
  sf.amd = Permutation::from_forward(std::vector<index_t>(v.amd_forward, v.amd_forward + v.n));
  if (v.col_perm_forward) {
    MatchingResult m;
    m.col_perm = Permutation::from_forward(std::vector<index_t>(v.col_perm_forward, v.col_perm_forward + v.n));
    m.scaling.row_scale.assign(v.row_scale, v.row_scale + v.n);
    m.scaling.col_scale.assign(v.col_scale, v.col_scale + v.n);
    m.matched_product = matched;
    sf.match = std::move(m);
  }
  sf.source_pattern.nrows = A.nrows;
  sf.source_pattern.ncols = A.ncols;
  sf.source_pattern.row_offsets = A.row_offsets;
  sf.source_pattern.col_indices = A.col_indices;
  sf.fill_count = fill;
  if (with_row_lookup) sf.row_lookup.build(sf.combined_pattern);
  return sf;
}

// Maps the C status codes back onto the reference's exception types (include/rlu/errors.hpp).
inline void raise(b200lu_handle* h, b200lu_status st, std::int64_t row) {
  if (st == B200LU_OK) return;
  const std::string msg = b200lu_last_error(h);
  switch (st) {
    case B200LU_ZERO_PIVOT: throw ZeroPivotError(msg, row);
    case B200LU_PATTERN_MISMATCH: throw PatternMismatchError("matrix pattern differs from the analyzed pattern");
    case B200LU_DIMENSION: throw DimensionError(msg);
    default: throw Error(msg);
  }
}

// Device-side NumericFactors: same life cycle as rlu::NumericFactors (numeric.hpp:22-31).
struct DeviceFactors {
  std::shared_ptr<const SymbolicFactors> symbolic;
  std::shared_ptr<b200lu_handle> handle;
  DeviceFactors(std::shared_ptr<const SymbolicFactors> sym, double pivot_floor = 1e-30)
      : symbolic(std::move(sym)) {
    b200lu_options o;
    b200lu_default_options(&o);
    o.pivot_floor = pivot_floor;
    const b200lu_symbolic_view v = view_of(*symbolic);
    b200lu_handle* h = nullptr;
    const b200lu_status st = b200lu_create(&v, &o, &h);
    handle.reset(h, b200lu_destroy);
    raise(h, st, -1);
  }
};

inline void reset_values(DeviceFactors& f, const CsrMatrix& A) {           // numeric.cpp:75-77
  if (!pattern_equal(A, f.symbolic->source_pattern))                        // numeric.cpp:15-17, unchanged
    throw PatternMismatchError("matrix pattern differs from the analyzed pattern");
  raise(f.handle.get(), b200lu_reset_values(f.handle.get(), A.values.data(), 0), -1);
}
inline void factorize_scattered(DeviceFactors& f) {                         // numeric.cpp:79
  std::int64_t row = -1;
  const b200lu_status st = b200lu_factorize_scattered(f.handle.get(), &row);  // call first: `row` is an output
  raise(f.handle.get(), st, row);
}
inline void refactorize(DeviceFactors& f, const CsrMatrix& A) {             // numeric.cpp:70-73
  reset_values(f, A);
  factorize_scattered(f);
}
inline void solve_system(const DeviceFactors& f, const DenseVector& b, DenseVector& x) {  // trisolve.cpp:90-119
  x.resize(b.size());
  std::int64_t row = -1;
  const b200lu_status st =
      b200lu_solve(f.handle.get(), static_cast<std::int64_t>(b.size()), b.data(), x.data(), 0, &row);
  raise(f.handle.get(), st, row);
}
inline RefineOutcome fgmres_refine(const DeviceFactors& f, const DenseVector& b, const DenseVector& x0,
                                   const RefineConfig& cfg) {               // refine.cpp:39-142
  RefineOutcome out;
  out.x.resize(b.size());
  b200lu_refine_config c{cfg.max_iterations, cfg.tolerance};
  b200lu_refine_outcome o{};
  raise(f.handle.get(),
        b200lu_refine_fgmres(f.handle.get(), b.data(), x0.data(), out.x.data(), 0, 1, &c, &o), -1);
  out.iterations = o.iterations;
  out.converged = o.converged != 0;
  out.residual_history.assign(o.residual_history, o.residual_history + o.history_len);
  return out;
}

inline Cgs2Result cgs2_orthonormalize(const DeviceFactors& f, const std::vector<DenseVector>& basis,
                                      const DenseVector& v) {              // refine.cpp:8-26
  Cgs2Result res;
  res.coefficients.assign(basis.size(), 0.0);
  res.vector.resize(v.size());
  std::vector<double> flat;
  for (const DenseVector& q : basis) flat.insert(flat.end(), q.begin(), q.end());
  int breakdown = 0;
  raise(f.handle.get(),
        b200lu_cgs2_orthonormalize(f.handle.get(), static_cast<std::int64_t>(basis.size()), flat.data(), v.data(), 0,
                                   res.coefficients.data(), res.vector.data(), &res.norm, &breakdown),
        -1);
  res.breakdown = breakdown != 0;
  return res;
}
// NumericFactors::values (numeric.hpp:24): the combined L+U values, copied to the host.
inline std::vector<double> values(const DeviceFactors& f) {
  std::vector<double> out(static_cast<std::size_t>(f.symbolic->combined_pattern.nnz()));
  raise(f.handle.get(), b200lu_get_values(f.handle.get(), out.data()), -1);
  return out;
}

}  // namespace rlu::b200
