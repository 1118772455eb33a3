// rlu/b200_backend.hpp — the reference-side adapter: drop this header into the reference's include/rlu/
// and add -lb200lu to the link line. Same names, argument meaning and exception types as the reference's
// own hot-path entry points (include/rlu/numeric.hpp:42-53, trisolve.hpp:23-39, refine.hpp:35-52), on a
// DeviceFactors instead of a NumericFactors. This file is COMPILED against the unmodified reference
// headers and sources by oracle/Makefile (target _ref/adapter_test) and exercised on the GPU by
// tests/test_adapter.py with the loop of cli::solve_sequence (src/cli.cpp:96-135).
#pragma once
#include <memory>
#include <string>

#include "rlu/numeric.hpp"
#include "rlu/refine.hpp"
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
