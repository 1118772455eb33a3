// rlu_b200.hpp — header-only C++ mirror of the reference's numeric / triangular-solve /
// refinement interface over the b200lu C ABI (include/b200lu.h).
//
// Same names, argument meaning and error behaviour as the reference (paths relative to the
// reference's proj/):
//   factorize / refactorize / reset_values / factorize_scattered   include/rlu/numeric.hpp:42-53
//   lower_solve / upper_solve / solve_system                        include/rlu/trisolve.hpp:23-39
//   fgmres_refine / classic_refine                                  include/rlu/refine.hpp:43-52
//   Error / DimensionError / ZeroPivotError / PatternMismatchError  include/rlu/errors.hpp:11-54
//
// The reference's own SymbolicFactors cannot be named here (this repo never includes reference
// headers); SymbolicView carries the same fields as borrowed pointers, and INTEGRATION.md shows the
// ten-line adapter from rlu::SymbolicFactors.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "b200lu.h"

namespace rlu_b200 {

using index_t = std::int64_t;             // include/rlu/sparse.hpp:10
using DenseVector = std::vector<double>;  // include/rlu/sparse.hpp:11

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
class DimensionError : public Error {
 public:
  using Error::Error;
};
class ZeroPivotError : public Error {
 public:
  ZeroPivotError(const std::string& msg, std::int64_t r) : Error(msg), row(r) {}
  std::int64_t row;
};
class PatternMismatchError : public Error {
 public:
  using Error::Error;
};
class DeviceError : public Error {  // CUDA failure / no device: there is no CPU fallback
 public:
  using Error::Error;
};

// rlu::CsrMatrix (include/rlu/sparse.hpp:31-47)
struct CsrMatrix {
  index_t nrows = 0, ncols = 0;
  std::vector<index_t> row_offsets, col_indices;
  std::vector<double> values;
  bool has_values() const { return values.size() == col_indices.size(); }
};

// Borrowed image of rlu::SymbolicFactors (include/rlu/symbolic.hpp:48-59).
using SymbolicView = b200lu_symbolic_view;

struct FactorOptions {  // include/rlu/numeric.hpp:12-15 (+ placement)
  double pivot_floor = 1e-30;
  int device = 0;
  void* stream = nullptr;
  int refine_capacity = 20;
  bool strict_order = false;  // sweeps in the reference's summation order
  int concurrency = 1;        // handles sharing the device at the same time
};

struct RefineConfig {  // include/rlu/refine.hpp:13-17
  int max_iterations = 20;
  double tolerance = 1e-14;
  bool enabled = true;
};

struct RefineOutcome {  // include/rlu/refine.hpp:19-24
  DenseVector x;
  int iterations = 0;
  std::vector<double> residual_history;
  bool converged = false;
};

// rlu::NumericFactors (include/rlu/numeric.hpp:22-31) with its SolveWorkspace folded in.
class NumericFactors {
 public:
  NumericFactors(const SymbolicView& sym, const FactorOptions& opt = {}) : n_(sym.n), nnz_(sym.nnz_factors) {
    b200lu_options o;
    b200lu_default_options(&o);
    o.pivot_floor = opt.pivot_floor;
    o.device = opt.device;
    o.stream = opt.stream;
    o.refine_capacity = opt.refine_capacity;
    o.flags = opt.strict_order ? B200LU_FLAG_STRICT_ORDER : 0;
    o.concurrency = opt.concurrency;
    b200lu_handle* h = nullptr;
    const b200lu_status st = b200lu_create(&sym, &o, &h);
    if (st != B200LU_OK) {
      const std::string msg = h ? b200lu_last_error(h) : "";
      b200lu_destroy(h);
      if (st == B200LU_NO_DEVICE) throw DeviceError("no CUDA device: the b200lu path has no CPU fallback");
      if (st == B200LU_CUDA_ERROR) throw DeviceError(msg);
      throw Error("b200lu_create: " + msg);
    }
    h_.reset(h, b200lu_destroy);
  }

  bool valid() const { return b200lu_valid(h_.get()) != 0; }
  std::uint64_t generation() const { return b200lu_generation(h_.get()); }
  index_t n() const { return n_; }
  std::vector<double> values() const {
    std::vector<double> v(static_cast<std::size_t>(nnz_));
    check(b200lu_get_values(h_.get(), v.data()), -1);
    return v;
  }
  void set_values(const std::vector<double>& v, bool valid) {
    check(b200lu_set_values(h_.get(), v.data(), valid ? 1 : 0), -1);
  }
  b200lu_handle* handle() const { return h_.get(); }

  void check(b200lu_status st, std::int64_t row) const {
    if (st == B200LU_OK) return;
    std::string msg = b200lu_last_error(h_.get());
    if (msg.empty()) msg = b200lu_status_string(st);
    switch (st) {
      case B200LU_ZERO_PIVOT: throw ZeroPivotError(msg, row);
      case B200LU_PATTERN_MISMATCH: throw PatternMismatchError("matrix pattern differs from the analyzed pattern");
      case B200LU_DIMENSION: throw DimensionError(msg);
      case B200LU_CUDA_ERROR:
      case B200LU_NO_DEVICE: throw DeviceError(msg);
      default: throw Error(msg);
    }
  }

 private:
  std::shared_ptr<b200lu_handle> h_;
  index_t n_, nnz_;
};

namespace detail {
inline void guard(const NumericFactors& f, const CsrMatrix& A) {  // src/numeric.cpp:15-18
  b200lu_status st = B200LU_PATTERN_MISMATCH;
  if (A.nrows == A.ncols && static_cast<index_t>(A.row_offsets.size()) == A.nrows + 1) {
    st = b200lu_check_pattern(f.handle(), A.nrows, A.row_offsets.data(), A.col_indices.data());
  }
  if (st != B200LU_OK) throw PatternMismatchError("matrix pattern differs from the analyzed pattern");
  if (!A.has_values()) throw Error("scatter_values: matrix has no values");
}
}  // namespace detail

inline void reset_values(NumericFactors& f, const CsrMatrix& A) {  // src/numeric.cpp:75-77
  detail::guard(f, A);
  f.check(b200lu_reset_values(f.handle(), A.values.data(), 0), -1);
}
inline void factorize_scattered(NumericFactors& f) {  // src/numeric.cpp:79
  std::int64_t row = -1;
  const b200lu_status st = b200lu_factorize_scattered(f.handle(), &row);  // call first: `row` is an output
  f.check(st, row);
}
inline void refactorize(NumericFactors& f, const CsrMatrix& A) {  // src/numeric.cpp:70-73
  detail::guard(f, A);
  std::int64_t row = -1;
  const b200lu_status st = b200lu_refactorize(f.handle(), A.values.data(), 0, &row);
  f.check(st, row);
}
inline NumericFactors factorize(const SymbolicView& sym, const CsrMatrix& A, const FactorOptions& opt = {}) {
  NumericFactors f(sym, opt);  // src/numeric.cpp:62-68
  refactorize(f, A);
  return f;
}

inline DenseVector lower_solve(const NumericFactors& f, const DenseVector& y) {  // src/trisolve.cpp:72-79
  DenseVector x(y.size());
  f.check(b200lu_lower_solve(f.handle(), static_cast<index_t>(y.size()), y.data(), x.data(), 0), -1);
  return x;
}
inline DenseVector upper_solve(const NumericFactors& f, const DenseVector& y) {  // src/trisolve.cpp:81-88
  DenseVector x(y.size());
  std::int64_t row = -1;
  const b200lu_status st =
      b200lu_upper_solve(f.handle(), static_cast<index_t>(y.size()), y.data(), x.data(), 0, &row);
  f.check(st, row);
  return x;
}
inline void solve_system(const NumericFactors& f, const DenseVector& b, DenseVector& x) {  // src/trisolve.cpp:90-119
  if (x.size() != b.size()) x.resize(b.size());
  std::int64_t row = -1;
  const b200lu_status st = b200lu_solve(f.handle(), static_cast<index_t>(b.size()), b.data(), x.data(), 0, &row);
  f.check(st, row);
}
inline DenseVector solve_system(const NumericFactors& f, const DenseVector& b) {
  DenseVector x;
  solve_system(f, b, x);
  return x;
}

namespace detail {
template <class Fn>
RefineOutcome refine(Fn fn, const NumericFactors& f, const DenseVector& b, const DenseVector& x0,
                     const RefineConfig& cfg, bool preconditioned) {
  if (static_cast<index_t>(b.size()) != f.n() || static_cast<index_t>(x0.size()) != f.n()) {
    throw DimensionError("refine: vector length " + std::to_string(b.size()) + ", expected " + std::to_string(f.n()));
  }
  RefineOutcome out;
  out.x.resize(b.size());
  b200lu_refine_config c{cfg.max_iterations, cfg.tolerance};
  b200lu_refine_outcome o{};
  f.check(fn(f.handle(), b.data(), x0.data(), out.x.data(), 0, preconditioned ? 1 : 0, &c, &o), -1);
  out.iterations = o.iterations;
  out.converged = o.converged != 0;
  out.residual_history.assign(o.residual_history, o.residual_history + o.history_len);
  return out;
}
}  // namespace detail

// fgmres_refine (src/refine.cpp:39-142) with A = the matrix last handed to reset_values /
// refactorize and the preconditioner solve_system(f, .) — the pairing of src/cli.cpp:121-135.
inline RefineOutcome fgmres_refine(const NumericFactors& f, const DenseVector& b, const DenseVector& x0,
                                   const RefineConfig& cfg = {}, bool preconditioned = true) {
  return detail::refine(b200lu_refine_fgmres, f, b, x0, cfg, preconditioned);
}
inline RefineOutcome classic_refine(const NumericFactors& f, const DenseVector& b, const DenseVector& x0,
                                    const RefineConfig& cfg = {}, bool preconditioned = true) {
  return detail::refine(b200lu_refine_classic, f, b, x0, cfg, preconditioned);  // src/refine.cpp:150-188
}

// ---------------------------------------------------------------------------------------------
// Host-side symbolic analysis (b200lu_analyze, csrc/analyze.cpp): rlu::symbolic_analyze(A, AnalyzeOptions)
// (include/rlu/symbolic.hpp:67-75, src/symbolic.cpp:156-203) — the same product bit for bit, owned by this object.
class ZeroDiagonalError : public Error {  // include/rlu/errors.hpp:37-42
 public:
  ZeroDiagonalError(const std::string& msg, std::int64_t r) : Error(msg), row(r) {}
  std::int64_t row;
};
class StructurallySingularError : public Error {  // include/rlu/errors.hpp:27-34
 public:
  StructurallySingularError(const std::string& msg, std::vector<std::int64_t> rows) : Error(msg), deficient_rows(std::move(rows)) {}
  std::vector<std::int64_t> deficient_rows;
};
struct AnalyzeOptions {  // include/rlu/symbolic.hpp:67-70
  bool use_scaling = true;
  bool use_amd = true;
};
class SymbolicAnalysis {
 public:
  SymbolicAnalysis(const CsrMatrix& A, const AnalyzeOptions& opt = {}) {
    if (A.nrows != A.ncols) throw DimensionError("symbolic_analyze: matrix must be square");
    if (static_cast<index_t>(A.row_offsets.size()) != A.nrows + 1) throw Error("row_offsets length must be nrows + 1");
    if (opt.use_scaling && !(A.has_values() && !A.values.empty())) throw Error("mc64_scale: matrix has no values");
    const b200lu_status st = b200lu_analyze(A.nrows, A.row_offsets.data(), A.col_indices.data(),
                                            opt.use_scaling ? A.values.data() : nullptr, opt.use_scaling, opt.use_amd, &h_);
    if (!h_) throw Error(std::string("symbolic_analyze: ") + b200lu_status_string(st));
    if (st != B200LU_OK) {
      std::int64_t row = -1, count = 0;
      const std::int64_t* rows = nullptr;
      b200lu_analysis_status(h_, &row, &rows, &count);
      const std::string msg = b200lu_analysis_message(h_);
      std::vector<std::int64_t> deficient(rows, rows + count);
      b200lu_analysis_destroy(h_);
      h_ = nullptr;
      if (st == B200LU_ZERO_DIAGONAL) throw ZeroDiagonalError(msg, row);
      if (st == B200LU_STRUCTURALLY_SINGULAR) throw StructurallySingularError(msg, std::move(deficient));
      throw Error(msg);
    }
    b200lu_analysis_view(h_, &view_, &fill_count_);
  }
  SymbolicAnalysis(const SymbolicAnalysis&) = delete;
  SymbolicAnalysis& operator=(const SymbolicAnalysis&) = delete;
  ~SymbolicAnalysis() { b200lu_analysis_destroy(h_); }
  const SymbolicView& view() const { return view_; }  // valid while this object lives
  index_t fill_count() const { return fill_count_; }

 private:
  b200lu_analysis* h_ = nullptr;
  SymbolicView view_{};
  std::int64_t fill_count_ = 0;
};

// ---------------------------------------------------------------------------------------------
// Scenario batches (b200lu_batch_*): `batch` systems over one SymbolicView, factorized and solved
// together. Arrays are scenario-major: values [batch][nnz(A)], vectors [batch][n].
class BatchedFactors {
 public:
  BatchedFactors(const SymbolicView& sym, index_t batch, const FactorOptions& opt = {})
      : n_(sym.n), nnz_(sym.nnz_factors), nnz_source_(sym.nnz_source), batch_(batch) {
    b200lu_options o;
    b200lu_default_options(&o);
    o.pivot_floor = opt.pivot_floor;
    o.device = opt.device;
    o.stream = opt.stream;
    o.refine_capacity = opt.refine_capacity;
    b200lu_batch* h = nullptr;
    const b200lu_status st = b200lu_batch_create(&sym, &o, batch, &h);
    if (st != B200LU_OK) {
      const std::string msg = h ? b200lu_batch_last_error(h) : "";
      b200lu_batch_destroy(h);
      if (st == B200LU_NO_DEVICE) throw DeviceError("no CUDA device: the b200lu path has no CPU fallback");
      if (st == B200LU_CUDA_ERROR) throw DeviceError(msg);
      throw Error("b200lu_batch_create: " + msg);
    }
    h_.reset(h, b200lu_batch_destroy);
  }
  index_t n() const { return n_; }
  index_t batch() const { return batch_; }
  b200lu_batch* handle() const { return h_.get(); }
  bool valid(index_t scenario) const { return b200lu_batch_valid(h_.get(), scenario) != 0; }
  std::vector<double> values(index_t scenario) const {
    std::vector<double> v(static_cast<std::size_t>(nnz_));
    check(b200lu_batch_get_values(h_.get(), scenario, v.data()), {});
    return v;
  }
  // refactorize (src/numeric.cpp:70-73) per scenario. Throws ZeroPivotError carrying the first
  // failing scenario's row; failed_rows() then holds every scenario's row (-1 = factorized).
  void refactorize(const std::vector<double>& values) {
    if (static_cast<index_t>(values.size()) != batch_ * nnz_source_) throw DimensionError("refactorize: expected batch * nnz(A) values");
    failed_.assign(static_cast<std::size_t>(batch_), -1);
    const b200lu_status st = b200lu_batch_refactorize(h_.get(), values.data(), 0, failed_.data());
    check(st, failed_);
  }
  const std::vector<std::int64_t>& failed_rows() const { return failed_; }
  std::vector<double> solve_system(const std::vector<double>& b) const {  // src/trisolve.cpp:90-119 per scenario
    if (static_cast<index_t>(b.size()) != batch_ * n_) throw DimensionError("solve_system: expected batch * n values");
    std::vector<double> x(b.size());
    std::vector<std::int64_t> failed(static_cast<std::size_t>(batch_), -1);
    const b200lu_status st = b200lu_batch_solve(h_.get(), b.data(), x.data(), 0, failed.data());
    check(st, failed);
    return x;
  }
  std::vector<double> relative_residual(const std::vector<double>& x, const std::vector<double>& b) const {
    std::vector<double> out(static_cast<std::size_t>(batch_));
    check(b200lu_batch_relative_residual(h_.get(), x.data(), b.data(), 0, out.data()), {});
    return out;
  }
  // fgmres_refine (src/refine.cpp:39-142) per scenario; x of scenario s is out[s].x.
  std::vector<RefineOutcome> fgmres_refine(const std::vector<double>& b, const std::vector<double>& x0,
                                           const RefineConfig& cfg = {}, bool preconditioned = true) const {
    if (static_cast<index_t>(b.size()) != batch_ * n_ || x0.size() != b.size()) throw DimensionError("refine: expected batch * n values");
    std::vector<double> x(b.size());
    std::vector<b200lu_refine_outcome> oc(static_cast<std::size_t>(batch_));
    b200lu_refine_config c{cfg.max_iterations, cfg.tolerance};
    check(b200lu_batch_refine_fgmres(h_.get(), b.data(), x0.data(), x.data(), 0, preconditioned ? 1 : 0, &c, oc.data()), {});
    std::vector<RefineOutcome> out(static_cast<std::size_t>(batch_));
    for (index_t s = 0; s < batch_; ++s) {
      out[s].x.assign(x.begin() + s * n_, x.begin() + (s + 1) * n_);
      out[s].iterations = oc[s].iterations;
      out[s].converged = oc[s].converged != 0;
      out[s].residual_history.assign(oc[s].residual_history, oc[s].residual_history + oc[s].history_len);
    }
    return out;
  }

 private:
  void check(b200lu_status st, const std::vector<std::int64_t>& failed) const {
    if (st == B200LU_OK) return;
    std::string msg = b200lu_batch_last_error(h_.get());
    if (msg.empty()) msg = b200lu_status_string(st);
    std::int64_t row = -1;
    for (std::int64_t r : failed) {
      if (r >= 0) {
        row = r;
        break;
      }
    }
    switch (st) {
      case B200LU_ZERO_PIVOT: throw ZeroPivotError(msg, row);
      case B200LU_PATTERN_MISMATCH: throw PatternMismatchError("matrix pattern differs from the analyzed pattern");
      case B200LU_DIMENSION: throw DimensionError(msg);
      case B200LU_CUDA_ERROR:
      case B200LU_NO_DEVICE: throw DeviceError(msg);
      default: throw Error(msg);
    }
  }
  std::shared_ptr<b200lu_batch> h_;
  index_t n_, nnz_, nnz_source_, batch_;
  std::vector<std::int64_t> failed_;
};

}  // namespace rlu_b200
