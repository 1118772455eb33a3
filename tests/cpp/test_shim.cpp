// C++ parity tests of the rlu_b200 mirror (include/rlu_b200.hpp) — restating the reference's own
// known-answer tests (proj/tests/test_numeric.cpp, test_trisolve.cpp, test_refine.cpp) against the
// CUDA path. Built and run by tests/test_cpp_shim.py on the GPU box. Prints "ok <name>" per case
// and exits non-zero on the first failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#include "rlu_b200.hpp"

using namespace rlu_b200;
using Dense = std::vector<std::vector<double>>;

namespace {

// Natural-order analysis products of a small dense matrix (use_scaling = use_amd = false): the
// fill pattern by symbolic elimination (proj/tests/oracles.hpp:112-123), diag_pos, scatter map.
struct Sym {
  index_t n = 0;
  std::vector<index_t> ro, ci, dp, smap, amd, sro, sci;
  std::vector<double> sscale;
  CsrMatrix A;
  SymbolicView view{};

  explicit Sym(const Dense& M) {
    n = static_cast<index_t>(M.size());
    std::vector<std::vector<char>> P(n, std::vector<char>(n, 0));
    for (index_t i = 0; i < n; ++i)
      for (index_t j = 0; j < n; ++j) P[i][j] = M[i][j] != 0.0;
    for (index_t k = 0; k < n; ++k)
      for (index_t i = k + 1; i < n; ++i)
        if (P[i][k])
          for (index_t j = k + 1; j < n; ++j)
            if (P[k][j]) P[i][j] = 1;
    ro.push_back(0);
    sro.push_back(0);
    A.nrows = A.ncols = n;
    for (index_t i = 0; i < n; ++i) {
      for (index_t j = 0; j < n; ++j) {
        if (!P[i][j]) continue;
        if (j == i) dp.push_back(static_cast<index_t>(ci.size()));
        if (M[i][j] != 0.0) {
          smap.push_back(static_cast<index_t>(ci.size()));
          sci.push_back(j);
          A.values.push_back(M[i][j]);
        }
        ci.push_back(j);
      }
      ro.push_back(static_cast<index_t>(ci.size()));
      sro.push_back(static_cast<index_t>(sci.size()));
      amd.push_back(i);
    }
    sscale.assign(smap.size(), 1.0);
    A.row_offsets = sro;
    A.col_indices = sci;
    view.n = n;
    view.nnz_factors = static_cast<index_t>(ci.size());
    view.nnz_source = static_cast<index_t>(smap.size());
    view.row_offsets = ro.data();
    view.col_indices = ci.data();
    view.diag_pos = dp.data();
    view.scatter_map = smap.data();
    view.scatter_scale = sscale.data();
    view.amd_forward = amd.data();
    view.source_row_offsets = sro.data();
    view.source_col_indices = sci.data();
  }
  index_t find(index_t i, index_t j) const {
    for (index_t k = ro[i]; k < ro[i + 1]; ++k)
      if (ci[k] == j) return k;
    return -1;
  }
};

int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);          \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

void run(const char* name, const std::function<void()>& fn) {
  const int before = failures;
  try {
    fn();
  } catch (const std::exception& e) {
    std::printf("FAIL %s: unexpected exception: %s\n", name, e.what());
    ++failures;
  }
  std::printf("%s %s\n", failures == before ? "ok" : "FAILED", name);
}

const FactorOptions kStrict{1e-30, 0, nullptr, 20, true, 1};

}  // namespace

int main() {
  if (b200lu_device_count() == 0) {
    std::printf("no CUDA device: nothing can be computed (no CPU fallback)\n");
    return 3;
  }

  run("factorize dense 2x2 matches the hand elimination (test_numeric.cpp:142-157)", [] {
    Sym s({{4, 3}, {6, 3}});
    NumericFactors f = factorize(s.view, s.A);
    const auto v = f.values();
    CHECK(v[s.find(1, 0)] == 1.5);
    CHECK(v[s.dp[0]] == 4.0);
    CHECK(v[s.find(0, 1)] == 3.0);
    CHECK(v[s.dp[1]] == -1.5);
    CHECK(f.valid() && f.generation() == 1);
  });

  run("SymbolicAnalysis: natural-order product == symbolic elimination; MC64 + AMD product factorizes and solves", [] {
    const Dense M = {{4, 1, 0, 1, 0}, {1, 5, 2, 0, 0}, {0, 2, 6, 0, 1}, {1, 0, 0, 7, 3}, {0, 0, 1, 3, 8}};
    Sym s(M);
    SymbolicAnalysis plain(s.A, AnalyzeOptions{false, false});
    const SymbolicView& v = plain.view();
    CHECK(v.nnz_factors == s.view.nnz_factors && v.col_perm_forward == nullptr);
    for (index_t k = 0; k < v.nnz_factors; ++k) CHECK(v.col_indices[k] == s.ci[k]);
    for (index_t i = 0; i < s.n; ++i) CHECK(v.diag_pos[i] == s.dp[i] && v.amd_forward[i] == i);
    for (index_t k = 0; k < v.nnz_source; ++k) CHECK(v.scatter_map[k] == s.smap[k] && v.scatter_scale[k] == 1.0);
    CHECK(plain.fill_count() == v.nnz_factors - v.nnz_source);
    SymbolicAnalysis full(s.A);  // use_scaling = use_amd = true, the reference's defaults
    NumericFactors f = factorize(full.view(), s.A);
    const DenseVector xt = {1, -2, 3, -4, 5};
    DenseVector b(5, 0.0);
    for (int i = 0; i < 5; ++i)
      for (int j = 0; j < 5; ++j) b[i] += M[i][j] * xt[j];
    const DenseVector x = solve_system(f, b);
    for (int i = 0; i < 5; ++i) CHECK(std::fabs(x[i] - xt[i]) <= 1e-13);
    bool threw = false;
    try {
      CsrMatrix Z = s.A;  // drop the (2, 2) entry: structurally zero diagonal (src/symbolic.cpp:121-123)
      const index_t pos = Z.row_offsets[2] + 1;
      Z.col_indices.erase(Z.col_indices.begin() + pos);
      Z.values.erase(Z.values.begin() + pos);
      for (index_t i = 3; i <= 5; ++i) Z.row_offsets[i]--;
      SymbolicAnalysis bad(Z, AnalyzeOptions{false, false});
    } catch (const ZeroDiagonalError& e) {
      threw = e.row == 2;
    }
    CHECK(threw);
  });

  run("scatter zeroes exactly the fill slots; pattern change is rejected (test_numeric.cpp:105-123)", [] {
    Sym s({{4, 1, 1, 1}, {1, 3, 0, 0}, {1, 0, 3, 0}, {1, 0, 0, 3}});
    NumericFactors f(s.view);
    reset_values(f, s.A);
    const auto v = f.values();
    int zeros = 0;
    for (double e : v) zeros += e == 0.0;
    CHECK(v.size() == 16 && zeros == 6);
    Sym ident({{1, 0, 0, 0}, {0, 1, 0, 0}, {0, 0, 1, 0}, {0, 0, 0, 1}});
    bool thrown = false;
    try {
      reset_values(f, ident.A);
    } catch (const PatternMismatchError&) {
      thrown = true;
    }
    CHECK(thrown);
  });

  run("zero pivot fails with the offending row (test_numeric.cpp:173-184)", [] {
    Sym s({{1, 1, 0}, {1, 1, 1}, {0, 1, 1}});
    NumericFactors f(s.view);
    std::int64_t row = -1;
    try {
      refactorize(f, s.A);
    } catch (const ZeroPivotError& e) {
      row = e.row;
    }
    CHECK(row == 1);
    CHECK(!f.valid());
    bool thrown = false;
    try {
      solve_system(f, {1, 1, 1});
    } catch (const Error&) {
      thrown = true;
    }
    CHECK(thrown);  // "factors are not valid", src/trisolve.cpp:20
  });

  run("refactorize is bitwise identical to factorize (test_numeric.cpp:223-253)", [] {
    Sym s({{5, 1, 0, 2}, {1, 6, 1, 0}, {0, 1, 7, 1}, {2, 0, 1, 8}});
    NumericFactors reused = factorize(s.view, s.A);
    CsrMatrix A = s.A;
    for (int step = 1; step < 6; ++step) {
      for (std::size_t k = 0; k < A.values.size(); ++k) A.values[k] *= 1.0 + 0.01 * ((k * 7 + step) % 11);
      refactorize(reused, A);
      NumericFactors fresh = factorize(s.view, A);
      CHECK(reused.values() == fresh.values());
      CHECK(reused.generation() == static_cast<std::uint64_t>(step + 1));
    }
  });

  run("lower/upper/solve known answers (test_trisolve.cpp:56-100)", [] {
    {
      Sym s({{1, 0}, {0, 1}});
      NumericFactors f = factorize(s.view, s.A, kStrict);
      CHECK(lower_solve(f, {3, 4}) == (DenseVector{3, 4}));
      CHECK(upper_solve(f, {5, 6}) == (DenseVector{5, 6}));
      CHECK(solve_system(f, {7, 8}) == (DenseVector{7, 8}));
    }
    {
      Sym s({{1, 0}, {2, 1}});
      CHECK(lower_solve(factorize(s.view, s.A, kStrict), {1, 4}) == (DenseVector{1, 2}));
    }
    {
      Dense M(4, std::vector<double>(4, 0.0));
      for (int i = 0; i < 4; ++i) M[i][i] = 1.0;
      for (int i = 1; i < 4; ++i) M[i][i - 1] = -1.0;
      Sym s(M);
      CHECK(lower_solve(factorize(s.view, s.A, kStrict), {1, 1, 1, 1}) == (DenseVector{1, 2, 3, 4}));
    }
    {
      Sym s({{2, 1}, {0, 4}});
      CHECK(upper_solve(factorize(s.view, s.A, kStrict), {4, 8}) == (DenseVector{1, 2}));
    }
    {
      Sym s({{4, 3}, {6, 3}});
      const DenseVector x = solve_system(factorize(s.view, s.A, kStrict), {10, 12});
      CHECK(std::fabs(x[0] - 1.0) <= 1e-14 && std::fabs(x[1] - 2.0) <= 2e-14);
    }
  });

  run("exact zero diagonal and dimension errors (test_trisolve.cpp:171-192)", [] {
    Sym s({{1.0}});
    NumericFactors f = factorize(s.view, s.A);
    f.set_values({0.0}, true);
    std::int64_t row = -1;
    try {
      upper_solve(f, {1.0});
    } catch (const ZeroPivotError& e) {
      row = e.row;
    }
    CHECK(row == 0);
    Sym t({{1, 0}, {0, 1}});
    NumericFactors g = factorize(t.view, t.A);
    int dim = 0;
    try { lower_solve(g, {1, 2, 3}); } catch (const DimensionError&) { ++dim; }
    try { upper_solve(g, {1}); } catch (const DimensionError&) { ++dim; }
    try { solve_system(g, {1, 2, 3}); } catch (const DimensionError&) { ++dim; }
    CHECK(dim == 3);
  });

  run("fgmres contracts (test_refine.cpp:81-159)", [] {
    {
      Sym s({{1, 0, 0}, {0, 2, 0}, {0, 0, 3}});
      NumericFactors f = factorize(s.view, s.A);
      const RefineOutcome out = fgmres_refine(f, {1, 2, 3}, {0, 0, 0}, {}, false);
      CHECK(out.converged && out.iterations <= 3);
      for (double xi : out.x) CHECK(std::fabs(xi - 1.0) <= 1e-12);
    }
    {
      Sym s({{2, 0}, {0, 2}});
      NumericFactors f = factorize(s.view, s.A);
      const RefineOutcome out = fgmres_refine(f, {2, 2}, {1, 1}, {}, false);
      CHECK(out.converged && out.iterations == 0 && out.x == (DenseVector{1, 1}));
    }
    {
      Sym s({{1, 0, 0}, {0, 1e-8, 0}, {0, 0, 1}});
      NumericFactors f = factorize(s.view, s.A);
      const RefineOutcome out = fgmres_refine(f, {1, 1, 1}, {0, 0, 0}, RefineConfig{2, 1e-16, true}, false);
      CHECK(!out.converged && out.iterations == 2);
    }
    {
      Sym s({{5, 1, 0, 2}, {1, 6, 1, 0}, {0, 1, 7, 1}, {2, 0, 1, 8}});
      NumericFactors f = factorize(s.view, s.A);
      const RefineOutcome out = fgmres_refine(f, {1, -2, 3, 0.5}, {0, 0, 0, 0});
      CHECK(out.converged && out.iterations == 1);  // exact preconditioner: one iteration
      const RefineOutcome cl = classic_refine(f, {1, -2, 3, 0.5}, {0, 0, 0, 0});
      CHECK(cl.converged && cl.iterations <= 2);
    }
  });

  run("scenario batch: every scenario equals its single-system run, bit for bit", [] {
    Sym s({{5, 1, 0, 2}, {1, 6, 1, 0}, {0, 1, 7, 1}, {2, 0, 1, 8}});
    const index_t B = 3, n = s.n;
    std::vector<double> vals, rhs;
    std::vector<CsrMatrix> mats;
    for (index_t sc = 0; sc < B; ++sc) {
      CsrMatrix A = s.A;
      for (std::size_t k = 0; k < A.values.size(); ++k) A.values[k] *= 1.0 + 0.125 * static_cast<double>(sc) * ((k % 3) + 1);
      vals.insert(vals.end(), A.values.begin(), A.values.end());
      for (index_t i = 0; i < n; ++i) rhs.push_back(1.0 + static_cast<double>(i + sc));
      mats.push_back(A);
    }
    BatchedFactors bf(s.view, B);
    bf.refactorize(vals);
    const std::vector<double> x = bf.solve_system(rhs);
    const auto outs = bf.fgmres_refine(rhs, x);
    const auto res = bf.relative_residual(x, rhs);
    for (index_t sc = 0; sc < B; ++sc) {
      NumericFactors f = factorize(s.view, mats[sc], kStrict);
      CHECK(bf.valid(sc) && bf.values(sc) == f.values());
      const DenseVector b(rhs.begin() + sc * n, rhs.begin() + (sc + 1) * n);
      CHECK(DenseVector(x.begin() + sc * n, x.begin() + (sc + 1) * n) == solve_system(f, b));
      CHECK(res[sc] <= 1e-14 && outs[sc].converged);
    }
    // a singular scenario fails alone (test_numeric.cpp:173-184 inside a batch)
    Sym z({{1, 1, 0}, {1, 1, 1}, {0, 1, 1}});
    std::vector<double> zv = z.A.values, good = {4, 1, 1, 4, 1, 1, 4};
    std::vector<double> both = good;
    both.insert(both.end(), zv.begin(), zv.end());
    BatchedFactors bz(z.view, 2);
    std::int64_t row = -1;
    try {
      bz.refactorize(both);
    } catch (const ZeroPivotError& e) {
      row = e.row;
    }
    CHECK(row == 1 && bz.failed_rows()[0] == -1 && bz.failed_rows()[1] == 1);
    CHECK(bz.valid(0) && !bz.valid(1));
  });

  std::printf("%s (%d failure%s)\n", failures ? "FAILED" : "all ok", failures, failures == 1 ? "" : "s");
  return failures ? 1 : 0;
}
