// TEST INFRASTRUCTURE. The reference-side adapter (integration/rlu/b200_backend.hpp) compiled against the
// UNMODIFIED reference (headers + 9 core sources, see oracle/Makefile) and linked with libb200lu.so:
// the per-system loop of cli::solve_sequence (src/cli.cpp:96-135) over a generated KKT sequence, once with
// the reference's CPU entry points and once with their rlu::b200:: twins. Checks, per system: L/U values
// bit for bit, same refinement iteration count, final relative residual at or below the CPU run's (both
// sit at the rounding floor: a few ulps of slack, stated below), and the error mapping (pattern mismatch,
// zero pivot with the lowest failing row). Prints "ok <what>" lines and "all ok"; exit 3 without a device.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>

#include "rlu/b200_backend.hpp"
#include "rlu/kkt.hpp"
#include "rlu/symbolic.hpp"

using namespace rlu;

static int fail(const char* what) {
  std::printf("FAILED %s\n", what);
  return 1;
}

int main(int argc, char** argv) {
  GenConfig cfg;
  cfg.n = argc > 1 ? std::atoll(argv[1]) : 1400;
  cfg.m = argc > 2 ? std::atoll(argv[2]) : 600;
  cfg.num_systems = 10;
  const KktSequence seq = gen_sequence(cfg);
  // symbolic_analyze through the adapter (b200lu_analyze) against the reference's own, field by field, with and
  // without MC64 — the values of the matching's scale factors compared bitwise (src/symbolic.cpp:156-203)
  for (const bool scaling : {false, true}) {
    AnalyzeOptions o;
    o.use_scaling = scaling;
    const SymbolicFactors want = symbolic_analyze(seq.systems[0].K, o);
    const SymbolicFactors got = b200::symbolic_analyze(seq.systems[0].K, o, /*with_row_lookup=*/true);
    bool same = got.n == want.n && got.combined_pattern.row_offsets == want.combined_pattern.row_offsets &&
                got.combined_pattern.col_indices == want.combined_pattern.col_indices && got.diag_pos == want.diag_pos &&
                got.scatter_map == want.scatter_map && got.amd.forward == want.amd.forward && got.amd.inverse == want.amd.inverse &&
                got.fill_count == want.fill_count && got.match.has_value() == want.match.has_value() &&
                got.scatter_scale.size() == want.scatter_scale.size() &&
                std::memcmp(got.scatter_scale.data(), want.scatter_scale.data(), got.scatter_scale.size() * sizeof(double)) == 0;
    if (same && want.match) {
      same = got.match->col_perm.forward == want.match->col_perm.forward &&
             std::memcmp(got.match->scaling.row_scale.data(), want.match->scaling.row_scale.data(), sizeof(double) * want.n) == 0 &&
             std::memcmp(got.match->scaling.col_scale.data(), want.match->scaling.col_scale.data(), sizeof(double) * want.n) == 0 &&
             got.match->matched_product == want.match->matched_product;
    }
    if (!same) return fail("b200::symbolic_analyze differs from the reference's symbolic_analyze");
    // and the product is a full SymbolicFactors: the reference's own CPU factorization runs on it
    const auto shared = std::make_shared<const SymbolicFactors>(got);
    NumericFactors on_fast(shared, FactorOptions{});
    NumericFactors on_ref(std::make_shared<const SymbolicFactors>(want), FactorOptions{});
    refactorize(on_fast, seq.systems[0].K);
    refactorize(on_ref, seq.systems[0].K);
    if (on_fast.values != on_ref.values) return fail("reference factorization on the adapter's analysis differs");
    std::printf("ok symbolic_analyze (%s): identical product, fill %lld\n", scaling ? "mc64 + amd" : "amd", static_cast<long long>(got.fill_count));
  }
  if (b200lu_device_count() == 0) {
    std::printf("no CUDA device: the b200 backend has no CPU fallback\n");
    return 3;
  }
  AnalyzeOptions aopt;
  aopt.use_scaling = false;  // the KLU-style path of the north star (cli.hpp:14)
  const auto sym = std::make_shared<const SymbolicFactors>(symbolic_analyze(seq.systems[0].K, aopt));
  NumericFactors cpu(sym, FactorOptions{});
  b200::DeviceFactors dev(sym);
  SolveWorkspace ws;
  RefineConfig rc;
  int worse = 0;
  for (std::size_t k = 0; k < seq.systems.size(); ++k) {
    const KktSystem& sys = seq.systems[k];
    // --- reference, src/cli.cpp:105-135
    reset_values(cpu, sys.K);
    factorize_scattered(cpu);
    DenseVector x;
    solve_system(cpu, sys.rhs, ws, x, ExecPolicy{});
    const LinearOperator precond = [&](const DenseVector& in, DenseVector& out) { solve_system(cpu, in, ws, out, ExecPolicy{}); };
    const RefineOutcome ref = fgmres_refine(sys.K, sys.rhs, x, precond, rc);
    const double res_ref = relative_residual(sys.K, ref.x, sys.rhs);
    // --- the same four calls on the device
    b200::reset_values(dev, sys.K);
    b200::factorize_scattered(dev);
    DenseVector xd;
    b200::solve_system(dev, sys.rhs, xd);
    const RefineOutcome got = b200::fgmres_refine(dev, sys.rhs, xd, rc);
    const double res_dev = relative_residual(sys.K, got.x, sys.rhs);

    const std::vector<double> lu = b200::values(dev);
    if (lu.size() != cpu.values.size() || std::memcmp(lu.data(), cpu.values.data(), lu.size() * sizeof(double)) != 0) {
      return fail("L/U values differ from the reference's");
    }
    if (got.iterations != ref.iterations || got.converged != ref.converged) return fail("refinement outcome differs");
    if (!(res_dev <= std::fmax(4.0 * res_ref, 1e-15))) return fail("final residual above the reference's");
    worse += res_dev > res_ref;
    std::printf("ok system %zu: L/U bitwise, iterations %d, relres %.3e (reference %.3e)\n", k, got.iterations, res_dev, res_ref);
  }
  std::printf("ok sequence: %d of %zu systems with relres_dev > relres_ref\n", worse, seq.systems.size());

  // cgs2_orthonormalize through the adapter (tests/test_refine.cpp:34-55)
  {
    const std::size_t n = static_cast<std::size_t>(sym->n);
    DenseVector e0(n, 0.0), v(n, 0.0);
    e0[0] = 1.0;
    v[0] = 1.0;
    v[1] = 1.0;
    const Cgs2Result r = b200::cgs2_orthonormalize(dev, {e0}, v);
    if (r.breakdown || r.coefficients[0] != 1.0 || r.vector[1] != 1.0 || r.vector[0] != 0.0) return fail("cgs2 projection");
    if (!b200::cgs2_orthonormalize(dev, {e0}, e0).breakdown) return fail("cgs2 breakdown");
    std::printf("ok cgs2\n");
  }
  // error mapping: a changed pattern (numeric.cpp:15-17) and a zero pivot (numeric.cpp:48-55)
  {
    CsrMatrix bad = seq.systems[0].K;
    bad.col_indices[1] = bad.col_indices[1] == bad.col_indices[0] + 1 ? bad.col_indices[1] + 1 : bad.col_indices[0] + 1;
    bool thrown = false;
    try {
      b200::reset_values(dev, bad);
    } catch (const PatternMismatchError&) {
      thrown = true;
    }
    if (!thrown) return fail("PatternMismatchError");
    CsrMatrix zero = seq.systems[0].K;
    for (double& e : zero.values) e = 0.0;
    std::int64_t row_ref = -2, row_dev = -3;
    try {
      reset_values(cpu, zero);
      factorize_scattered(cpu);
    } catch (const ZeroPivotError& e) {
      row_ref = e.row;
    }
    try {
      b200::refactorize(dev, zero);
    } catch (const ZeroPivotError& e) {
      row_dev = e.row;
    }
    if (row_ref != row_dev) return fail("ZeroPivotError row");
    std::printf("ok errors: pattern mismatch, zero pivot at row %lld\n", static_cast<long long>(row_dev));
  }
  std::printf("all ok\n");
  return 0;
}
