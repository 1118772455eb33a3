"""Sequence driver: cli::solve_sequence (reference proj/src/cli.cpp:57-173) over the device path.

Analyze once, then per system reset_values -> factorize_scattered -> solve_system -> refinement,
with the reference's escalation policy on a zero pivot or a residual above kAcceptRelres: first
doubled regularization (generated sequences only, cli.cpp:148-154), then a fresh analysis of the
current system, then "failed". The symbolic analysis is NOT part of this package — it stays the
reference's host code — so the caller passes it in as `analyze(K) -> SymbolicFactors`.

For a generated sequence whose KKT blocks are known (`KktDiagonal`), every system after the first
one of a pattern is submitted through the device-resident value path (b200lu_kkt_update): only D_y
crosses the bus, and the regularization escalation is a device-side diagonal rewrite.

The report carries the reference's field names (include/rlu/report.hpp:14-48, src/report.cpp:30-66).
"""
from __future__ import annotations

import json
import math
import time
from dataclasses import asdict, dataclass, field

import numpy as np

from . import solver as rlu

K_ACCEPT_RELRES = 1e-8  # include/rlu/cli.hpp:25


@dataclass
class PipelineOptions:
    """cli::PipelineOptions (include/rlu/cli.hpp:13-22); ExecPolicy is CPU-specific. use_scaling /
    use_amd are handed to the caller's analyze()."""
    use_scaling: bool = True
    use_amd: bool = True
    refine: str = "none"          # "none" | "fgmres" | "classic"
    refine_tol: float = 1e-14
    refine_maxit: int = 20
    pivot_floor: float = 1e-30
    device: int = 0


@dataclass
class SystemRecord:
    """rlu::SystemRecord (include/rlu/report.hpp:14-27)."""
    k: int = 0
    n: int = 0
    nnz: int = 0
    analyze_ms: float = 0.0
    scatter_ms: float = 0.0
    factor_ms: float = 0.0
    trisolve_ms: float = 0.0
    refine_ms: float = 0.0
    refine_iters: int = 0
    relres_direct: float = 0.0
    relres_final: float = 0.0
    status: str = "ok"


@dataclass
class SolveReport:
    """rlu::SolveReport (include/rlu/report.hpp:29-41)."""
    systems: list = field(default_factory=list)
    total_ms: float = 0.0
    mean_analyze_ms: float = 0.0
    mean_scatter_ms: float = 0.0
    mean_factor_ms: float = 0.0
    mean_trisolve_ms: float = 0.0
    mean_refine_ms: float = 0.0
    systems_solved: int = 0
    reanalysis_count: int = 0

    def finalize(self):  # src/report.cpp:11-28
        count = float(len(self.systems)) if self.systems else 1.0
        for name in ("analyze", "scatter", "factor", "trisolve", "refine"):
            setattr(self, f"mean_{name}_ms", sum(getattr(r, f"{name}_ms") for r in self.systems) / count)
        self.systems_solved = sum(1 for r in self.systems if r.status == "ok")

    def to_json(self) -> str:  # report_to_json, src/report.cpp:30-66: same keys, same nesting
        return json.dumps({
            "systems": [asdict(r) for r in self.systems],
            "aggregate": {"total_ms": self.total_ms,
                          "mean_phase_ms": {"analyze": self.mean_analyze_ms, "scatter": self.mean_scatter_ms,
                                            "factor": self.mean_factor_ms, "trisolve": self.mean_trisolve_ms,
                                            "refine": self.mean_refine_ms},
                          "systems_solved": self.systems_solved, "reanalysis_count": self.reanalysis_count}}, indent=2)


    def to_csv(self) -> str:  # report_to_csv, src/report.cpp:100-119: same header, %.17g numbers, '#' trailer
        def g(x):
            return f"{x:.17g}"
        out = ["k,n,nnz,analyze_ms,scatter_ms,factor_ms,trisolve_ms,refine_ms,refine_iters,relres_direct,relres_final,status"]
        for r in self.systems:
            out.append(",".join([str(r.k), str(r.n), str(r.nnz), g(r.analyze_ms), g(r.scatter_ms), g(r.factor_ms),
                                 g(r.trisolve_ms), g(r.refine_ms), str(r.refine_iters), g(r.relres_direct),
                                 g(r.relres_final), r.status]))
        out.append("# total_ms," + g(self.total_ms))
        for name in ("analyze", "scatter", "factor", "trisolve", "refine"):
            out.append(f"# mean_{name}_ms," + g(getattr(self, f"mean_{name}_ms")))
        out.append(f"# systems_solved,{self.systems_solved}")
        out.append(f"# reanalysis_count,{self.reanalysis_count}")
        return "\n".join(out) + "\n"

    @staticmethod
    def from_json(text: str) -> "SolveReport":  # report_from_json, src/report.cpp:68-98
        try:
            d = json.loads(text)
            rep = SolveReport()
            for jr in d["systems"]:
                rep.systems.append(SystemRecord(**{k: jr[k] for k in SystemRecord.__dataclass_fields__}))
            agg = d["aggregate"]
            rep.total_ms = float(agg["total_ms"])
            for name in ("analyze", "scatter", "factor", "trisolve", "refine"):
                setattr(rep, f"mean_{name}_ms", float(agg["mean_phase_ms"][name]))
            rep.systems_solved = int(agg["systems_solved"])
            rep.reanalysis_count = int(agg["reanalysis_count"])
            return rep
        except (KeyError, TypeError, ValueError) as e:
            raise rlu.Error(f"malformed report: {e}")


@dataclass
class KktSystem:
    """rlu::KktSystem (include/rlu/kkt.hpp:23-28)."""
    K: rlu.CsrMatrix
    rhs: np.ndarray
    k: int = 0
    mu: float = 0.0


@dataclass
class KktDiagonal:
    """What the device value path needs of the sequence's KktBlocks (include/rlu/kkt.hpp:14-21):
    H's own diagonal and, per system, D_y and the two regularization shifts."""
    n_primal: int
    h_diag: np.ndarray
    d_y: list
    delta_p: list
    delta_d: list


def doubled(delta: float) -> float:
    """src/cli.cpp:53."""
    return 1e-12 if delta == 0.0 else 2.0 * delta


def _diag_positions(K: rlu.CsrMatrix) -> np.ndarray:
    ro, ci = np.asarray(K.row_offsets), np.asarray(K.col_indices)
    rows = np.repeat(np.arange(K.nrows), np.diff(ro))
    pos = np.nonzero(rows == ci)[0]
    if pos.size != K.nrows:
        raise rlu.Error("KKT matrix must store every diagonal entry (include/rlu/kkt.hpp:43-46)")
    return pos


def _ms(t0: float) -> float:
    return (time.perf_counter() - t0) * 1e3


def solve_sequence(systems: list, analyze, options: PipelineOptions | None = None,
                   blocks: KktDiagonal | None = None, keep_solutions: bool = False):
    """cli::solve_sequence. `systems`: KktSystem list with one pattern (until it changes);
    `analyze(K, use_scaling, use_amd) -> SymbolicFactors`; `blocks`: present for generated sequences
    (enables the regularization step of the escalation and the diagonal-only value path).
    Returns SolveReport (and the solutions when keep_solutions)."""
    opt = options or PipelineOptions()
    t_total = time.perf_counter()
    rep = SolveReport()
    sym = None
    numeric: rlu.NumericFactors | None = None
    cfg = rlu.RefineConfig(opt.refine_maxit, opt.refine_tol)
    solutions = []
    resident = False  # the handle holds a full set of values of the current pattern
    deltas = None if blocks is None else [list(blocks.delta_p), list(blocks.delta_d)]

    def same_pattern(K):
        return (sym is not None and K.nrows == sym.n and np.array_equal(K.row_offsets, sym.src_row_offsets)
                and np.array_equal(K.col_indices, sym.src_col_indices))

    for sys_ in systems:
        r = SystemRecord(k=sys_.k, n=sys_.K.nrows, nnz=int(np.size(sys_.K.col_indices)))
        reg_doubled = reanalyzed = force_analyze = solved = False
        x = None
        while not solved:
            attempt_failed = False
            try:
                pattern_changed = sym is not None and not same_pattern(sys_.K)
                if pattern_changed:
                    rep.reanalysis_count += 1
                if sym is None or pattern_changed or force_analyze:
                    force_analyze = False
                    t = time.perf_counter()
                    sym = analyze(sys_.K, opt.use_scaling, opt.use_amd)
                    if numeric is not None:
                        numeric.close()
                    numeric = rlu.NumericFactors(sym, rlu.FactorOptions(pivot_floor=opt.pivot_floor, device=opt.device,
                                                                        refine_capacity=max(opt.refine_maxit, 1)))
                    if blocks is not None:
                        rlu.kkt_bind(numeric, blocks.n_primal, blocks.h_diag, _diag_positions(sys_.K))
                    resident = False
                    r.analyze_ms += _ms(t)

                t = time.perf_counter()
                if blocks is not None and resident:
                    # same pattern as the resident values, which differ only in the diagonal: D_y of this
                    # system and the (possibly doubled) regularization are written on the device
                    rlu.kkt_update(numeric, blocks.d_y[sys_.k], deltas[0][sys_.k], deltas[1][sys_.k])
                else:
                    rlu.reset_values(numeric, sys_.K)
                    resident = True
                    if blocks is not None and reg_doubled:  # sys.K = assemble_kkt(doubled blocks), cli.cpp:152-153
                        rlu.kkt_update(numeric, blocks.d_y[sys_.k], deltas[0][sys_.k], deltas[1][sys_.k])
                numeric.synchronize()
                r.scatter_ms += _ms(t)

                t = time.perf_counter()
                rlu.factorize_scattered(numeric)
                r.factor_ms += _ms(t)

                t = time.perf_counter()
                x = rlu.solve_system(numeric, sys_.rhs)
                r.trisolve_ms += _ms(t)

                r.relres_direct = rlu.relative_residual(numeric, x, sys_.rhs)
                r.relres_final = r.relres_direct
                r.refine_iters = 0
                if opt.refine != "none":
                    t = time.perf_counter()
                    out = (rlu.fgmres_refine if opt.refine == "fgmres" else rlu.classic_refine)(numeric, sys_.rhs, x, cfg)
                    r.refine_ms += _ms(t)
                    r.refine_iters = out.iterations
                    x = out.x
                    r.relres_final = rlu.relative_residual(numeric, x, sys_.rhs)
                solved = math.isfinite(r.relres_final) and r.relres_final <= K_ACCEPT_RELRES
                attempt_failed = not solved
            except rlu.Error:
                # zero pivot, or an analysis that failed outright: same escalation (cli.cpp:140-144)
                attempt_failed = True
            if not attempt_failed:
                break
            if blocks is not None and not reg_doubled:
                reg_doubled = True
                deltas[0][sys_.k] = doubled(deltas[0][sys_.k])
                deltas[1][sys_.k] = doubled(deltas[1][sys_.k])
            elif not reanalyzed:
                reanalyzed = True
                force_analyze = True
                rep.reanalysis_count += 1
            else:
                r.status = "failed"
                break
        if solved:
            r.status = "ok"
        rep.systems.append(r)
        if keep_solutions:
            solutions.append(x)
    if numeric is not None:
        numeric.close()
    rep.total_ms = _ms(t_total)
    rep.finalize()
    return (rep, solutions) if keep_solutions else rep
