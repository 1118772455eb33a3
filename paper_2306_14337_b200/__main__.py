"""`python -m paper_2306_14337_b200` — the device-path counterpart of the reference's `rlu` CLI
(proj/src/cli.cpp:216-321; same subcommands, option names, report formats and exit codes where they apply):

    solve-seq --input MANIFEST [--analyzer MODULE:FUNCTION] [--scaling mc64|none] [--ordering amd|natural]
              [--refine fgmres|classic|none] [--refine-tol T] [--refine-maxit N] [--format json|csv] [--out PATH]
              [--device D]
    report    REPORT.json [--format json|csv] [--out PATH]

`solve-seq` reads the reference's sequence format (a manifest of Matrix Market files, src/kkt.cpp:209-256,
src/io.cpp:25-87), runs cli::solve_sequence's loop (analyze once, refactorize + solve + refine per system,
escalation on failure: sequence.py) on the GPU and writes the SolveReport with the reference's field names
(src/report.cpp:30-119). Exit code 0 when every system was solved, 2 otherwise, 1 on an error — cli.cpp:304-318.

The symbolic analysis (MC64, AMD, fill pattern) defaults to the package's own host code (analysis.py over
csrc/analyze.cpp: the reference's product bit for bit); `--analyzer` substitutes another provider,
`analyze(K: CsrMatrix, use_scaling: bool, use_amd: bool) -> SymbolicFactors` — e.g. a thin binding of the
reference's symbolic_analyze. There is no `gen` subcommand (the generator is the reference's); sequences
written by `rlu gen --out DIR` load unchanged.
"""
from __future__ import annotations

import argparse
import importlib
import sys

from . import solver as rlu
from .mmio import IoError, load_sequence
from .sequence import PipelineOptions, SolveReport, solve_sequence


def _emit(text: str, out_path: str):
    if not out_path:
        sys.stdout.write(text if text.endswith("\n") else text + "\n")
        return
    try:
        with open(out_path, "w") as f:
            f.write(text if text.endswith("\n") else text + "\n")
    except OSError:
        raise IoError(f"cannot open {out_path} for writing")


def _load_callable(spec: str):
    mod, _, fn = spec.partition(":")
    if not mod or not fn:
        raise rlu.Error("--analyzer expects MODULE:FUNCTION")
    return getattr(importlib.import_module(mod), fn)


def _builtin_analyze(K, use_scaling: bool, use_amd: bool):
    from .analysis import AnalyzeOptions, symbolic_analyze
    return symbolic_analyze(K, AnalyzeOptions(use_scaling, use_amd))


def run_cli(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2306_14337_b200",
                                 description="sparse LU refactorization solver for fixed-pattern KKT sequences (B200 path)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    solve = sub.add_parser("solve-seq", help="solve a sequence, analyzing once and refactorizing the rest")
    solve.add_argument("--input", required=True, help="sequence manifest file")
    solve.add_argument("--analyzer", default="", help="MODULE:FUNCTION providing the host-side symbolic analysis "
                       "(default: the built-in analysis)")
    solve.add_argument("--scaling", default="mc64", choices=["mc64", "none"])
    solve.add_argument("--ordering", default="amd", choices=["amd", "natural"])
    solve.add_argument("--refine", default="none", choices=["fgmres", "classic", "none"])
    solve.add_argument("--refine-tol", type=float, default=1e-14)
    solve.add_argument("--refine-maxit", type=int, default=20)
    solve.add_argument("--format", default="json", choices=["json", "csv"])
    solve.add_argument("--out", default="")
    solve.add_argument("--device", type=int, default=0)
    rep_cmd = sub.add_parser("report", help="render a JSON report as CSV or JSON")
    rep_cmd.add_argument("input", help="report JSON file")
    rep_cmd.add_argument("--format", default="json", choices=["json", "csv"])
    rep_cmd.add_argument("--out", default="")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 1
    try:
        if args.cmd == "solve-seq":
            analyze = _load_callable(args.analyzer) if args.analyzer else _builtin_analyze
            systems = load_sequence(args.input)
            opt = PipelineOptions(use_scaling=args.scaling == "mc64", use_amd=args.ordering == "amd", refine=args.refine,
                                  refine_tol=args.refine_tol, refine_maxit=args.refine_maxit, device=args.device)
            rep = solve_sequence(systems, analyze, opt)
            _emit(rep.to_json() if args.format == "json" else rep.to_csv(), args.out)
            return 0 if rep.systems_solved == len(rep.systems) else 2
        try:
            text = open(args.input).read()
        except OSError:
            raise IoError(f"cannot open {args.input}")
        rep = SolveReport.from_json(text)
        _emit(rep.to_json() if args.format == "json" else rep.to_csv(), args.out)
        return 0
    except rlu.Error as e:
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(run_cli())
