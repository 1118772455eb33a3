"""Scenario batches on one GPU: many independent systems that share one sparsity pattern.

A single factorization is bound by its dependency chain, not by the machine: while
one system walks its 1,000+ dependency levels most SMs idle. Independent scenario / contingency
systems fill that idle time: `ScenarioBatch` keeps `streams` handles — one CUDA stream
each, created with `FactorOptions(concurrency=streams)` so their persistent kernels share the SMs
— and a host thread per handle (the C ABI calls release the GIL), and pushes the scenarios through
refactorize -> solve_system -> fgmres_refine concurrently. Every scenario is processed by exactly
one handle from start to finish, so its result is bit-identical to a lone run with the same options.
"""
from __future__ import annotations

import queue
import threading

from . import solver as rlu
from .sharding import SystemRecord


class ScenarioBatch:
    def __init__(self, sym: rlu.SymbolicFactors, streams: int = 8, device: int = 0,
                 options: rlu.FactorOptions | None = None):
        import torch
        base = options or rlu.FactorOptions()
        self.device = device
        self.streams = [torch.cuda.Stream(device=device) for _ in range(streams)]
        self.handles = [
            rlu.NumericFactors(sym, rlu.FactorOptions(pivot_floor=base.pivot_floor, device=device,
                                                      stream=s.cuda_stream, refine_capacity=base.refine_capacity,
                                                      strict_order=base.strict_order, concurrency=streams))
            for s in self.streams
        ]

    def close(self):
        for h in self.handles:
            h.close()
        self.handles = []

    def run(self, matrices, rhs, refine: bool = True, config: rlu.RefineConfig | None = None,
            keep_x: bool = True):
        """matrices[s]: CsrMatrix of scenario s (values on the host or on the device); rhs[s]: its
        right-hand side (numpy array or CUDA tensor). Returns (records, xs) ordered by scenario."""
        import torch
        n = len(matrices)
        todo: "queue.SimpleQueue[int]" = queue.SimpleQueue()
        for s in range(n):
            todo.put(s)
        records = [None] * n
        xs = [None] * n
        errors = []

        def worker(slot: int):
            f = self.handles[slot]
            with torch.cuda.stream(self.streams[slot]):
                while True:
                    try:
                        s = todo.get_nowait()
                    except queue.Empty:
                        return
                    try:
                        failed = -1
                        try:
                            rlu.refactorize(f, matrices[s])
                        except rlu.ZeroPivotError as e:
                            failed = e.row
                            records[s] = SystemRecord(s, float("nan"), float("nan"), 0, failed)
                            continue
                        x = rlu.solve_system(f, rhs[s])
                        direct = rlu.relative_residual(f, x, rhs[s])
                        its, final = 0, direct
                        if refine:
                            out = rlu.fgmres_refine(f, rhs[s], x, config)
                            x, its = out.x, out.iterations
                            final = min(direct, out.residual_history[-1]) if out.residual_history else direct
                            final = rlu.relative_residual(f, x, rhs[s])
                        records[s] = SystemRecord(s, direct, final, its, failed)
                        if keep_x:
                            xs[s] = x
                    except Exception as e:  # noqa: BLE001 - reported to the caller below
                        errors.append((s, e))
                        return

        threads = [threading.Thread(target=worker, args=(k,), daemon=True) for k in range(len(self.handles))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errors:
            s, e = errors[0]
            raise RuntimeError(f"scenario {s} failed: {e}") from e
        return records, xs
