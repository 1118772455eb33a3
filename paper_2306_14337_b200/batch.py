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


# ----------------------------------------------------------------------------------------------
# Interleaved scenario batches: ONE handle, all scenarios factorized and solved together
# (include/b200lu.h, b200lu_batch_*; kernels in csrc/batch.cuh).

import ctypes as C

import numpy as np

from . import _capi


def _symbolic_view(sym: rlu.SymbolicFactors):
    v = _capi.SymbolicView()
    v.n = sym.n
    v.nnz_factors = int(sym.row_offsets[-1]) if len(sym.row_offsets) else 0
    v.nnz_source = len(sym.scatter_map)
    v.row_offsets, v.col_indices, v.diag_pos = (a.ctypes.data for a in (sym.row_offsets, sym.col_indices, sym.diag_pos))
    v.scatter_map, v.scatter_scale, v.amd_forward = (a.ctypes.data for a in (sym.scatter_map, sym.scatter_scale, sym.amd_forward))
    v.source_row_offsets, v.source_col_indices = sym.src_row_offsets.ctypes.data, sym.src_col_indices.ctypes.data
    if sym.col_perm_forward is not None:
        v.col_perm_forward = sym.col_perm_forward.ctypes.data
        v.row_scale = sym.row_scale.ctypes.data
        v.col_scale = sym.col_scale.ctypes.data
    return v


_OUTCOME_DTYPE = np.dtype({"names": ["iterations", "converged", "history_len", "residual_history"],
                           "formats": [np.int32, np.int32, np.int32, (np.float64, 66)],
                           "offsets": [_capi.RefineOutcome.iterations.offset, _capi.RefineOutcome.converged.offset,
                                       _capi.RefineOutcome.history_len.offset, _capi.RefineOutcome.residual_history.offset],
                           "itemsize": C.sizeof(_capi.RefineOutcome)})


class BatchedFactors:
    """`batch` NumericFactors (include/rlu/numeric.hpp:22-31) over one SymbolicFactors, stored
    scenario-interleaved on the device. Value arrays are [batch, nnz(A)], vectors [batch, n]
    (numpy arrays, or contiguous float64 CUDA tensors used in place). Every scenario's L/U values,
    triangular solves and SpMV are bit-identical to the reference's single-system results."""

    def __init__(self, sym: rlu.SymbolicFactors, batch: int, options: rlu.FactorOptions | None = None):
        self.symbolic = sym
        self.batch = int(batch)
        self.options = options or rlu.FactorOptions()
        self._h = C.c_void_p()
        L = _capi.lib()
        v = _symbolic_view(sym)
        o = _capi.Options()
        L.b200lu_default_options(C.byref(o))
        o.pivot_floor = self.options.pivot_floor
        o.device = self.options.device
        o.stream = self.options.stream
        o.refine_capacity = self.options.refine_capacity
        st = L.b200lu_batch_create(C.byref(v), C.byref(o), self.batch, C.byref(self._h))
        if st != _capi.OK:
            msg = L.b200lu_batch_last_error(self._h).decode() if self._h else ""
            if self._h:
                L.b200lu_batch_destroy(self._h)
                self._h = C.c_void_p()
            if st == _capi.NO_DEVICE:
                raise rlu.DeviceError("no CUDA device: the b200lu path has no CPU fallback")
            raise (rlu.DeviceError if st == _capi.CUDA_ERROR else rlu.Error)(
                f"b200lu_batch_create: {L.b200lu_status_string(st).decode()}: {msg}")
        self._verified = set()

    def close(self):
        if getattr(self, "_h", None):
            _capi.lib().b200lu_batch_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- plumbing ------------------------------------------------------------
    def _check(self, st, failed=None):
        if st == _capi.OK:
            return
        L = _capi.lib()
        msg = L.b200lu_batch_last_error(self._h).decode() or L.b200lu_status_string(st).decode()
        if st == _capi.ZERO_PIVOT:
            rows = [] if failed is None else [int(r) for r in failed]
            bad = [s for s, r in enumerate(rows) if r >= 0]
            e = rlu.ZeroPivotError(msg, rows[bad[0]] if bad else -1)
            e.rows = rows            # per scenario, -1 = factorized
            e.scenarios = bad
            raise e
        if st == _capi.PATTERN_MISMATCH:
            raise rlu.PatternMismatchError("matrix pattern differs from the analyzed pattern")
        if st == _capi.DIMENSION:
            raise rlu.DimensionError(msg)
        if st in (_capi.CUDA_ERROR, _capi.NO_DEVICE):
            raise rlu.DeviceError(msg)
        raise rlu.Error(msg)

    def _arr_in(self, a, width, what):
        """[batch, width] array -> (pointer, on_device, keepalive)."""
        if rlu._is_device_tensor(a):
            import torch
            if a.dtype != torch.float64 or not a.is_contiguous() or a.numel() != self.batch * width:
                raise rlu.DimensionError(f"{what}: expected a contiguous float64 [{self.batch}, {width}] tensor")
            return a.data_ptr(), 1, a
        h = np.ascontiguousarray(a, dtype=np.float64)
        if h.size != self.batch * width:
            raise rlu.DimensionError(f"{what}: expected [{self.batch}, {width}] values, got {h.size}")
        return h.ctypes.data, 0, h

    def _vec_out(self, like):
        n = self.symbolic.n
        if rlu._is_device_tensor(like):
            import torch
            out = torch.empty((self.batch, n), dtype=torch.float64, device=like.device)
            return out.data_ptr(), out
        out = np.empty((self.batch, n), dtype=np.float64)
        return out.ctypes.data, out

    def check_pattern(self, row_offsets, col_indices):
        """pattern_equal guard of scatter_values (src/numeric.cpp:15-17)."""
        ro, ci = rlu._i64(row_offsets), rlu._i64(col_indices)
        st = _capi.PATTERN_MISMATCH
        if ro.size == self.symbolic.n + 1 and ci.size == len(self.symbolic.src_col_indices):
            st = _capi.lib().b200lu_batch_check_pattern(self._h, self.symbolic.n, ro.ctypes.data, ci.ctypes.data)
        self._check(st)

    # -- the reference's calls, per scenario -----------------------------------
    def reset_values(self, values):
        p, dev, keep = self._arr_in(values, len(self.symbolic.scatter_map), "reset_values")
        self._check(_capi.lib().b200lu_batch_reset_values(self._h, p, dev))

    def kkt_bind(self, n_primal: int, h_diag, diag_source_pos):
        """b200lu_batch_kkt_bind: H's own diagonal and the position of every K_ii in source-CSR order."""
        hd, pos = rlu._f64(h_diag), rlu._i64(diag_source_pos)
        if hd.size != n_primal or pos.size != self.symbolic.n:
            raise rlu.DimensionError("kkt_bind: h_diag needs n_primal entries, diag_source_pos needs n")
        self._check(_capi.lib().b200lu_batch_kkt_bind(self._h, n_primal, hd.ctypes.data, pos.ctypes.data))
        self._kkt_n_primal = n_primal

    def kkt_update(self, d_y, delta_p: float, delta_d: float):
        """assemble_kkt's value path on the device for every scenario (src/kkt.cpp:53-77): d_y is
        [batch, n_primal]; replaces reset_values for scenarios that differ from the loaded values only
        in their barrier diagonal / regularization. Follow with factorize_scattered."""
        p, dev, keep = self._arr_in(d_y, getattr(self, "_kkt_n_primal", -1), "kkt_update")
        self._check(_capi.lib().b200lu_batch_kkt_update(self._h, p, dev, float(delta_p), float(delta_d)))

    def factorize_scattered(self):
        failed = np.full(self.batch, -1, dtype=np.int64)
        self._check(_capi.lib().b200lu_batch_factorize_scattered(self._h, failed.ctypes.data), failed)

    def refactorize(self, values, raise_on_zero_pivot=True):
        """refactorize (src/numeric.cpp:70-73) for every scenario. Returns the per-scenario failed
        rows (-1 = factorized); raises ZeroPivotError (with .rows / .scenarios) unless told not to."""
        p, dev, keep = self._arr_in(values, len(self.symbolic.scatter_map), "refactorize")
        failed = np.full(self.batch, -1, dtype=np.int64)
        st = _capi.lib().b200lu_batch_refactorize(self._h, p, dev, failed.ctypes.data)
        if st == _capi.ZERO_PIVOT and not raise_on_zero_pivot:
            return failed
        self._check(st, failed)
        return failed

    def valid(self, scenario: int) -> bool:
        return bool(_capi.lib().b200lu_batch_valid(self._h, scenario))

    def values(self, scenario: int) -> np.ndarray:
        out = np.empty(int(self.symbolic.row_offsets[-1]) if self.symbolic.n else 0, dtype=np.float64)
        self._check(_capi.lib().b200lu_batch_get_values(self._h, scenario, out.ctypes.data))
        return out

    def lower_solve(self, y):
        p, dev, keep = self._arr_in(y, self.symbolic.n, "lower_solve")
        po, out = self._vec_out(y)
        self._check(_capi.lib().b200lu_batch_lower_solve(self._h, p, po, dev))
        return out

    def upper_solve(self, y):
        p, dev, keep = self._arr_in(y, self.symbolic.n, "upper_solve")
        po, out = self._vec_out(y)
        failed = np.full(self.batch, -1, dtype=np.int64)
        self._check(_capi.lib().b200lu_batch_upper_solve(self._h, p, po, dev, failed.ctypes.data), failed)
        return out

    def solve_system(self, b):
        p, dev, keep = self._arr_in(b, self.symbolic.n, "solve_system")
        po, out = self._vec_out(b)
        failed = np.full(self.batch, -1, dtype=np.int64)
        self._check(_capi.lib().b200lu_batch_solve(self._h, p, po, dev, failed.ctypes.data), failed)
        return out

    def relative_residual(self, x, b) -> np.ndarray:
        px, dev, k1 = self._arr_in(x, self.symbolic.n, "relative_residual")
        pb, dev2, k2 = self._arr_in(b, self.symbolic.n, "relative_residual")
        if dev != dev2:
            raise rlu.Error("relative_residual: x and b must both be host arrays or both device tensors")
        out = np.empty(self.batch, dtype=np.float64)
        self._check(_capi.lib().b200lu_batch_relative_residual(self._h, px, pb, dev, out.ctypes.data))
        return out

    def classic_refine(self, b, x0, config: rlu.RefineConfig | None = None, preconditioned: bool = True):
        """classic_refine (src/refine.cpp:150-188) per scenario. Returns (x [batch, n], outcomes)."""
        return self._refine("b200lu_batch_refine_classic", b, x0, config, preconditioned)

    def fgmres_refine(self, b, x0, config: rlu.RefineConfig | None = None, preconditioned: bool = True):
        """fgmres_refine (src/refine.cpp:39-142) per scenario. Returns (x [batch, n], outcomes)."""
        return self._refine("b200lu_batch_refine_fgmres", b, x0, config, preconditioned)

    def _refine(self, fn_name, b, x0, config, preconditioned):
        config = config or rlu.RefineConfig()
        pb, dev, k1 = self._arr_in(b, self.symbolic.n, "fgmres_refine")
        px, dev2, k2 = self._arr_in(x0, self.symbolic.n, "fgmres_refine")
        if dev != dev2:
            raise rlu.Error("refine: b and x0 must both be host arrays or both device tensors")
        po, out = self._vec_out(b)
        cfg = _capi.RefineConfig(config.max_iterations, config.tolerance)
        ocs = (_capi.RefineOutcome * self.batch)()
        self._check(getattr(_capi.lib(), fn_name)(self._h, pb, px, po, dev, 1 if preconditioned else 0,
                                                  C.byref(cfg), C.cast(ocs, C.c_void_p)))
        return out, self._outcomes(ocs, out)

    def _outcomes(self, ocs, out):
        """RefineOutcome per scenario from the C records: one numpy view of the records instead of 256 x (tensor
        indexing + ctypes field reads) — at C2 x 256 those per-scenario Python objects cost more host time than the
        three read-backs of the refinement itself."""
        rec = np.frombuffer(ocs, dtype=_OUTCOME_DTYPE, count=self.batch)
        its, conv, hl, hist = rec["iterations"].tolist(), rec["converged"].tolist(), rec["history_len"].tolist(), rec["residual_history"]
        xs = out.unbind(0) if hasattr(out, "unbind") else out
        return [rlu.RefineOutcome(xs[s], its[s], hist[s, :hl[s]].tolist(), bool(conv[s])) for s in range(self.batch)]

    # -- staged (pipelined) submission ------------------------------------------
    def _host_ptr(self, a, width, what):
        """Buffer of a staged call — numpy array or CPU torch tensor (ideally page-locked), or a CUDA tensor on the handle's
        device — -> (pointer, keepalive)."""
        if a is None:
            return None, None
        if hasattr(a, "data_ptr") and not rlu._is_device_tensor(a):  # CPU torch tensor (pin_memory() keeps copies async)
            import torch
            if a.dtype != torch.float64 or not a.is_contiguous() or a.numel() != self.batch * width:
                raise rlu.DimensionError(f"{what}: expected a contiguous float64 [{self.batch}, {width}] tensor")
            return a.data_ptr(), a
        if rlu._is_device_tensor(a):  # memory of the handle's device: the staged copies are device-to-device then
            import torch
            if a.dtype != torch.float64 or not a.is_contiguous() or a.numel() != self.batch * width:
                raise rlu.DimensionError(f"{what}: expected a contiguous float64 [{self.batch}, {width}] tensor")
            return a.data_ptr(), a
        h = np.ascontiguousarray(a, dtype=np.float64)
        if h.size != self.batch * width:
            raise rlu.DimensionError(f"{what}: expected [{self.batch}, {width}] values, got {h.size}")
        return h.ctypes.data, h

    def stage_inputs(self, values=None, rhs=None):
        """Starts the host-to-device copy of the NEXT batch's values and/or right-hand sides on the handle's
        copy stream and returns at once (b200lu_batch_stage_inputs). The buffers must stay alive and
        unchanged until the matching *_staged call has been issued and the device has caught up."""
        pv, kv = self._host_ptr(values, len(self.symbolic.scatter_map), "stage_inputs")
        pr, kr = self._host_ptr(rhs, self.symbolic.n, "stage_inputs")
        self._staged_keep = getattr(self, "_staged_keep", [])[-4:] + [kv, kr]
        self._check(_capi.lib().b200lu_batch_stage_inputs(self._h, pv, pr))

    def refactorize_staged(self, raise_on_zero_pivot=True):
        """refactorize (src/numeric.cpp:70-73) on the staged values."""
        failed = np.full(self.batch, -1, dtype=np.int64)
        st = _capi.lib().b200lu_batch_refactorize_staged(self._h, failed.ctypes.data)
        if st == _capi.ZERO_PIVOT and not raise_on_zero_pivot:
            return failed
        self._check(st, failed)
        return failed

    def solve_refine_staged(self, out, config: rlu.RefineConfig | None = None, refine: bool = True):
        """solve_system on the staged right-hand sides, then fgmres_refine from that solution; the result is
        copied into the host buffer `out` ([batch, n]) asynchronously: read it after staged_wait().
        Returns the refinement outcomes (their .x is a view of `out`)."""
        po, keep = self._host_ptr(out, self.symbolic.n, "solve_refine_staged")
        config = config or rlu.RefineConfig()
        cfg = _capi.RefineConfig(config.max_iterations, config.tolerance)
        ocs = (_capi.RefineOutcome * self.batch)()
        failed = np.full(self.batch, -1, dtype=np.int64)
        self._check(_capi.lib().b200lu_batch_solve_refine_staged(self._h, 1 if refine else 0, C.byref(cfg), po,
                                                                 C.cast(ocs, C.c_void_p), failed.ctypes.data), failed)
        if not refine:
            return []
        return self._outcomes(ocs, out if not isinstance(out, np.ndarray) or out.ndim == 2 else out.reshape(self.batch, -1))

    def staged_wait(self):
        self._check(_capi.lib().b200lu_batch_staged_wait(self._h))

    # -- reporting -------------------------------------------------------------
    @property
    def info(self) -> dict:
        s = _capi.BatchInfo()
        self._check(_capi.lib().b200lu_batch_get_info(self._h, C.byref(s)))
        return {k: int(getattr(s, k)) for k, _ in _capi.BatchInfo._fields_}

    def set_timing(self, enabled: bool = True):
        self._check(_capi.lib().b200lu_batch_set_timing(self._h, 1 if enabled else 0))

    def phase_times(self, reset: bool = True) -> dict:
        n = len(_capi.PHASES)
        ms, cnt = (C.c_double * n)(), (C.c_int64 * n)()
        self._check(_capi.lib().b200lu_batch_get_phase_times(self._h, ms, cnt, 1 if reset else 0))
        return {p: (float(ms[i]), int(cnt[i])) for i, p in enumerate(_capi.PHASES)}

    def synchronize(self):
        self._check(_capi.lib().b200lu_batch_synchronize(self._h))
