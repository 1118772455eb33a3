#!/usr/bin/env python
"""Headline benchmark: refactorize + solve (+ FGMRES) per KKT system, systems/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5] [--impl b200|reference]

Workloads (BASELINE.json configs):
  C5 (default)  a batch of independent ACTIVSg2000-shaped scenario systems per GPU (256 by default)
                that share one pattern and one symbolic analysis; one "step" takes the whole batch
                through the hot path with the interleaved scenario-batch kernels
                (b200lu_batch_*): value scatter, numeric refactorization, solve_system, FGMRES
                refinement — per scenario exactly what cli::solve_sequence does for one system
                (reference proj/src/cli.cpp:105-135). The same line carries `single_system`: one
                ACTIVSg10k-shaped system (C3) through the single-system kernels, i.e. the latency
                of one refactor+solve.
  C1..C4        one system per step through the single-system kernels.

Inputs are the reference's own synthetic generator (gen_sequence, proj/src/kkt.cpp:94-207) and its
host-side symbolic analysis, produced once before the timed region through the reference bridge
(input fixture, not the measured path).

  value   device-resident: values and rhs already in HBM, x stays in HBM.
  e2e     same steps through the public API with HOST buffers: values + rhs copied H2D from pinned
          memory and x copied D2H inside the timed region, every step.
  --impl reference   the unmodified reference CPU implementation (oracle/_ref) on this box's cores.

Multi-GPU (BASELINE config 5: "batch of 256 ... sharded over 1/2/4/8 B200"): `--gpus N` shards the
`--scenarios` (256) scenarios of the batch over the N ranks in contiguous blocks — 256/N per GPU, the
total fixed: STRONG scaling — with no data-path collective; NCCL only carries the per-rank timings,
residuals and per-system records to rank 0. `--scenarios-per-gpu S` fixes the per-GPU batch instead
(weak scaling line). Without a launcher (`WORLD_SIZE` unset) and N > 1 the script re-executes itself
under `python -m torch.distributed.run --nproc-per-node N` on 127.0.0.1.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (n, m, description)  — SURVEY §8d / BASELINE.json configs
    "C1": (6300, 2700, "ACTIVSg200-shaped KKT, n+m=9000"),
    "C2": (39000, 16700, "ACTIVSg2000-shaped KKT, n+m=55700"),
    "C3": (166600, 71400, "ACTIVSg10k-shaped KKT, n+m=238000"),
    "C4": (1120000, 480000, "ACTIVSg70k-shaped KKT, n+m=1600000"),
}
BATCH_WORKLOAD = "C5"   # scenarios of C2, batched
METRIC = "systems/sec (refactor+solve+FGMRES per KKT system)"
UNIT = "systems/s"


def algorithmic_bytes(n, nnz_a, nnz_f, fgmres_iters=1):
    """SURVEY §8(d) compulsory-traffic model, int32 indices on the device."""
    scatter = 12 * nnz_a + 8 * nnz_f
    eliminate = 20 * nnz_f + 8 * n
    solve = 12 * nnz_f + 76 * n
    spmv = 12 * nnz_a + 20 * n
    j = fgmres_iters
    fgmres = (j + 2) * spmv + j * solve + 8 * n * (4 * sum(i + 1 for i in range(j)) + 6 * j + 4) if j else 2 * spmv
    return dict(scatter=scatter, eliminate=eliminate, solve=solve, spmv=spmv, fgmres=fgmres,
                total=scatter + eliminate + solve + fgmres)


def batch_algorithmic_bytes(batch, n, nnz_a, nnz_f, fgmres_iters=1):
    """per-scenario VALUE traffic of every phase, the int32 index arrays once
    per phase (they are shared by all scenarios of a launch)."""
    j = fgmres_iters
    scatter = batch * (8 * nnz_a + 8 * nnz_f) + 4 * nnz_f
    eliminate = batch * 16 * nnz_f + 4 * nnz_f + 8 * n
    solve = batch * (8 * nnz_f + 60 * n) + 4 * nnz_f + 16 * n
    spmv = batch * (8 * nnz_a + 16 * n) + 4 * nnz_a + 4 * n
    fgmres = (j + 2) * spmv + j * solve + batch * 8 * n * (4 * sum(i + 1 for i in range(j)) + 6 * j + 4) if j else 2 * spmv
    return dict(scatter=scatter, eliminate=eliminate, solve=solve, spmv=spmv, fgmres=fgmres,
                total=scatter + eliminate + solve + fgmres)


def recorded_traffic(key):
    """DRAM bytes per launch of the dominant kernel. NOT measured in this run (a bench value is never
    taken under a profiler): the figure is the one recorded by the last `ncu --set full` capture of the
    same command (tools/gpu_bench_profile.sh writes profiles/traffic.json), and the line says so."""
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(tp):
        return None, "none recorded"
    rec = json.load(open(tp)).get(key, {})
    if "factor_kernel_dram_bytes" not in rec:
        return None, "none recorded for this workload"
    return rec["factor_kernel_dram_bytes"], ("recorded constant from " + rec.get("source", "profiles/traffic.json") +
                                             " (ncu --set full capture, dram__bytes_read.sum + dram__bytes_write.sum); "
                                             "not re-measured in this run")


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks / throttle reasons sampled DURING the timed region: NVML read from a thread of this process every
    5 ms (the counters `nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.*` prints — a separate
    nvidia-smi process needs ~0.5 s before its first sample, longer than a default timed region), nvidia-smi -lms as
    the fallback when NVML cannot be loaded. `window()` brackets the timed steps: only samples taken inside it count."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    BITS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
            0x80: "hw_power_brake_slowdown"}

    def __init__(self, device_index):
        self.samples, self.t0, self.t1 = [], None, None   # (time, sm MHz, max sm MHz, reason bits)
        self.p = self.f = self.thread = None
        self.stop_flag = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            # the CUDA ordinal -> the NVML device: CUDA_VISIBLE_DEVICES may renumber (indices) or name (UUIDs) the devices
            vis = [v.strip() for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
            ent = vis[device_index] if device_index < len(vis) else str(device_index)
            if ent.isdigit():
                h = pynvml.nvmlDeviceGetHandleByIndex(int(ent))
            else:
                h = pynvml.nvmlDeviceGetHandleByUUID(ent.encode() if hasattr(ent, "encode") else ent)
            smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            reasons_fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
            period = float(os.environ.get("B200LU_BENCH_SMI_MS", "5")) / 1e3

            def run():
                while not self.stop_flag.is_set():
                    try:
                        self.samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                             smax, int(reasons_fn(h))))
                    except Exception:
                        pass
                    self.stop_flag.wait(period)
            self.source = "nvml"
            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.thread = None
        self.source = "nvidia-smi"
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "20", "-i", str(device_index)], stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.6)   # its first sample takes that long
        except Exception:
            self.p = None

    def window_start(self):
        self.t0 = time.perf_counter()

    def window_stop(self):
        self.t1 = time.perf_counter()

    def stop(self):
        if self.thread is not None:
            self.stop_flag.set()
            self.thread.join(timeout=2)
            inside = [s for s in self.samples if self.t0 is not None and self.t0 <= s[0] <= (self.t1 or 1e300)]
            use = inside or self.samples
            bits = 0
            for s in use:
                bits |= s[3]
            return {"sm_mhz": statistics.median([s[1] for s in use]) if use else None,
                    "sm_max_mhz": max(s[2] for s in use) if use else None, "samples": len(use),
                    "samples_inside_timed_region": len(inside), "source": "nvml, 5 ms period, thread of the bench process",
                    "reasons": sorted(nm for b, nm in self.BITS.items() if bits & b)}
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml and nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [r.strip().split(", ") for r in open(self.f.name) if r.strip()]
        os.unlink(self.f.name)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                smax.append(float(r[2]))
                for nm, val in zip(names, r[5:9]):
                    if val.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "source": "nvidia-smi -lms 20", "reasons": sorted(reasons)}


def nccl_init_lines():
    """The communicator lines NCCL logged at init (NCCL_DEBUG=INFO, subsystem INIT, into
    NCCL_DEBUG_FILE — set in run_b200): rank count, transport, NVLS, so the reader can check that the N
    ranks really formed one communicator."""
    path = os.environ.get("B200LU_NCCL_LOG")
    if not path or not os.path.exists(path):
        return []
    keep = []
    for ln in open(path, errors="replace"):
        if any(k in ln for k in ("nranks", "Init COMPLETE", "NVLS", "Connected all", "via P2P", "NET/")):
            keep.append(ln.strip()[:240])
    for ln in keep[:12]:
        print("[nccl] " + ln, file=sys.stderr)
    return keep[:12]


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def reference_pass(num, seq, k, refine=True):
    """One system through the reference with the best execution policy per phase (measured on this
    host: scheduled_parallel helps eliminate, hurts the triangular solves — SURVEY §6)."""
    return num.run_system(seq, k, refine=refine)


def calibrate_reference(ref_sym, seq, rb):
    """Times both ExecModes once and keeps the better one per phase (factor / solve)."""
    threads = rb.max_threads()
    num = rb.RefNumeric(ref_sym)
    seq_run = num.run_system(seq, 0)
    best = {"factor_parallel": False, "solve_parallel": False, "threads": threads,
            "sequential": {k: float(seq_run[k]) for k in ("scatter_ms", "factor_ms", "trisolve_ms", "refine_ms")}}
    if threads > 1:
        num.set_exec(True, threads)
        par_run = num.run_system(seq, 0)
        best["parallel"] = {k: float(par_run[k]) for k in ("scatter_ms", "factor_ms", "trisolve_ms", "refine_ms")}
        best["factor_parallel"] = bool(par_run["factor_ms"] < seq_run["factor_ms"])
        best["solve_parallel"] = bool(par_run["trisolve_ms"] + par_run["refine_ms"]
                                      < seq_run["trisolve_ms"] + seq_run["refine_ms"])
    num.set_exec(best["factor_parallel"], threads)
    num.set_solve_exec(best["solve_parallel"], threads)
    return num, best



def analyze_for_bench(rlu, rb, A, np):
    """Host-side symbolic analysis of the workload (untimed part of the fixture): the package's own
    b200lu_analyze (csrc/analyze.cpp) provides the product the GPU path runs on; the reference's symbolic_analyze
    (needed anyway by the CPU baseline) is compared with it array by array. Returns (sym, ref_sym, report)."""
    ro, ci, va = A.arrays()
    sym, tm = rlu.symbolic_analyze(rlu.CsrMatrix(A.n, A.n, ro, ci, va), rlu.AnalyzeOptions(False, True), with_times=True)
    ref_sym = rb.RefSymbolic(A, use_scaling=False, use_amd=True)
    r = ref_sym.arrays()
    same = all(np.array_equal(np.asarray(getattr(sym, k)), np.asarray(getattr(r, k)))
               for k in ("row_offsets", "col_indices", "diag_pos", "scatter_map", "scatter_scale", "amd_forward"))
    if not same:
        raise SystemExit("bench.py: b200lu_analyze and the reference's symbolic_analyze disagree")
    return sym, ref_sym, {"b200lu_analyze_ms": round(tm.total_ms, 1), "reference_symbolic_analyze_ms": round(ref_sym.analyze_ms, 1),
                          "identical_product": True, "host_threads": 1,
                          "stages_ms": {"ordering": round(tm.ordering_ms, 1), "fill": round(tm.fill_ms, 1),
                                        "scatter_map": round(tm.scatter_map_ms, 1)}}

def run_reference(args):
    """--impl reference: the unmodified reference CPU path on this box's host cores."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    from oracle import refbridge as rb
    n, m, desc = WORKLOADS[args.workload]
    seq = rb.RefSequence(n, m)
    ref_sym = rb.RefSymbolic(seq.matrix(0), use_scaling=False, use_amd=True)
    num, policy = calibrate_reference(ref_sym, seq, rb)
    nsys = len(seq)
    for w in range(args.warmup):
        num.run_system(seq, w % nsys)
    t0 = time.perf_counter()
    phases = {"scatter_ms": 0.0, "factor_ms": 0.0, "trisolve_ms": 0.0, "refine_ms": 0.0}
    worst = 0.0
    for s in range(args.steps):
        r = num.run_system(seq, s % nsys)
        for k in phases:
            phases[k] += r[k]
        worst = max(worst, r["relres_final"])
    wall = time.perf_counter() - t0
    hot_ms = sum(phases.values()) / args.steps
    value = 1000.0 / hot_ms
    cores = policy["threads"]
    sample = (f"{args.steps} systems of the {args.workload} sequence (k = 0..), one system per step; eliminate "
              f"{'scheduled_parallel x' + str(cores) if policy['factor_parallel'] else 'sequential'}, solves "
              f"{'scheduled_parallel x' + str(cores) if policy['solve_parallel'] else 'sequential'} (best mode per phase)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": hot_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {desc}; scatter+eliminate+solve_system+fgmres_refine per system "
                               "(cli.cpp:105-135 clocks); reference CPU path", "n": seq.n, "nnz": seq.nnz,
                   "nnz_factors": ref_sym.nnz_factors, "analysis": "use_scaling=false,use_amd=true"},
        "phases_ms": {k: v / args.steps for k, v in phases.items()},
        "wall_ms_per_step": 1000.0 * wall / args.steps, "worst_relres_final": worst,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample,
                         "calibration": policy},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line))


def measure_single(args, workload, steps, with_cpu_baseline):
    """One system per step through the single-system kernels. Returns the JSON line (rank 0) or None."""
    import torch
    import torch.distributed as dist

    import paper_2306_14337_b200 as rlu
    from oracle import refbridge as rb  # input fixtures + CPU baseline arm only

    rank, local_rank, world = dist_env()
    n, m, desc = WORKLOADS[workload]
    # ---- input fixture (untimed): the reference's generator + host-side symbolic analysis
    seq = rb.RefSequence(n, m, y_seed=2 + rank)
    sym, ref_sym, analysis = analyze_for_bench(rlu, rb, seq.matrix(0), np)
    ro, ci = seq.pattern()
    nsys = len(seq)
    N, nnz_a, nnz_f = seq.n, seq.nnz, ref_sym.nnz_factors

    stream = torch.cuda.current_stream()
    f = rlu.NumericFactors(sym, rlu.FactorOptions(device=local_rank, stream=stream.cuda_stream))
    cfg = rlu.RefineConfig(args.refine_maxit, args.refine_tol)

    host_vals = [torch.from_numpy(seq.values(k)).pin_memory() for k in range(nsys)]
    host_rhs = [torch.from_numpy(seq.rhs(k)).pin_memory() for k in range(nsys)]
    dev_vals = [v.cuda(non_blocking=True) for v in host_vals]
    dev_rhs = [b.cuda(non_blocking=True) for b in host_rhs]
    host_x = torch.empty(N, dtype=torch.float64).pin_memory()
    dev_b = torch.empty(N, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    torch.cuda.synchronize()

    # One CsrMatrix per system, built once: the pattern guard (pattern_equal) runs on the first
    # submission of each object, in the warm-up, as it would for a caller that keeps its matrices.
    dev_mats = [rlu.CsrMatrix(N, N, ro, ci, dev_vals[k]) for k in range(nsys)]
    host_mats = [rlu.CsrMatrix(N, N, ro, ci, host_vals[k].numpy()) for k in range(nsys)]

    def step_resident(k):
        rlu.refactorize(f, dev_mats[k])
        x = rlu.solve_system(f, dev_rhs[k])
        if args.no_refine:
            return x, 0
        out = rlu.fgmres_refine(f, dev_rhs[k], x, cfg)
        return out.x, out.iterations

    def step_e2e(k):
        # host values -> H2D inside refactorize; rhs H2D; x D2H — all on the handle's stream
        rlu.refactorize(f, host_mats[k])
        dev_b.copy_(host_rhs[k], non_blocking=True)
        x = rlu.solve_system(f, dev_b)
        its = 0
        if not args.no_refine:
            out = rlu.fgmres_refine(f, dev_b, x, cfg)
            x, its = out.x, out.iterations
        host_x.copy_(x, non_blocking=True)
        stream.synchronize()
        return host_x, its

    def timed(step_fn, steps, warmup, sample_clocks):
        for w in range(max(warmup, nsys)):  # every matrix object is submitted (and guarded) once
            step_fn(w % nsys)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        sampler = ClockSampler(local_rank) if sample_clocks else None
        if sampler:
            sampler.window_start()
        f.set_timing(True)
        launches0 = f.launch_count
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        iters = []
        for s in range(steps):
            flush.zero_()  # L2 flush between timed iterations (outside the timed pair)
            ev[s][0].record()
            _, its = step_fn(s % nsys)
            ev[s][1].record()
            iters.append(its)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if sampler:
            sampler.window_stop()
        clocks = sampler.stop() if sampler else None
        per_step = [a.elapsed_time(b) for a, b in ev]
        phases = f.phase_times()
        f.set_timing(False)
        return sum(per_step), per_step, iters, phases, f.launch_count - launches0, clocks

    total_ms, per_step, iters, phases, launches, clocks = timed(step_resident, steps, args.warmup, True)
    e2e_total_ms, e2e_steps, _, _, _, _ = timed(step_e2e, steps, max(1, args.warmup // 2), False)

    # ---- parity spot check on the last system processed (oracle/reference as the checker only)
    k_last = (steps - 1) % nsys
    x_last, _ = step_resident(k_last)
    relres = seq.matrix(k_last).relative_residual(x_last.cpu().numpy(), seq.rhs(k_last))
    st = f.stats
    f.close()

    # ---- the same step with B200LU_FLAG_STRICT_ORDER: both sweeps fold in the reference's ascending column order, so
    # solve_system is bit-identical to the CPU result (the path the bitwise parity tests run); the default above folds
    # U rows in production order and is checked on the residual. Reported beside it, never as the headline.
    strict = None
    if not args.no_refine:
        fs = rlu.NumericFactors(sym, rlu.FactorOptions(device=local_rank, stream=stream.cuda_stream, strict_order=True))

        def step_strict(k):
            rlu.refactorize(fs, dev_mats[k])
            x = rlu.solve_system(fs, dev_rhs[k])
            return rlu.fgmres_refine(fs, dev_rhs[k], x, cfg)
        for w in range(3):
            step_strict(w % nsys)
        torch.cuda.synchronize()
        sev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for s_ in range(steps):
            flush.zero_()
            sev[s_][0].record()
            out_s = step_strict(s_ % nsys)
            sev[s_][1].record()
        torch.cuda.synchronize()
        strict = {"ms_per_step": sum(a.elapsed_time(b) for a, b in sev) / steps,
                  "relres_final": float(seq.matrix((steps - 1) % nsys).relative_residual(out_s.x.cpu().numpy(), seq.rhs((steps - 1) % nsys))),
                  "note": "same step on a handle created with strict_order (B200LU_FLAG_STRICT_ORDER): lower/upper/solve_system "
                          "bit-identical to the reference (tests/test_gpu_parity.py, test_gpu_fullsize.py)"}
        fs.close()

    # ---- max over ranks
    t = torch.tensor([total_ms, e2e_total_ms, relres], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms_max, e2e_ms_max, relres_max = (float(v) for v in t.cpu())
    if rank != 0:
        return None

    ms_per_step = total_ms_max / steps
    value = world * steps / (total_ms_max / 1000.0)
    e2e_value = world * steps / (e2e_ms_max / 1000.0)
    med_iters = int(statistics.median(iters)) if iters else 0
    ab = algorithmic_bytes(N, nnz_a, nnz_f, 0 if args.no_refine else max(med_iters, 0))
    peak, peak_src = measured_peak()
    fac_ms, fac_n = phases["factor"]
    fac_avg_ms = fac_ms / max(fac_n, 1)
    achieved = ab["eliminate"] / (fac_avg_ms * 1e-3) / 1e9 if fac_avg_ms > 0 else 0.0
    traffic, traffic_src = recorded_traffic(workload)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {
            "workload": f"{workload}: {desc}; one system per step per GPU: scatter + refactorize + "
                        f"solve_system{'' if args.no_refine else ' + fgmres_refine(tol=%g)' % args.refine_tol}; "
                        "10-system mu sequence, gen_sequence defaults, AMD-only analysis (KLU-style path)",
            "n": N, "nnz": nnz_a, "nnz_factors": nnz_f, "update_pairs": st["update_pairs"],
            "levels": st["lower_levels"], "scenario_per_rank": "y_seed = 2 + rank, shared pattern",
            "l2": "256 MiB device buffer zeroed between timed steps (outside the per-step event pair); "
                  "the per-step working set (values + destination table) also exceeds the 126 MB L2",
            "timing": "per-step CUDA events on the launching stream, summed over steps; max over ranks",
        },
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms_max / steps,
                "h2d_bytes_per_step": 8 * nnz_a + 8 * N, "d2h_bytes_per_step": 8 * N,
                "note": "values + rhs from pinned host memory H2D and x D2H inside the timed region, through "
                        "the public refactorize/solve_system/fgmres_refine calls"},
        "gpu_launches": launches,
        "analysis": analysis,
        "strict_order": strict,
        "phases_ms_per_step": {p: v[0] / steps for p, v in phases.items()},
        "launches_per_step": {p: v[1] / steps for p, v in phases.items()},
        "refine_iters_median": med_iters, "relres_final_max": relres_max,
        "roofline": {
            "kernel": "factor_kernel (K2 numeric refactorization)", "bound": "hbm",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak if peak else None,
            "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": ab["eliminate"], "avg_launch_ms": fac_avg_ms,
            "bytes_model": "SURVEY 8(d): eliminate = 20*nnz(L+U) + 8*N per system, one system per launch",
            "whole_step": {"algorithmic_bytes": ab["total"],
                           "achieved_gbs": ab["total"] / (ms_per_step * 1e-3) / 1e9,
                           "frac": ab["total"] / (ms_per_step * 1e-3) / 1e9 / peak},
            "second_bound": f"critical path: {st['lower_levels']} dependency levels per sweep x 3 sweeps",
        },
    }
    if world == 1 and with_cpu_baseline:
        num, policy = calibrate_reference(ref_sym, seq, rb)
        reps = max(1, args.cpu_reps)
        tot = 0.0
        for r in range(reps):
            o = num.run_system(seq, r % nsys, refine=not args.no_refine, max_iterations=args.refine_maxit,
                               tolerance=args.refine_tol)
            tot += o["scatter_ms"] + o["factor_ms"] + o["trisolve_ms"] + o["refine_ms"]
        cpu_ms = tot / reps
        # the reference's own final residual on the system the parity spot check used (checker only)
        line["relres_final_reference_same_system"] = float(num.run_system(
            seq, k_last, refine=not args.no_refine, max_iterations=args.refine_maxit, tolerance=args.refine_tol)["relres_final"])
        line["cpu_baseline"] = {
            "value": 1000.0 / cpu_ms, "unit": UNIT, "ms_per_system": cpu_ms, "cores": policy["threads"],
            "kind": "reference",
            "sample": f"{reps} systems of the same {workload} sequence through the unmodified reference "
                      "(oracle/_ref), best ExecMode per phase after one calibration pass of each mode",
            "calibration": policy}
    return line


def measure_c3_batch(args, scenarios=64, steps=5, warmup=3):
    """The bandwidth-bound C3 figure: `scenarios` C3-shaped scenario systems (one pattern, y_seed = 2 + scenario) per
    step through the scenario-batch kernels, buffers resident in HBM, K steps through the staged submission calls under
    one event pair — the C3 counterpart of the headline, next to `single_system` (one C3 system alone, latency-bound)."""
    import torch

    import paper_2306_14337_b200 as rlu
    from paper_2306_14337_b200.batch import BatchedFactors
    from oracle import refbridge as rb  # input fixtures only

    _, local_rank, _ = dist_env()
    n, m, desc = WORKLOADS["C3"]
    seqs = [rb.RefSequence(n, m, y_seed=2 + sc, num_systems=1) for sc in range(scenarios)]
    sym, ref_sym, _ = analyze_for_bench(rlu, rb, seqs[0].matrix(0), np)
    N, nnz_a, nnz_f = seqs[0].n, seqs[0].nnz, ref_sym.nnz_factors
    stream = torch.cuda.current_stream()
    f = BatchedFactors(sym, scenarios, rlu.FactorOptions(device=local_rank, stream=stream.cuda_stream,
                                                         refine_capacity=args.refine_maxit))
    cfg = rlu.RefineConfig(args.refine_maxit, args.refine_tol)
    dev_vals = torch.from_numpy(np.stack([q.values(0) for q in seqs])).cuda()
    dev_rhs = torch.from_numpy(np.stack([q.rhs(0) for q in seqs])).cuda()
    outs = [torch.empty((scenarios, N), dtype=torch.float64, device="cuda") for _ in range(2)]

    def loop(K):
        f.stage_inputs(dev_vals, dev_rhs)
        for k in range(K):
            if k + 1 < K:
                f.stage_inputs(dev_vals, dev_rhs)
            f.refactorize_staged()
            f.solve_refine_staged(outs[k % 2], cfg, refine=not args.no_refine)
        f.staged_wait()
    loop(max(2, warmup))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    loop(steps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    # per-phase times and the residuals through the synchronous calls
    f.set_timing(True)
    f.refactorize(dev_vals)
    x = f.solve_system(dev_rhs)
    its = [0] * scenarios
    if not args.no_refine:
        x, ro = f.fgmres_refine(dev_rhs, x, cfg)
        its = [o.iterations for o in ro]
    torch.cuda.synchronize()
    phases = f.phase_times()
    f.set_timing(False)
    worst = float(f.relative_residual(x, dev_rhs).max())
    ab = batch_algorithmic_bytes(scenarios, N, nnz_a, nnz_f, int(statistics.median(its)))
    peak, peak_src = measured_peak()
    fac_ms = phases["factor"][0] / max(phases["factor"][1], 1)
    info = f.info
    f.close()
    return {"value": scenarios / (ms / 1000.0), "unit": UNIT, "ms_per_step": ms, "ms_per_system": ms / scenarios,
            "steps": steps, "warmup": warmup,
            "config": {"workload": f"C3 x {scenarios}: {scenarios} independent {desc} scenario systems in one batch on one GPU, "
                                   "same step as the headline (scatter + refactorize + solve_system + fgmres_refine) through "
                                   "the staged submission calls, buffers resident in HBM",
                       "n": N, "nnz": nnz_a, "nnz_factors": nnz_f, "device_gb": round(info["device_bytes"] / 1e9, 2)},
            "phases_ms": {p: v[0] for p, v in phases.items()}, "refine_iters_median": int(statistics.median(its)),
            "relres_final_max": worst,
            "roofline": {"kernel": "batched K2 refactorization (head + trailing launch)", "bound": "hbm",
                         "achieved": ab["eliminate"] / (fac_ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": ab["eliminate"] / (fac_ms * 1e-3) / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": ab["eliminate"], "avg_launch_ms": fac_ms,
                         "whole_step_frac": ab["total"] / (ms * 1e-3) / 1e9 / peak}}


def reference_batch_sample(rb, ref_sym, seqs, threads, refine=True, max_iterations=20, tolerance=1e-14):
    """The reference on a block of independent scenarios: one scenario per host thread, each through
    reset_values + factorize_scattered + solve_system + fgmres_refine in ExecMode::sequential (the
    calls release the GIL). Returns (wall seconds, per-scenario outcomes)."""
    from concurrent.futures import ThreadPoolExecutor
    nums = [rb.RefNumeric(ref_sym) for _ in range(threads)]

    def work(t):
        out = []
        for s in range(t, len(seqs), threads):
            out.append(nums[t].run_system(seqs[s], 0, refine=refine, max_iterations=max_iterations, tolerance=tolerance))
        return out

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(work, range(threads)))
    return time.perf_counter() - t0, [o for r in res for o in r]


def reference_batch_best(rb, ref_sym, seqs, threads, refine, max_iterations, tolerance):
    """Times the reference on the scenarios `seqs` in both of its ways of using all host threads and
    keeps the faster: (a) one scenario per thread, ExecMode::sequential inside each; (b) one scenario
    at a time with the best ExecMode per phase (scheduled_parallel elimination on all threads).
    Returns (systems/s, description, calibration dict, worst relres)."""
    wall_a, outs_a = reference_batch_sample(rb, ref_sym, seqs, threads, refine, max_iterations, tolerance)
    num, policy = calibrate_reference(ref_sym, seqs[0], rb)
    t0 = time.perf_counter()
    outs_b = [num.run_system(q, 0, refine=refine, max_iterations=max_iterations, tolerance=tolerance)
              for q in seqs[:max(2, len(seqs) // 4)]]
    hot_b = sum(o["scatter_ms"] + o["factor_ms"] + o["trisolve_ms"] + o["refine_ms"] for o in outs_b) / 1000.0
    wall_b = time.perf_counter() - t0
    rate_a, rate_b = len(seqs) / wall_a, len(outs_b) / hot_b
    cal = {"one_scenario_per_thread": {"systems_per_s": rate_a, "scenarios": len(seqs), "threads": threads},
           "one_at_a_time_best_exec_mode": {"systems_per_s": rate_b, "scenarios": len(outs_b), "policy": policy,
                                            "wall_s": wall_b}}
    if rate_a >= rate_b:
        return rate_a, (f"{len(seqs)} scenarios, one per host thread ({threads} threads, ExecMode::sequential inside "
                        "each), wall clock over the block"), cal, max(o["relres_final"] for o in outs_a)
    return rate_b, (f"{len(outs_b)} scenarios one at a time, eliminate "
                    f"{'scheduled_parallel x' + str(threads) if policy['factor_parallel'] else 'sequential'}, solves "
                    f"{'scheduled_parallel' if policy['solve_parallel'] else 'sequential'} (best mode per phase), "
                    "sum of the four phase clocks"), cal, max(o["relres_final"] for o in outs_b)


def run_batch(args):
    """Default workload: a scenario batch per GPU through the interleaved batch kernels."""
    import torch
    import torch.distributed as dist

    import paper_2306_14337_b200 as rlu
    from paper_2306_14337_b200.batch import BatchedFactors
    from paper_2306_14337_b200.sharding import SystemRecord, gather_records, scenario_assignment
    from oracle import refbridge as rb  # input fixtures + CPU baseline arm only

    rank, local_rank, world = dist_env()
    n, m, desc = WORKLOADS["C2"]
    if args.scenarios_per_gpu > 0:   # weak line: fixed batch per GPU
        total_scen, scaling = args.scenarios_per_gpu * world, "weak"
    else:                            # BASELINE config 5: the batch is sharded, its size is fixed
        total_scen, scaling = args.scenarios, "strong"
    mine = scenario_assignment(total_scen, world, rank)
    S = len(mine)
    if S == 0:
        raise SystemExit(f"bench.py: {total_scen} scenarios cannot be sharded over {world} ranks")
    S_max = -(-total_scen // world)
    # ---- input fixture (untimed): one generated scenario per y_seed, one symbolic analysis
    seqs = [rb.RefSequence(n, m, y_seed=2 + sc, num_systems=1, keep_blocks=True) for sc in mine]
    sym, ref_sym, analysis = analyze_for_bench(rlu, rb, seqs[0].matrix(0), np)
    ro, ci = seqs[0].pattern()
    N, nnz_a, nnz_f = seqs[0].n, seqs[0].nnz, ref_sym.nnz_factors
    diag_pos = np.nonzero(np.repeat(np.arange(N), np.diff(ro)) == ci)[0]
    delta_p, delta_d = seqs[0].deltas(0)

    stream = torch.cuda.current_stream()
    f = BatchedFactors(sym, S, rlu.FactorOptions(device=local_rank, stream=stream.cuda_stream,
                                                 refine_capacity=args.refine_maxit))
    f.check_pattern(ro, ci)  # pattern_equal guard, once per pattern (src/numeric.cpp:15-17)
    cfg = rlu.RefineConfig(args.refine_maxit, args.refine_tol)
    host_vals = torch.from_numpy(np.stack([q.values(0) for q in seqs])).pin_memory()
    host_rhs = torch.from_numpy(np.stack([q.rhs(0) for q in seqs])).pin_memory()
    host_dy = torch.from_numpy(np.stack([q.d_y(0) for q in seqs])).pin_memory()  # the scenarios' barrier diagonals
    f.kkt_bind(n, seqs[0].h_diag(0), diag_pos)
    dev_vals, dev_rhs = host_vals.cuda(), host_rhs.cuda()
    dev_b = torch.empty_like(dev_rhs)
    host_x = torch.empty((S, N), dtype=torch.float64).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()

    def step_resident():
        f.refactorize(dev_vals)
        x = f.solve_system(dev_rhs)
        if args.no_refine:
            return x, [0] * S
        xr, outs = f.fgmres_refine(dev_rhs, x, cfg)
        return xr, [o.iterations for o in outs]

    def step_e2e():
        f.refactorize(host_vals.numpy())          # H2D of the values inside the call
        dev_b.copy_(host_rhs, non_blocking=True)  # rhs H2D on the handle's stream
        x = f.solve_system(dev_b)
        its = [0] * S
        if not args.no_refine:
            x, outs = f.fgmres_refine(dev_b, x, cfg)
            its = [o.iterations for o in outs]
        host_x.copy_(x, non_blocking=True)
        stream.synchronize()
        return host_x, its

    host_xs = [torch.empty((S, N), dtype=torch.float64).pin_memory() for _ in range(2)]

    dev_xs = [torch.empty((S, N), dtype=torch.float64, device="cuda") for _ in range(2)]

    def timed_pipelined(steps, warmup, resident=False, sampler=None):
        """K batches through the staged submission calls (b200lu_batch_stage_inputs / refactorize_staged /
        solve_refine_staged) under ONE event pair. resident=False is the e2e number: HOST buffers, every step's values
        and right-hand sides copied H2D from pinned memory and its solutions D2H, all inside the timed region; the
        copies of batch k + 1 overlap the factorization and solves of batch k (own copy streams). resident=True is the
        same loop on buffers that already live in HBM (`value`): nothing between the steps waits for the host."""
        vals_in, rhs_in, outs = (dev_vals, dev_rhs, dev_xs) if resident else (host_vals, host_rhs, host_xs)

        def loop(K):
            f.stage_inputs(vals_in, rhs_in)
            for k in range(K):
                if k + 1 < K:
                    f.stage_inputs(vals_in, rhs_in)   # the next batch starts moving now
                f.refactorize_staged()
                f.solve_refine_staged(outs[k % 2], cfg, refine=not args.no_refine)
            f.staged_wait()
        loop(max(2, warmup))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if sampler:
            sampler.window_start()
        e0.record()
        loop(steps)
        e1.record()
        torch.cuda.synchronize()
        if sampler:
            sampler.window_stop()
        if world > 1:
            dist.barrier()
        return e0.elapsed_time(e1)

    def step_e2e_kkt():
        # the scenarios share H and J and differ in D_y: only D_y and the rhs cross the bus,
        # the diagonal of every K is rewritten on the device (b200lu_batch_kkt_update)
        f.kkt_update(host_dy.numpy(), delta_p, delta_d)
        f.factorize_scattered()
        dev_b.copy_(host_rhs, non_blocking=True)
        x = f.solve_system(dev_b)
        its = [0] * S
        if not args.no_refine:
            x, outs = f.fgmres_refine(dev_b, x, cfg)
            its = [o.iterations for o in outs]
        host_x.copy_(x, non_blocking=True)
        stream.synchronize()
        return host_x, its

    def timed(step_fn, steps, warmup, sample_clocks):
        for _ in range(warmup):
            step_fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        sampler = ClockSampler(local_rank) if sample_clocks else None
        if sampler:
            sampler.window_start()
        f.set_timing(True)
        launches0 = f.info["launches"]
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        its = None
        for s in range(steps):
            flush.zero_()  # L2 flush between timed iterations (outside the timed pair)
            ev[s][0].record()
            _, its = step_fn()
            ev[s][1].record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if sampler:
            sampler.window_stop()
        clocks = sampler.stop() if sampler else None
        phases = f.phase_times()
        f.set_timing(False)
        return sum(a.elapsed_time(b) for a, b in ev), its, phases, f.info["launches"] - launches0, clocks

    total_ms, iters, phases, launches, clocks = timed(step_resident, args.steps, args.warmup, True)
    e2e_serial_ms, _, _, _, _ = timed(step_e2e, args.steps, max(1, args.warmup // 2), False)
    e2e_total_ms = timed_pipelined(args.steps, max(1, args.warmup // 2))
    pipelined_same = bool(torch.equal(host_xs[(args.steps - 1) % 2], step_e2e()[0]))  # same bits as the plain calls
    # `value`: the same K steps with every buffer resident in HBM, through the same staged calls (clocks sampled here too)
    sampler_res = ClockSampler(local_rank)
    res_total_ms = timed_pipelined(args.steps, args.warmup, resident=True, sampler=sampler_res)
    clocks_res = sampler_res.stop()
    resident_same = bool(torch.equal(dev_xs[(args.steps - 1) % 2], step_resident()[0]))
    kkt_total_ms, _, _, _, _ = timed(step_e2e_kkt, args.steps, max(1, args.warmup // 2), False)
    x_kkt, _ = step_e2e_kkt()
    kkt_same = bool(torch.equal(x_kkt, step_e2e()[0]))  # diagonal-only submission == full-value submission, bit for bit

    # ---- per-system records (the fields of SystemRecord, include/rlu/report.hpp:14-27) and a parity
    # spot check against the reference (the checker, not the measured path)
    x_direct = f.solve_system(dev_rhs)
    direct = f.relative_residual(x_direct, dev_rhs)
    x_final, its = step_resident()
    final = f.relative_residual(x_final, dev_rhs)
    recs = [SystemRecord(mine[s], float(direct[s]), float(final[s]), int(its[s]), -1) for s in range(S)]
    spot = [0, S - 1]
    ref_relres = max(seqs[s].matrix(0).relative_residual(x_final[s].cpu().numpy(), seqs[s].rhs(0)) for s in spot)
    info = f.info
    f.close()
    allrecs = gather_records(recs, total_scen, device="cuda")

    t = torch.tensor([total_ms, e2e_total_ms, ref_relres, kkt_total_ms, e2e_serial_ms, res_total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms_max, e2e_ms_max, relres_max, kkt_ms_max, e2e_serial_max, res_ms_max = (float(v) for v in t.cpu())

    # the single-system measurements ride on the N = 1 line only (they do not shard)
    single = c4 = c3b = None
    if not args.no_single and world == 1:
        if not args.no_c3_batch:
            c3b = measure_c3_batch(args)
        single = measure_single(args, args.single_workload, min(args.steps * 2, 20), False)
        if not args.no_c4:
            c4 = measure_single(args, "C4", min(args.steps, 10), False)

    nccl_lines = nccl_init_lines() if world > 1 else None
    if rank == 0:
        ms_per_step = res_ms_max / args.steps
        value = total_scen * args.steps / (res_ms_max / 1000.0)
        plain_ms_per_step = total_ms_max / args.steps
        e2e_value = total_scen * args.steps / (e2e_ms_max / 1000.0)
        med_iters = int(statistics.median(iters)) if iters else 0
        ab = batch_algorithmic_bytes(S, N, nnz_a, nnz_f, 0 if args.no_refine else max(med_iters, 0))
        peak, peak_src = measured_peak()
        fac_ms, fac_n = phases["factor"]
        fac_avg_ms = fac_ms / max(fac_n, 1)
        achieved = ab["eliminate"] / (fac_avg_ms * 1e-3) / 1e9 if fac_avg_ms > 0 else 0.0
        traffic, traffic_src = recorded_traffic(f"C5x{S}")
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {
                "workload": f"C5: batch of {total_scen} independent scenario systems sharded over {world} GPU(s) in "
                            f"contiguous blocks ({S_max} per GPU), each "
                            f"{desc} (C2-shaped), one shared pattern / symbolic analysis, y_seed = 2 + scenario; one "
                            f"step = the whole batch through scatter + refactorize + solve_system"
                            f"{'' if args.no_refine else ' + fgmres_refine(tol=%g)' % args.refine_tol} with the "
                            "interleaved scenario-batch kernels; gen_sequence defaults, AMD-only analysis (KLU-style path)",
                "scenarios_total": total_scen, "scenarios_per_gpu": S_max, "n": N, "nnz": nnz_a, "nnz_factors": nnz_f,
                "update_pairs": info["update_pairs"], "levels": info["lower_levels"],
                "unit_scenarios": info["unit_scenarios"], "device_gb": round(info["device_bytes"] / 1e9, 2),
                "l2": "inputs larger than L2: every step streams its own 0.75 GB of values and 4.5 GB of factor values "
                      "(256 scenarios) through the 126 MB L2; the per-phase loop (`plain_calls`) additionally zeroes a "
                      "256 MiB device buffer between steps, outside its per-step event pairs",
                "timing": "`value`, `ms_per_step`: K steps through the staged submission calls with every buffer resident in "
                          "HBM, ONE CUDA event pair around the K steps on the handle's stream, a barrier and a device "
                          "synchronisation on both sides, max over ranks. `e2e`: the same loop with HOST buffers (copies "
                          "inside). `plain_calls`: the same steps through the synchronous calls (refactorize / solve_system "
                          "/ fgmres_refine), per-step event pairs; each of those calls ends with a host read-back (failed "
                          "rows, norms), so 1-3 ms of host-dependent gaps per step are inside it — it is where the "
                          "per-phase times and the roofline's launch duration are measured",
            },
            "clocks": clocks_res,
            "clocks_plain_calls": clocks,
            "plain_calls": {"value": total_scen * args.steps / (total_ms_max / 1000.0), "unit": UNIT, "ms_per_step": plain_ms_per_step,
                            "bitwise_equal_to_staged_resident": resident_same},
            "ms_per_system": ms_per_step / total_scen,
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms_max / args.steps,
                    "h2d_bytes_per_step": 8 * total_scen * (nnz_a + N), "d2h_bytes_per_step": 8 * total_scen * N,
                    "bitwise_equal_to_plain_calls": pipelined_same,
                    "note": "values + rhs of every scenario from pinned host memory H2D and every x D2H inside the timed "
                            "region, every step, through the staged submission calls of the C ABI with HOST pointers "
                            "(b200lu_batch_stage_inputs / refactorize_staged / solve_refine_staged / staged_wait): the copies "
                            "of batch k+1 run on their own streams under the factorization and solves of batch k; one event "
                            "pair around the K-step loop; inputs (> 126 MB per step) cannot stay in L2"},
            "e2e_unpipelined": {"value": total_scen * args.steps / (e2e_serial_max / 1000.0), "unit": UNIT,
                                "ms_per_step": e2e_serial_max / args.steps,
                                "note": "the same bytes through the plain refactorize / solve_system / fgmres_refine calls with "
                                        "host pointers: copies and kernels serialised on one stream"},
            "e2e_kkt_diagonal": {
                "value": total_scen * args.steps / (kkt_ms_max / 1000.0), "unit": UNIT,
                "ms_per_step": kkt_ms_max / args.steps, "h2d_bytes_per_step": 8 * total_scen * (n + N),
                "d2h_bytes_per_step": 8 * total_scen * N, "bitwise_equal_to_full_value_submission": kkt_same,
                "note": "same step submitted through the device-resident KKT value path (b200lu_batch_kkt_update, "
                        "SURVEY 8f-1): the scenarios share H and J, so only each scenario's barrier diagonal D_y "
                        "(n_primal doubles) and rhs are copied H2D and K's diagonal is rewritten on the device"},
            "gpu_launches": launches,
            "analysis": analysis,
            "phases_ms_per_step": {p: v[0] / args.steps for p, v in phases.items()},
            "launches_per_step": {p: v[1] / args.steps for p, v in phases.items()},
            "refine_iters_median": med_iters, "relres_final_max_vs_reference_residual": relres_max,
            "records": None if allrecs is None else {
                "systems": len(allrecs), "worst_relres_direct": max(r.relres_direct for r in allrecs),
                "worst_relres_final": max(r.relres_final for r in allrecs),
                "median_refine_iters": int(statistics.median(r.refine_iters for r in allrecs)),
                "failed": sum(1 for r in allrecs if r.failed_row >= 0)},
            "roofline": {
                "kernel": "bfactor_kernel + the trailing launch (bfactor_block_team_kernel: row blocks, one warp per row, pivot rows staged by cp.async.bulk on an mbarrier; bfactor_tile_kernel up to 32 scenarios per GPU) — K2 numeric refactorization, scenario-batched, timed as one", "bound": "hbm",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak if peak else None,
                "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": ab["eliminate"], "avg_launch_ms": fac_avg_ms,
                "bytes_model": f"SURVEY 8(d) C5 row: eliminate = {S} scenarios x 16*nnz(L+U) value bytes + one copy of "
                               "the int32 indices (4*nnz(L+U) + 8*N), all scenarios in one launch",
                "whole_step": {"algorithmic_bytes": ab["total"],
                               "achieved_gbs": ab["total"] / (ms_per_step * 1e-3) / 1e9,
                               "frac": ab["total"] / (ms_per_step * 1e-3) / 1e9 / peak},
                "second_bound": "L2 atomic unit: every update is a 256-byte red.add.f64 performed by L2 (95.8 GB per "
                                "refactorization at 256 scenarios); ncu lts__d_atomic_input_cycles_active = 77 % of peak "
                                f"(profiles/); critical path: {info['lower_levels']} dependency levels per sweep, shared by "
                                "all scenarios of the batch",
            },
        }
        keys = ("value", "unit", "ms_per_step", "config", "e2e", "phases_ms_per_step", "refine_iters_median",
                "relres_final_max", "roofline", "gpu_launches")
        if single is not None:
            line["single_system"] = {k: single[k] for k in keys}
            line["single_system"]["analysis"] = single.get("analysis")
            line["single_system"]["strict_order"] = single.get("strict_order")
        if c4 is not None:
            line["c4"] = {k: c4[k] for k in keys}
            line["c4"]["analysis"] = c4.get("analysis")
        if c3b is not None:
            line["c3_batch"] = c3b
        if nccl_lines is not None:
            line["nccl"] = nccl_lines
        if not args.no_cpu_baseline:  # rank 0, at every N: the reference on this box's host cores
            threads = rb.max_threads()
            sample = min(S, threads * max(1, args.cpu_reps // 2))
            rate, how, cal, worst = reference_batch_best(rb, ref_sym, seqs[:sample], threads, not args.no_refine,
                                                         args.refine_maxit, args.refine_tol)
            line["cpu_baseline"] = {
                "value": rate, "unit": UNIT, "ms_per_system": 1000.0 / rate, "cores": threads, "kind": "reference",
                "sample": f"of the {S} scenarios of rank 0, through the unmodified reference (oracle/_ref): {how}",
                "calibration": cal, "worst_relres_final": worst}
        print(json.dumps(line))
    if world > 1:
        dist.barrier()  # the other ranks wait for rank 0's CPU baseline before tearing the group down
        dist.destroy_process_group()


def run_reference_batch(args):
    """--impl reference, workload C5: the reference on blocks of independent scenarios, one per thread."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    from oracle import refbridge as rb
    n, m, desc = WORKLOADS["C2"]
    threads = rb.max_threads()
    block = threads  # one bounded sample per step: one scenario per host thread
    nseq = block * max(1, min(args.steps + args.warmup, 4))
    seqs = [rb.RefSequence(n, m, y_seed=2 + sc, num_systems=1) for sc in range(nseq)]
    ref_sym = rb.RefSymbolic(seqs[0].matrix(0), use_scaling=False, use_amd=True)
    rate0, how0, cal, _ = reference_batch_best(rb, ref_sym, seqs[:block], threads, True, args.refine_maxit, args.refine_tol)
    per_thread = cal["one_scenario_per_thread"]["systems_per_s"] >= cal["one_at_a_time_best_exec_mode"]["systems_per_s"]
    num, _policy = calibrate_reference(ref_sym, seqs[0], rb)

    def one_step(lo):
        """One bounded sample: `block` scenarios in the faster of the two modes; returns (seconds, outcomes)."""
        if per_thread:
            return reference_batch_sample(rb, ref_sym, seqs[lo:lo + block], threads, max_iterations=args.refine_maxit,
                                          tolerance=args.refine_tol)
        outs = [num.run_system(q, 0, max_iterations=args.refine_maxit, tolerance=args.refine_tol) for q in seqs[lo:lo + block]]
        return sum(o["scatter_ms"] + o["factor_ms"] + o["trisolve_ms"] + o["refine_ms"] for o in outs) / 1000.0, outs

    for w in range(args.warmup):
        one_step(0)
    tot, worst, phases = 0.0, 0.0, {"scatter_ms": 0.0, "factor_ms": 0.0, "trisolve_ms": 0.0, "refine_ms": 0.0}
    for s in range(args.steps):
        wall, outs = one_step((s * block) % nseq)
        tot += wall
        worst = max(worst, max(o["relres_final"] for o in outs))
        for k in phases:
            phases[k] += sum(o[k] for o in outs) / len(outs)
    value = args.steps * block / tot
    sample = (f"each step = {block} of the C5 scenarios (y_seed = 2 + scenario); mode: " +
              ("one scenario per host thread, ExecMode::sequential inside each, wall clock over the block" if per_thread
               else "one scenario at a time, best ExecMode per phase, sum of the four phase clocks") +
              f"; {threads} host threads")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * tot / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C5: independent scenario systems, each {desc} (C2-shaped), shared pattern; "
                               "scatter+eliminate+solve_system+fgmres_refine per system (cli.cpp:105-135); reference CPU path",
                   "scenarios_per_step": block, "n": seqs[0].n, "nnz": seqs[0].nnz, "nnz_factors": ref_sym.nnz_factors,
                   "analysis": "use_scaling=false,use_amd=true"},
        "ms_per_system": 1000.0 * tot / (args.steps * block),
        "phases_ms_per_system_thread": {k: v / args.steps for k, v in phases.items()},
        "worst_relres_final": worst,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample,
                         "calibration": cal},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }))


def run_b200(args):
    import torch
    import torch.distributed as dist

    rank, local_rank, world = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device — the b200lu path has no CPU fallback")
    # One rank per GPU over NCCL. Test hook for boxes with a single GPU (the multi-rank control flow —
    # scenario assignment, barriers, max-over-ranks, record gather — can then be exercised with
    # `B200LU_BENCH_ONE_DEVICE=1 torchrun --nproc-per-node 2 ...`): every rank uses cuda:0 and gloo.
    one_device = os.environ.get("B200LU_BENCH_ONE_DEVICE") == "1"
    if one_device:
        os.environ["LOCAL_RANK"] = "0"
        local_rank = 0
    torch.cuda.set_device(local_rank)
    if world > 1:
        if one_device:
            dist.init_process_group("gloo")
        else:
            if "NCCL_DEBUG" not in os.environ:  # rank lines for the record, kept out of stdout (one JSON line only)
                log = os.path.join(tempfile.gettempdir(), f"b200lu_nccl_{os.getpid()}.log")
                os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT", NCCL_DEBUG_FILE=log, B200LU_NCCL_LOG=log)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.workload == BATCH_WORKLOAD:
        run_batch(args)
        return
    line = measure_single(args, args.workload, args.steps, not args.no_cpu_baseline)
    if line is not None:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default=BATCH_WORKLOAD, choices=sorted(WORKLOADS) + [BATCH_WORKLOAD])
    ap.add_argument("--scenarios", type=int, default=256, help="C5: scenarios of the batch in TOTAL, sharded over the GPUs")
    ap.add_argument("--scenarios-per-gpu", type=int, default=0, help="C5: fix the per-GPU batch instead (weak scaling)")
    ap.add_argument("--no-c4", action="store_true", help="C5: skip the C4 (n = 1.6 M) single-system block")
    ap.add_argument("--no-c3-batch", action="store_true", help="C5: skip the C3 x 64 scenario-batch block")
    ap.add_argument("--single-workload", default="C3", choices=sorted(WORKLOADS),
                    help="C5: the single-system measurement reported next to the batch")
    ap.add_argument("--no-single", action="store_true", help="C5: skip the single-system measurement")
    ap.add_argument("--no-refine", action="store_true")
    ap.add_argument("--refine-tol", type=float, default=1e-14)
    ap.add_argument("--refine-maxit", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-reps", type=int, default=5)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    # torchrun exports OMP_NUM_THREADS=1 to every rank unless the caller set it; the CPU arm (rank 0 alone: `--impl
    # reference`, and `cpu_baseline`) is to run on all the host threads it can use, so that default is undone before
    # libgomp is loaded (B200LU_BENCH_THREADS overrides the count)
    want = os.environ.get("B200LU_BENCH_THREADS")
    if want or ("TORCHELASTIC_RUN_ID" in os.environ and os.environ.get("OMP_NUM_THREADS") == "1"):
        os.environ["OMP_NUM_THREADS"] = want or str(len(os.sched_getaffinity(0)))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        # self-launch: one rank per GPU on this node (rendezvous on 127.0.0.1: the hostname may not resolve)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    if args.impl == "reference":
        (run_reference_batch if args.workload == BATCH_WORKLOAD else run_reference)(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
