"""Scenario sharding across GPUs.

A single factorization is one dependency DAG and stays on one GPU. Independent scenario /
contingency systems share one sparsity pattern — hence one symbolic analysis — and differ only in
their values, so a batch shards by scenario with NO data-path collective: every rank owns a handle,
its scenarios' values and right-hand sides. The only communication is the gather of the per-system
records (the fields of the reference's SystemRecord, include/rlu/report.hpp:14-27) to rank 0.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

RECORD_FIELDS = ("scenario", "relres_direct", "relres_final", "refine_iters", "failed_row")


def scenario_assignment(num_scenarios: int, world_size: int, rank: int) -> range:
    """Contiguous block of scenario ids owned by `rank`; sizes differ by at most one."""
    if not (0 <= rank < world_size):
        raise ValueError(f"rank {rank} outside world of {world_size}")
    base, extra = divmod(num_scenarios, world_size)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


@dataclass
class SystemRecord:
    scenario: int
    relres_direct: float
    relres_final: float
    refine_iters: int
    failed_row: int = -1

    def as_row(self) -> list:
        return [float(self.scenario), self.relres_direct, self.relres_final, float(self.refine_iters),
                float(self.failed_row)]


def gather_records(records: list, num_scenarios: int, group=None, device="cpu"):
    """All ranks call this; rank 0 gets the records of every scenario ordered by scenario id, the
    others get None. One all_gather of a (max_per_rank, 5) float64 block per rank: at most
    num_scenarios * 5 doubles in total (~10 KB for 256 scenarios). No factor or vector data moves."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return sorted(records, key=lambda r: r.scenario)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    cap = -(-num_scenarios // world)
    block = torch.full((cap, len(RECORD_FIELDS)), float("nan"), dtype=torch.float64, device=device)
    for i, r in enumerate(records):
        block[i] = torch.tensor(r.as_row(), dtype=torch.float64)
    out = [torch.empty_like(block) for _ in range(world)]
    dist.all_gather(out, block, group=group)
    if rank != 0:
        return None
    rows = torch.cat(out).cpu().numpy()
    rows = rows[~np.isnan(rows[:, 0])]
    rows = rows[np.argsort(rows[:, 0])]
    return [SystemRecord(int(r[0]), float(r[1]), float(r[2]), int(r[3]), int(r[4])) for r in rows]


def max_over_ranks(values, group=None, device="cpu"):
    """Element-wise MAX of a short list of floats over all ranks (timings are reported as the
    maximum over ranks, never by wall clock of one rank)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return [float(v) for v in t.cpu()]
