"""World-size-2 CPU (gloo) test of the multi-GPU host logic: scenario sharding, record gather,
max-over-ranks timing. The data path itself has no collective."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2306_14337_b200 import sharding
from oracle import oraclebridge as ob
from tests.fixtures import golden_fixture


def test_scenario_assignment_partitions_exactly():
    for n in (0, 1, 7, 256, 257):
        for world in (1, 2, 3, 8):
            blocks = [sharding.scenario_assignment(n, world, r) for r in range(world)]
            flat = [s for b in blocks for s in b]
            assert flat == list(range(n))
            assert max(len(b) for b in blocks) - min(len(b) for b in blocks) <= 1
    with pytest.raises(ValueError):
        sharding.scenario_assignment(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, num_scenarios, result_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fx = golden_fixture("kkt_small")
        mine = sharding.scenario_assignment(num_scenarios, world, rank)
        records = []
        for s in mine:
            # each "scenario" is one system of the committed sequence, solved by the CPU oracle here
            # (the device path is exercised by the gpu tests; this test is about the host plumbing)
            k = s % len(fx.values)
            lu, failed = fx.oracle.factorize(fx.values[k])
            x, _ = fx.oracle.solve_system(lu, fx.rhs[k])
            A = fx.oracle_csr(k)
            xr, it, conv, hist = ob.refine(A, fx.rhs[k], x, fx.oracle, lu)
            records.append(sharding.SystemRecord(s, A.relative_residual(x, fx.rhs[k]),
                                                 A.relative_residual(xr, fx.rhs[k]), it, failed))
        gathered = sharding.gather_records(records, num_scenarios)
        t = sharding.max_over_ranks([1.0 + rank, 10.0 - rank])
        if rank == 0:
            np.save(result_path, np.array([[r.scenario, r.relres_direct, r.relres_final, r.refine_iters,
                                            r.failed_row] for r in gathered] + [[-1, t[0], t[1], 0, 0]]))
        else:
            assert gathered is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("num_scenarios", [5, 8])
def test_two_rank_shard_and_gather(tmp_path, num_scenarios):
    world, port = 2, _free_port()
    out = str(tmp_path / "records.npy")
    mp.spawn(_worker, args=(world, port, num_scenarios, out), nprocs=world, join=True)
    rows = np.load(out)
    recs, timing = rows[:-1], rows[-1]
    assert list(recs[:, 0].astype(int)) == list(range(num_scenarios))
    fx = golden_fixture("kkt_small")
    for r in recs:
        k = int(r[0]) % len(fx.values)
        assert r[1] == float(fx.golden[f"relres_{k}"])      # identical to the reference's direct residual
        assert int(r[3]) == int(fx.golden[f"iters_{k}"]) and int(r[4]) == -1
        assert r[2] <= 1e-14
    assert timing[1] == 2.0 and timing[2] == 10.0           # max over ranks
