"""N>1 path on CPU: world_size-2 gloo runs of the batch partitioning and the
per-step result gather (dist.py), checked against the single-rank result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_07644_b200 import dist as D
from paper_2604_07644_b200 import scenarios


def test_shard_covers_exactly_once():
    for total in (0, 1, 5, 1024, 1031):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                first, cnt = D.shard(total, r, world)
                seen.extend(range(first, first + cnt))
            assert seen == list(range(total))
    with pytest.raises(ValueError):
        D.shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_step(states, nu):
    """Stand-in for the device step: deterministic per-instance results."""
    B = states.shape[0]
    u0 = torch.as_tensor(np.tanh(states[:, :nu]))
    its = torch.as_tensor((np.abs(states).sum(1) * 1e3).astype(np.int32) % 97 + 1)
    conv = torch.ones(B, dtype=torch.int32)
    rho = torch.zeros(B, dtype=torch.int32)
    cost = torch.as_tensor((states ** 2).sum(1))
    return D.pack_results(u0, its, conv, rho, cost)


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = scenarios.rti_workload("q61")
        counts = [D.shard(total, r, world)[1] for r in range(world)]
        first, cnt = D.shard(total, rank, world)
        local = _fake_step(wl.scenario_states(first, cnt), wl.model.nu)
        full = D.gather_results(local, world, counts=counts)
        ms = D.max_over_ranks(10.0 + rank, world)
        if rank == 0:
            q.put((full.numpy(), ms))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [8, 7])
def test_gloo_world2_gather_matches_single_rank(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, ms = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl = scenarios.rti_workload("q61")
    ref = _fake_step(wl.scenario_states(0, total), wl.model.nu).numpy()
    assert full.shape == ref.shape
    np.testing.assert_array_equal(full, ref)
    assert ms == 11.0
