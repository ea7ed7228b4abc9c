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


# --- SLS disturbance columns sharded over ranks -----------------------

def test_column_shards_cover_and_balance():
    for N in (1, 2, 7, 25, 64, 2047):
        for world in (1, 2, 3, 8):
            if world > N:
                with pytest.raises(ValueError):
                    D.column_shards(N, world)
                continue
            sh = D.column_shards(N, world)
            assert sh[0][0] == 0 and sh[-1][1] == N and len(sh) == world
            assert all(a < b for a, b in sh) and all(sh[r][1] == sh[r + 1][0] for r in range(world - 1))
            cells = [sum(N - j for j in range(a, b)) for a, b in sh]
            # within one (largest) column of the even split
            assert max(cells) - N * (N + 1) / 2 / world <= N


def _sls_problem(seed=0, N=9, nx=3, nu=2, nc=2):
    from oracle import sls as osls
    rng = np.random.default_rng(seed)
    A = np.eye(nx) + 0.1 * rng.standard_normal((N, nx, nx))
    B = rng.standard_normal((N, nx, nu))
    E = 0.05 * rng.standard_normal((N, nx, nx))
    C = rng.standard_normal((N, nc, nx))
    Dm = rng.standard_normal((N, nc, nu))
    CN = rng.standard_normal((1, nx))
    costs = osls.assemble_costs(None, C, Dm, CN, osls.Weights.identity(nx, nu))
    return A, B, E, C, Dm, CN, osls.synthesize(A, B, E, costs)


def _partial_tighten(resp, C, Dm, CN, j0, j1):
    """The shard's partial sums: columns j in [j0, j1) only (sls.py:329-341 restricted)."""
    from oracle import sls as osls
    N, nc, nf = resp.N, C.shape[1], CN.shape[0]
    h, hf = np.zeros((N, nc)), np.zeros(nf)
    for k in range(1, N):
        for j in range(j0, min(k, j1)):
            h[k] += osls.row_norms(C[k] @ resp.phi_x(k, j) + Dm[k] @ resp.phi_u(k, j))
    for j in range(j0, j1):
        hf += osls.row_norms(CN @ resp.phi_x(N, j))
    return h, hf


def _sls_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, B, E, C, Dm, CN, resp = _sls_problem()
        j0, j1 = D.column_shards(resp.N, world)[rank]
        h, hf = _partial_tighten(resp, C, Dm, CN, j0, j1)
        H, HF = D.allreduce_tightening(torch.as_tensor(h), torch.as_tensor(hf), world)
        if rank == 0:
            q.put((H.numpy(), HF.numpy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_tightening_matches_unsharded():
    from oracle import sls as osls
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sls_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    H, HF = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    A, B, E, C, Dm, CN, resp = _sls_problem()
    ref = osls.tighten(resp, C, Dm, CN)
    np.testing.assert_allclose(H, ref.h, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(HF, ref.hf, rtol=1e-12, atol=1e-12)
