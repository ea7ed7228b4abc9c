"""Multi-GPU: batches of independent MPC instances, and one long-horizon SLS.

* Batches: a batch of scenarios is split into contiguous per-rank
  blocks with no communication inside the step.  After each batched step the
  ranks exchange one compact result record per instance (``RESULT_FIELDS``)
  with a single ``all_gather_into_tensor`` — NCCL over NVLink on the GPU box,
  gloo in the CPU tests.  A single QP solve stays on one GPU (north star).
* One SLS across ranks: the disturbance columns of one
  synthesis are independent, so ``column_shards`` gives each rank a contiguous
  column range balanced by cell count, ``sls.synthesize_tighten_columns``
  synthesizes only that shard (``gsls_sls_set_columns``: storage and work divide
  by the rank count), and ``allreduce_tightening`` sums the partial h, hf.

The reference has no multi-process path at all (scan.py:97-128 is thread-level
only); this module is the build's addition on top of the drop-in entry points.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

# one float64 row per instance: u0 (nu) followed by these scalars
RESULT_FIELDS = ("admm_iterations", "converged", "rho_changes", "cost")


def env():
    """(rank, local_rank, world) from the torchrun environment (1 process = 1 GPU)."""
    import os
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block (first, count) of ``total`` instances owned by ``rank``;
    the first ``total % world`` ranks take one extra instance."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if total < 0:
        raise ValueError("total must be >= 0")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def pack_results(u0: torch.Tensor, iterations: torch.Tensor, converged: torch.Tensor, rho_changes: torch.Tensor,
                 cost: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """(B, nu + 4) float64 record of one batched step, on the engine's device."""
    B, nu = u0.shape
    if out is None:
        out = torch.empty(B, nu + len(RESULT_FIELDS), dtype=torch.float64, device=u0.device)
    out[:, :nu] = u0
    out[:, nu] = iterations
    out[:, nu + 1] = converged
    out[:, nu + 2] = rho_changes
    out[:, nu + 3] = cost
    return out


def pack_engine(engine, out: torch.Tensor | None = None) -> torch.Tensor:
    """The engine's record through the C ABI (gsls_rti_pack_results, one kernel)."""
    import ctypes
    from . import _native as nat
    from .device import stream_ptr
    if out is None:
        out = torch.empty(engine.B, engine.u0.shape[1] + len(RESULT_FIELDS), dtype=torch.float64,
                          device=engine.u0.device)
    ss = engine.stats.cstruct()
    nat.check(engine.ctx.lib.gsls_rti_pack_results(engine.ctx.handle, engine.u0.data_ptr(), ctypes.byref(ss),
                                                   engine.cost.data_ptr(), out.data_ptr(), stream_ptr()),
              "pack results")
    return out


def gather_results(local: torch.Tensor, world: int, out: torch.Tensor | None = None,
                   counts: list[int] | None = None) -> torch.Tensor:
    """All ranks receive every rank's records in global instance order.

    Equal blocks go through one ``all_gather_into_tensor``; ragged blocks
    (``counts`` from ``shard``) are padded to the largest block and trimmed."""
    if world == 1:
        return local if out is None else out.copy_(local)
    rows, width = local.shape
    if counts is None or len(set(counts)) == 1:
        if out is None:
            out = torch.empty(world * rows, width, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous())
        return out
    mx = max(counts)
    pad = torch.zeros(mx, width, dtype=local.dtype, device=local.device)
    pad[:rows] = local
    buf = torch.empty(world * mx, width, dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(buf, pad)
    parts = [buf[r * mx:r * mx + c] for r, c in enumerate(counts)]
    full = torch.cat(parts, 0)
    return full if out is None else out.copy_(full)


def column_shards(N: int, world: int) -> list[tuple[int, int]]:
    """Contiguous disturbance-column ranges [j0, j1), one per rank, balanced by SLS
    cell count (column j holds N - j cells, so early columns are heavier)."""
    if world < 1:
        raise ValueError(f"bad world {world}")
    if N < world:
        raise ValueError(f"{N} columns cannot be split over {world} ranks")
    total = N * (N + 1) // 2
    prefix = [j * N - j * (j - 1) // 2 for j in range(N + 1)]   # cells in columns [0, j)
    bounds = [0]
    for r in range(1, world):
        lo, hi = bounds[-1] + 1, N - (world - r)                 # at least one column per rank
        target = total * r / world
        bounds.append(min(range(lo, hi + 1), key=lambda j: abs(prefix[j] - target)))
    bounds.append(N)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def allreduce_tightening(h: torch.Tensor, hf: torch.Tensor, world: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Sum the per-shard partial tightenings over ranks (one all-reduce of N*nc + nf
    floats; NCCL on the GPU box, gloo in the CPU tests)."""
    if world == 1:
        return h, hf
    flat = torch.cat([h.reshape(-1), hf.reshape(-1)])
    dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    return flat[: h.numel()].reshape(h.shape), flat[h.numel():].reshape(hf.shape)


def sls_tighten_sharded(A, B, E, costs, C, D, CN, rank: int, world: int, executor=None):
    """SLS synthesis + tightening with the disturbance columns sharded over ranks
    (SURVEY §8f row 3): each rank synthesizes its columns only (memory and work
    divided by ~world) and the partial h, hf are all-reduced.  Returns
    (sls.Tightening on every rank, this rank's (j0, j1), its shard-local phix, phiu)."""
    from . import sls
    N = np.asarray(A).shape[0]
    cols = column_shards(N, world)[rank]
    h, hf, phix, phiu = sls.synthesize_tighten_columns(A, B, E, costs, C, D, CN, cols, executor)
    h, hf = allreduce_tightening(h, hf, world)
    return sls.Tightening(h=h.cpu().numpy(), hf=hf.cpu().numpy()), cols, phix, phiu


def max_over_ranks(ms: float, world: int, device=None) -> float:
    """Timing convention: the slowest rank's device time."""
    if world == 1:
        return float(ms)
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t)
