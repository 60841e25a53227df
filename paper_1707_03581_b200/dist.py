"""Multi-GPU plumbing for the batched mode.

One process per GPU.  Scenarios are independent (each has its own motion law and friction,
BASELINE.json config 4), so the batched mode shards by scenario with no data-path
collective: rank r advances the contiguous block `shard_range(S, r, world)` of scenarios on
its own GPU.  The only collectives are outside the data path: the max-over-ranks device time
of a timed region and, if a caller wants every scenario's field on one rank, a final gather.
A single-run implicit-Euler step does not shard in this build ("replicas only").

Everything here is host logic on `torch.distributed` (NCCL on the GPU box, gloo in the CPU
tests); no method arithmetic.
"""
from __future__ import annotations

import dataclasses
import os
from typing import List, Tuple

import numpy as np


def env_world() -> Tuple[int, int, int]:
    """(world, rank, local_rank) from the torchrun environment (1, 0, 0 without torchrun)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous block [lo, hi) of n units owned by `rank`: sizes differ by at most one,
    the first n % world ranks take the larger blocks, blocks are in rank order."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError(f"bad shard request n={n} rank={rank} world={world}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_config(cfg, rank: int, world: int):
    """The config restricted to this rank's scenario block (meshes and BCs shared)."""
    lo, hi = shard_range(cfg.n_scen, rank, world)
    if hi <= lo:
        raise ValueError(f"rank {rank} of {world} owns no scenario (S = {cfg.n_scen})")
    return dataclasses.replace(cfg, scenarios=list(cfg.scenarios[lo:hi]),
                               name=f"{cfg.name}[{lo}:{hi}]")


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. a device-timed region in ms) over all ranks."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_scenarios(local: np.ndarray, n_scen: int, device=None) -> np.ndarray:
    """Final gather of per-scenario fields: `local` is [S_local, N] for this rank's block;
    returns the full [n_scen, N] array (in scenario order) on every rank."""
    import torch
    import torch.distributed as dist
    local = np.ascontiguousarray(local, dtype=np.float64)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    blocks: List[Tuple[int, int]] = [shard_range(n_scen, r, world) for r in range(world)]
    smax = max(hi - lo for lo, hi in blocks)
    n = local.shape[1]
    buf = torch.zeros((smax, n), dtype=torch.float64, device=device)
    buf[:local.shape[0]] = torch.from_numpy(local).to(buf.device)
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf)
    return np.concatenate([out[r][:hi - lo].cpu().numpy() for r, (lo, hi) in enumerate(blocks)], axis=0)
