"""Host-side multi-GPU plumbing for the QMCUR path (one process per GPU,
torch.distributed over NCCL; gloo in the CPU tests).

SURVEY.md 8(e):
  * cfg1-cfg3 (one matrix <= 4000^2, ~10 ms FP64-bound on one GPU): replicas —
    every rank runs its own approximations, no data-path collective (weak scaling).
  * cfg4 (64 independent matrices): split by matrix, contiguous blocks, no
    collective; per-matrix results are gathered at the end (strong scaling).
Timing is always the maximum over ranks of device-measured time.
"""
from __future__ import annotations


def shard_range(total: int, world: int, rank: int) -> range:
    """Contiguous block of `total` units owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(int(total), world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def max_over_ranks(value: float, device=None) -> float:
    """Maximum of a per-rank scalar (elapsed ms) across the process group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_results(local: dict[int, float], total: int, device=None) -> list[float]:
    """Assemble per-unit results {unit: value} from every rank into a list of
    `total` values ordered by unit (each unit owned by exactly one rank)."""
    import torch
    import torch.distributed as dist

    out = torch.full((total,), float("nan"), dtype=torch.float64, device=device)
    for k, v in local.items():
        out[k] = v
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        # fill-by-owner: NaN elsewhere, so a MAX reduce keeps the owner's value
        mask = torch.isnan(out)
        out[mask] = -float("inf")
        dist.all_reduce(out, op=dist.ReduceOp.MAX)
    return [float(v) for v in out.cpu()]


def gather_rows(local: dict, total: int, width: int, device=None):
    """Assemble per-unit fixed-width rows {unit: sequence of `width` numbers} from every rank
    into a (total, width) float64 numpy array ordered by unit (index sets, statistics)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    out = torch.full((total, width), -float("inf"), dtype=torch.float64, device=device)
    for k, v in local.items():
        out[k] = torch.as_tensor(np.asarray(v, dtype=np.float64), device=out.device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(out, op=dist.ReduceOp.MAX)  # each row has exactly one owner
    return out.cpu().numpy()


def run_batch_split(total: int, approx_one, width: int, device=None):
    """cfg4's by-matrix split: this rank approximates its contiguous block of the
    `total` matrices with approx_one(b) -> row of `width` numbers (relative error, indices ...),
    and every rank receives the (total, width) table of all results.  No collective runs between
    the approximations; one all-reduce assembles the table at the end."""
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    local = {b: approx_one(b) for b in shard_range(total, world, rank)}
    return gather_rows(local, total, width, device=device)
