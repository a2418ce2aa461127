"""Multi-GPU plumbing for the SIDWT path: one process per GPU, rows sharded across
ranks, no collective on the data path.

The path shards over independent range lines: each rank
runs the whole hot path on its own rows; the only collectives are for timing
(max over ranks) and, optionally, gathering the per-row peak tables at rank 0.
torch.distributed is plumbing only (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations


def weak_rows(rank: int, rows_per_rank: int) -> tuple[int, int]:
    """Weak scaling: rank k owns global rows [k R, (k+1) R)."""
    return rank * rows_per_rank, rows_per_rank


def strong_rows(rank: int, world: int, total_rows: int) -> tuple[int, int]:
    """Strong scaling: a contiguous block of `total_rows` per rank (sizes differ by <= 1)."""
    base, rem = divmod(total_rows, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. the timed region in ms) over all ranks."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local, total_rows: int, device=None):
    """All-gather per-row results (first dim = rows, blocks in rank order) of a strong-scaling
    partition into a [total_rows, ...] tensor on every rank."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    world = dist.get_world_size()
    sizes = [strong_rows(r, world, total_rows)[1] for r in range(world)]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([b[:n] for b, n in zip(bufs, sizes)], dim=0)


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def timed_steps(step, steps: int, sync, timer, device=None) -> float:
    """The contract's timed region, shared by bench.py (NCCL, CUDA events) and the gloo test
    (CPU clock): barrier + sync, `steps` calls of `step`, sync + barrier, then the per-step
    time as the MAX over ranks.  `timer()` returns a (start, stop, elapsed_ms) triple of
    callables; `sync()` waits for the device."""
    start, stop, elapsed_ms = timer()
    barrier()
    sync()
    start()
    for _ in range(steps):
        step()
    stop()
    sync()
    barrier()
    return max_over_ranks(elapsed_ms() / steps, device=device)


def gather_weak(local, device=None):
    """All-gather equal-size per-rank row blocks of a weak-scaling run (rank order) into one
    [world * rows, ...] tensor on every rank (e.g. the per-row peak tables)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    bufs = [torch.empty_like(local) for _ in range(dist.get_world_size())]
    dist.all_gather(bufs, local.contiguous())
    return torch.cat(bufs, dim=0)
