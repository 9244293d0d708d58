"""Multi-GPU sharding of independent IK problems.

The problems are fully independent, so the batch is split into contiguous
index ranges, one per rank (one process per GPU); each rank solves its range
with no collective in the solve.  Results can be gathered with one
``all_gather`` (NCCL over NVLink on GPUs; gloo in the CPU tests) -- a few tens
of bytes per target -- or simply kept on the rank / copied to the host.
Results never depend on the rank count: every kernel is per-target
deterministic and targets are keyed by their global index.
"""

from __future__ import annotations


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [start, end) of rank `rank`; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_rows(local, total: int, group=None):
    """All-gather per-rank row blocks (torch tensors, same trailing shape) into the
    full [total, ...] array in global index order, on ``local``'s device.

    NCCL gathers device tensors directly (NVLink / NVSwitch); a gloo group only
    moves host tensors, so device blocks are staged through host memory there
    (several ranks sharing one GPU, or a CPU-only test)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [shard_range(total, world, r) for r in range(world)]
    width = max(e - s for s, e in sizes)
    via_host = dist.get_backend(group) == "gloo" and local.device.type != "cpu"
    dev = torch.device("cpu") if via_host else local.device
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=dev)
    pad[: local.shape[0]] = local.to(dev)
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    full = torch.cat([p[: e - s] for p, (s, e) in zip(parts, sizes)], dim=0)
    return full.to(local.device) if via_host else full


def solve_sharded(solver, targets_for, total: int, group=None, gather: bool = True):
    """Solve `total` targets split over the ranks of `group`.

    targets_for(start, end) -> device (end-start, 7) tensor of this rank's
    targets.  Returns this rank's BeamBatch (gather=False) or the full
    gathered fields on every rank (gather=True).
    """
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    s, e = shard_range(total, world, rank)
    out = solver.solve_device(targets_for(s, e))
    if not gather or world == 1:
        return out
    fields = {}
    for name in ("q", "cost", "history", "pos_error", "rot_error", "success"):
        fields[name] = gather_rows(getattr(out, name), total, group)
    return fields
