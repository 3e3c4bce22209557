"""Env-sharded multi-GPU plumbing ("Scaling is
near-linear across multiple GPUs").

Environments are independent units: rank r renders the contiguous env
slice [r*E/G, (r+1)*E/G) against its own replica of the scene set.  There
is no exchange on the render path; the only collective is one
all_gather of (frames, digest, elapsed_ns) per rank after the timed loop
(C1), plus barriers around timing (C2).  Works with NCCL (GPU) and gloo
(CPU tests).
"""
from __future__ import annotations

import os


def dist_env() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def env_slice(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [start, end) env slice of `rank` (sizes differ by <= 1)."""
    if world <= 0 or not (0 <= rank < world) or n_total < 0:
        raise ValueError("bad shard spec")
    base, rem = divmod(n_total, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def fold_digests(digests) -> int:
    """Fold per-env 64-bit digests in env order (order-dependent, so a
    rank-sliced run equals a single-GPU run of the same envs)."""
    h = 0xcbf29ce484222325
    for d in digests:
        h ^= int(d) & 0xFFFFFFFFFFFFFFFF
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def gather_stats(frames: int, digest: int, elapsed_ns: int, device=None):
    """C1: all_gather [frames, digest, elapsed_ns] from every rank.

    Returns (total_frames, max_elapsed_ns, digests_in_rank_order).  Single
    process (no process group) returns the local values."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return frames, elapsed_ns, [digest]
    world = dist.get_world_size()
    # digests are full 64-bit; carry them as int64 bit patterns
    d64 = digest - (1 << 64) if digest >= (1 << 63) else digest
    mine = torch.tensor([frames, d64, elapsed_ns], dtype=torch.int64, device=device)
    out = torch.zeros(world * 3, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, mine)
    rows = out.view(world, 3).cpu().tolist()
    total = sum(r[0] for r in rows)
    tmax = max(r[2] for r in rows)
    digs = [r[1] & 0xFFFFFFFFFFFFFFFF for r in rows]
    return total, tmax, digs


def gather_env_digests(dig) -> list:
    """All ranks' per-env digests (int64 tensors of equal length, 64-bit
    patterns) in rank order = global env order; a single process returns its own."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return [int(x) & 0xFFFFFFFFFFFFFFFF for x in dig.cpu().tolist()]
    import torch
    out = torch.zeros(dist.get_world_size() * dig.numel(), dtype=dig.dtype, device=dig.device)
    dist.all_gather_into_tensor(out, dig.contiguous())
    return [int(x) & 0xFFFFFFFFFFFFFFFF for x in out.cpu().tolist()]


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
