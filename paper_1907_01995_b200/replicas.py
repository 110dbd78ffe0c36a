"""Multi-GPU use of the sweep: independent replicas, no data-path collective.

The Gauss-Seidel chain over blocks is sequential (SPEC.md:184,
elastic_net.py:199-224), so a single solve does not shard.  Multi-GPU work
is a set of independent solves — the paper's (alpha, lambda) grid
(PAPER.md:311-312), seeds, or the SVM (C, sigma) grid (svm.py:349-404) —
spread one process per GPU.  The only communication is bookkeeping: the
max-over-ranks timing and gathering each rank's results.
"""

from __future__ import annotations

from typing import Sequence


def shard(cells: Sequence, rank: int, world: int) -> list:
    """Round-robin share of `cells` for `rank` (deterministic, covers every cell once)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    return [c for i, c in enumerate(cells) if i % world == rank]


def max_over_ranks(value: float, group=None) -> float:
    """Max of a scalar over all ranks (device timings are reported as the max)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_results(local: list, group=None) -> list:
    """All ranks' result lists concatenated in rank order (object all-gather)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return list(local)
    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, list(local), group=group)
    return [x for part in out for x in part]
