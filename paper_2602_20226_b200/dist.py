"""Multi-GPU plumbing for the batched zip-up.

configs[4] shards independent zip-ups across GPUs: rank g owns members
[g*M, (g+1)*M) and regenerates them from their seeds (no input scatter).  The only
cross-GPU exchange is one all-reduce (sum) of the 4-element fp64 summary
[sum delta^2, sum ||y||^2, sum ranks, member count] per batch, issued on the compute
stream through torch.distributed (NCCL over NVLink on the B200 box; gloo in the CPU
tests).  Timings are reduced with MAX over ranks.  There is no data-path collective.
"""
from __future__ import annotations

import math
from typing import Dict, List, Tuple


def member_range(rank: int, world: int, members_per_rank: int) -> Tuple[int, int]:
    """Weak scaling: every rank owns the same number of members, disjoint and contiguous."""
    if not (0 <= rank < world) or members_per_rank < 1:
        raise ValueError("bad rank/world/members")
    return rank * members_per_rank, (rank + 1) * members_per_rank


def strong_range(rank: int, world: int, total: int) -> Tuple[int, int]:
    """Strong scaling split of `total` members (balanced to within one member)."""
    base, rem = divmod(total, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def allreduce_summary(summary, dist=None):
    """In-place SUM all-reduce of the (4,) float64 summary tensor (the a8 collective)."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(summary)
    return summary


def max_over_ranks(value: float, device, dist=None) -> float:
    """Device-timed quantities are reported as the MAX over ranks."""
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def summary_dict(summary) -> Dict[str, float]:
    s = [float(v) for v in summary]
    return {"sum_delta2": s[0], "sum_norm2": s[1], "sum_ranks": s[2], "members": s[3],
            "sqrt_sum_delta2_over_sum_norm2": math.sqrt(s[0] / s[1]) if s[1] > 0 else float("nan")}


def local_summary(delta2_rows: List[List[float]], norm2: List[float], ranks_rows: List[List[int]]):
    """Host reference of qtt_zipup_summary (fixed order) -- used by the CPU tests."""
    s0 = sum(sum(r) for r in delta2_rows)
    s1 = sum(norm2)
    s2 = sum(sum(r[1:-1]) for r in ranks_rows)
    return [s0, s1, float(s2), float(len(norm2))]
