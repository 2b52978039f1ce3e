"""Multi-GPU plumbing for the match path: one process per GPU, the index replicated
on every rank, reads sharded with no data-path collective.  The only collectives are the ones a
report needs: an all_reduce(MAX) of elapsed device time and an all_gather of per-shard summaries.
Everything here is backend-agnostic (NCCL on the B200 box, gloo in the CPU tests)."""
from __future__ import annotations

from typing import List, Tuple

import torch
import torch.distributed as dist

GOLDEN = 0x9E3779B1


def shard(rank: int, world: int, reads_per_rank: int) -> Tuple[int, int]:
    """Weak scaling: rank r matches reads [r*Q, (r+1)*Q) of the seeded read stream."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return rank * reads_per_rank, reads_per_rank


def summarize(lohi: torch.Tensor) -> torch.Tensor:
    """[hits, sum of counts, checksum] of a [Q, 2] int32 tensor of uint32 (lo, hi) -> int64[3]."""
    lo = lohi[:, 0].to(torch.int64) & 0xFFFFFFFF
    hi = lohi[:, 1].to(torch.int64) & 0xFFFFFFFF
    packed = lo | (hi << 32)
    return torch.stack([(hi > lo).sum(), (hi - lo).sum(), (packed * GOLDEN).sum()]).to(torch.int64)


def max_over_ranks(value: float, device) -> float:
    """Max of a per-rank scalar (elapsed ms) over the default group; identity when not distributed."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    if dist.get_backend() != "nccl":
        device = "cpu"  # gloo reduces host tensors
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_summaries(summary: torch.Tensor) -> List[List[int]]:
    """All ranks' summaries, in rank order."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [summary.cpu().tolist()]
    if dist.get_backend() != "nccl":
        summary = summary.cpu()
    parts = [torch.empty_like(summary) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, summary)
    return [p.cpu().tolist() for p in parts]


def combine(summaries: List[List[int]]) -> List[int]:
    """Summary of the union of shards (hits and counts add; the checksum is a sum, so it adds too)."""
    mask = (1 << 64) - 1
    out = [0, 0, 0]
    for s in summaries:
        out[0] += s[0]
        out[1] += s[1]
        out[2] = (out[2] + s[2]) & mask
    if out[2] >= 1 << 63:
        out[2] -= 1 << 64
    return out
