"""Multi-GPU plumbing for the match path: one process per GPU, the index replicated
on every rank, reads sharded with no data-path collective.  The only collectives are the ones a
report needs: an all_reduce(MAX) of elapsed device time and an all_gather of per-shard summaries.
Everything here is backend-agnostic (NCCL on the B200 box, gloo in the CPU tests)."""
from __future__ import annotations

import os
from typing import List, Optional, Tuple

import torch
import torch.distributed as dist

GOLDEN = 0x9E3779B1


def shard(rank: int, world: int, reads: int, weak: bool = False) -> Tuple[int, int]:
    """(q_begin, q_count) of rank's reads in the seeded read stream.

    Strong scaling (default: "Q is split into g contiguous equal slices"): the job's
    `reads` are cut into `world` contiguous slices whose sizes differ by at most one.
    Weak scaling (opt-in): every rank matches its own `reads` reads, [rank*reads, (rank+1)*reads)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    if weak:
        return rank * reads, reads
    b = rank * reads // world
    return b, (rank + 1) * reads // world - b


def parse_cpulist(s: str) -> List[int]:
    """'0-3,8,10-11' -> [0, 1, 2, 3, 8, 10, 11] (the sysfs cpulist format)."""
    out: List[int] = []
    for part in s.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def gpu_local_cpus(device_index: int) -> Optional[List[int]]:
    """The host CPUs on the GPU's own NUMA node (sysfs local_cpulist of its PCI function), or None."""
    try:
        p = torch.cuda.get_device_properties(device_index)
        bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        with open(f"/sys/bus/pci/devices/{bdf}/local_cpulist") as f:
            cpus = parse_cpulist(f.read())
        return cpus or None
    except Exception:
        return None


def bind_numa_local(device_index: int) -> dict:
    """Pin this rank's process to the CPUs local to its GPU, so the pinned host buffers it allocates and
    first-touches afterwards (reads, results, the e2e staging) are placed on the GPU's NUMA node.
    Returns what was done, for the bench line."""
    cpus = gpu_local_cpus(device_index)
    if not cpus:
        return {"bound": False, "reason": "no local_cpulist for the GPU"}
    allowed = os.sched_getaffinity(0)
    use = sorted(set(cpus) & allowed)
    if not use:
        return {"bound": False, "reason": "GPU-local CPUs outside this process's affinity"}
    os.sched_setaffinity(0, use)
    return {"bound": True, "cpus": len(use), "first": use[0], "last": use[-1]}


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


def all_reduce_sum(value: int, device) -> int:
    """Sum of a per-rank integer (reads matched) over the default group; identity when not distributed."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return int(value)
    if dist.get_backend() != "nccl":
        device = "cpu"
    t = torch.tensor([value], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())


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


def partitioned_match(idx, words, lens=None, fixed_len=None, out=None):
    """match this rank's batch against a partitioned index (idx = this rank's part,
    csrc/sa_part.cu).

    route (order by route key, rows in that order, per-part offsets; reads shorter than the route key last:
    sa_match_route) -> pack the send buffer (block g = the rows routed to part g + every short row:
    sa_part_pack) -> all-to-all of the counts and of the rows -> match the received rows on this rank's
    slice -> all-to-all of the intervals back -> sa_part_collect (a routed read takes its part's interval,
    a short read the sum of the parts' clamped answers) into the batch's own order.  The all-to-alls run
    over the default process group (NCCL on GPUs; gloo stages through host memory)."""
    Q, stride = words.shape
    dev = words.device
    world = dist.get_world_size() if dist.is_initialized() else 1
    order, ow, ol, offs = idx.route(words, lens, fixed_len=fixed_len)
    o = offs.cpu().tolist()
    nparts = len(o) - 1
    if world != nparts:
        raise ValueError(f"{nparts} partitions but world size {world}")
    n_short = Q - o[nparts]
    send = [o[g + 1] - o[g] + n_short for g in range(nparts)]
    sw, sl = idx.part_pack(ow, ol, offs, sum(send))
    recv, rows, rlens = exchange_rows(send, sw, sl, dev)
    res = idx.match(rows, rlens, fixed_len=fixed_len) if rows.shape[0] else \
        torch.empty((0, 2), dtype=torch.int32, device=dev)
    back = exchange_back(res, recv, send, dev)
    return idx.part_collect(back, offs, order, Q, out=out)


def _host_staged():
    return dist.is_initialized() and dist.get_world_size() > 1 and dist.get_backend() != "nccl"


def exchange_rows(send, sw, sl, dev):
    """All-to-all of the send blocks: (received counts per source, received rows, received lengths or None).
    Rows from source s arrive in rank order: [block for me from rank 0, from rank 1, ...]."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    if world == 1:
        return list(send), sw, sl
    host = _host_staged()
    stage = (lambda t: t.cpu()) if host else (lambda t: t)
    cdev = "cpu" if host else dev
    st = torch.tensor(send, dtype=torch.int64, device=cdev)
    rt = torch.empty_like(st)
    dist.all_to_all_single(rt, st)
    recv = rt.cpu().tolist()
    rows = torch.empty((sum(recv),) + tuple(sw.shape[1:]), dtype=sw.dtype, device=cdev)
    dist.all_to_all_single(rows, stage(sw), output_split_sizes=recv, input_split_sizes=list(send))
    rlens = None
    if sl is not None:
        rlens = torch.empty(sum(recv), dtype=sl.dtype, device=cdev)
        dist.all_to_all_single(rlens, stage(sl), output_split_sizes=recv, input_split_sizes=list(send))
        rlens = rlens.to(dev)
    return recv, rows.to(dev), rlens


def exchange_back(res, recv, send, dev):
    """All-to-all of the answers back to the ranks that sent the rows (the inverse split sizes)."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    if world == 1:
        return res
    host = _host_staged()
    back = torch.empty((sum(send),) + tuple(res.shape[1:]), dtype=res.dtype, device="cpu" if host else dev)
    dist.all_to_all_single(back, res.cpu() if host else res, output_split_sizes=list(send), input_split_sizes=recv)
    return back.to(dev)
