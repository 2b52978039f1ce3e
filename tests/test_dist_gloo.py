"""The N>1 host path on CPU: world_size-2 gloo processes shard the read stream, each computes its
intervals (here with the oracle -- there is no GPU), and the collectives (max of elapsed, gather of
summaries) reproduce the single-process result exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_1303_3692_b200 import shard

N_REF, Q_RANK = 20_000, 500


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _intervals(q_begin, q_count):
    ref = synth.reference(synth.REF_REPEAT, N_REF, 9)
    S = oracle.encode(ref)
    words, lens = synth.reads(ref, q_count, 20, 60, 0.1, 0.0, 10, q_begin=q_begin)
    lohi = oracle.search_batch(S, oracle.sa_naive(S), words, lens).astype(np.uint32)
    return torch.from_numpy(lohi.view(np.int32))


def _worker(rank, world, port, outq):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q0, qn = shard.shard(rank, world, world * Q_RANK + 1)  # strong: contiguous slices of one job
    summ = shard.summarize(_intervals(q0, qn))
    gathered = shard.gather_summaries(summ)
    elapsed = shard.max_over_ranks(10.0 * (rank + 1), "cpu")
    outq.put((rank, gathered, elapsed))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    # every rank sees the same gathered summaries and the max elapsed
    assert res[0][1] == res[1][1]
    assert res[0][2] == res[1][2] == 20.0
    # shards are the contiguous slices of one read stream: combined == single-process summary
    single = shard.summarize(_intervals(0, world * Q_RANK + 1)).tolist()
    assert shard.combine(res[0][1]) == single


def test_shard_ranges():
    # strong scaling (default): contiguous slices of the job's reads that tile [0, Q)
    assert shard.shard(0, 4, 100) == (0, 25)
    assert shard.shard(3, 4, 100) == (75, 25)
    for Q in (0, 1, 7, 100_000_001):
        for world in (1, 2, 3, 8):
            sl = [shard.shard(r, world, Q) for r in range(world)]
            assert sl[0][0] == 0 and sum(c for _, c in sl) == Q
            assert all(a + c == b for (a, c), (b, _) in zip(sl, sl[1:]))
            assert max(c for _, c in sl) - min(c for _, c in sl) <= 1
    # weak scaling (opt-in): every rank its own Q reads
    assert shard.shard(3, 4, 100, weak=True) == (300, 100)
    with pytest.raises(ValueError):
        shard.shard(4, 4, 100)


def test_cpulist_parse():
    assert shard.parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert shard.parse_cpulist("5") == [5]
