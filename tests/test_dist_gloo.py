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


# ---- the partitioned index's exchange over a real 2-process group ---------------
class FakePart:
    """One part of a partitioned index computed on the CPU with the oracle, with the calls that
    shard.partitioned_match makes (include/sa.h's contract for sa_match_route / sa_part_pack /
    sa_match_batch on a part / sa_part_collect): the suffixes whose first rb bases (the route key, a short
    suffix placed as the k-mer table places it) lie in [keys[g], keys[g+1]) form part g, whose ranks
    [ranks[g], ranks[g+1]) tile [0, n); a part answers a read clamped to its ranks."""

    def __init__(self, S, sa_ref, part, nparts, rb):
        n = len(S)
        T = oracle.kmer_table(S, rb).astype(np.int64)  # T_r[K] = #{i : trunc_rb(S_i) < K}
        keys = [0] * (nparts + 1)
        keys[nparts] = 4 ** rb
        for g in range(1, nparts):
            keys[g] = keys[g - 1] + int(np.searchsorted(T[keys[g - 1]:], g * n // nparts, side="left"))
        self.S, self.sa, self.rb, self.P = S, sa_ref, rb, nparts
        self.keys = keys
        # (part 0 starts at rank 0: it also holds the all-'a' suffixes shorter than rb, e_rb = -1)
        self.ranks = [0] + [int(T[keys[g]]) for g in range(1, nparts)] + [n]
        self.r0, self.r1 = self.ranks[part], self.ranks[part + 1]

    def route(self, words, lens=None, fixed_len=None):
        w = words.numpy().view(np.uint64)
        m = lens.numpy().astype(np.int64) if lens is not None else np.full(w.shape[0], fixed_len, np.int64)
        rb = self.rb
        key = (w[:, 0] >> np.uint64(64 - 2 * rb)).astype(np.int64)
        short = m < rb
        key[short] = 4 ** rb
        order = np.argsort(key, kind="stable")
        offs = np.searchsorted(key[order], self.keys, side="left").astype(np.int64)
        ow = torch.from_numpy(w[order].view(np.int64).copy())
        ol = None if lens is None else torch.from_numpy(lens.numpy()[order].copy())
        return torch.from_numpy(order.astype(np.int32)), ow, ol, torch.from_numpy(offs)

    def part_pack(self, ow, ol, offs, send_rows):
        o = offs.tolist()
        idx = np.concatenate([np.r_[o[g]:o[g + 1], o[self.P]:ow.shape[0]] for g in range(self.P)]).astype(np.int64)
        assert idx.size == send_rows
        return ow[idx], (None if ol is None else ol[idx])

    def match(self, rows, rlens=None, fixed_len=None):
        r = rows.numpy().view(np.uint64)
        res = oracle.search_batch(self.S, self.sa, r, None if rlens is None else rlens.numpy().view(np.uint32),
                                  fixed_len=fixed_len)
        return torch.from_numpy(np.clip(res.astype(np.int64), self.r0, self.r1).astype(np.int32))

    def part_collect(self, back, offs, order, Q, out=None):
        o = offs.tolist()
        b = back.numpy().astype(np.int64)
        P, n_long = self.P, o[self.P]
        n_short = Q - n_long
        res = np.empty((Q, 2), np.int64)
        for g in range(P):
            B = o[g] + g * n_short
            res[o[g]:o[g + 1]] = b[B:B + o[g + 1] - o[g]]
        acc = np.zeros((n_short, 2), np.int64)
        for g in range(P):
            s0 = o[g + 1] + g * n_short
            acc += b[s0:s0 + n_short] - self.ranks[g]
        res[n_long:] = acc
        out = np.empty_like(res)
        out[order.numpy()] = res
        return torch.from_numpy(out.astype(np.int32))


def _part_worker(rank, world, port, outq):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ref = synth.reference(synth.REF_REPEAT, N_REF, 9)
    S = oracle.encode(ref)
    sa_ref = oracle.sa_naive(S)
    part = FakePart(S, sa_ref, rank, world, 4)
    # each rank its own batch, with reads shorter than the route key (sent to every part), and m = 0
    words, lens = synth.reads(ref, 400 + 37 * rank, 0, 40, 0.1, 0.0, 20 + rank)
    got = shard.partitioned_match(part, torch.from_numpy(words.view(np.int64)), torch.from_numpy(lens.view(np.int32)))
    want = oracle.search_batch(S, sa_ref, words, lens).astype(np.int64)
    outq.put((rank, bool(np.array_equal(got.numpy().astype(np.int64) & 0xFFFFFFFF, want)), int((lens < 4).sum())))
    dist.barrier()
    dist.destroy_process_group()


def test_partitioned_exchange_two_ranks_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_part_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert all(nshort > 0 for _, _, nshort in res)  # the multi-part (short read) path ran on both ranks
