"""the partitioned index (csrc/sa_part.cu) against the ORACLE.

Each part is built alone (its slice of the suffix array, of the k-mer table and of the records; the other
parts' suffixes are never sorted).  Checked here, through the C ABI, on one GPU:
  * every part's SA slice equals the oracle's comparison-sort SA over the part's rank range, the slices
    tile [0, n), and each part's table slice equals the oracle's histogram table clamped to its ranks;
  * route -> pack -> each part matches its block -> collect gives exactly the oracle's intervals for every
    read, including reads shorter than the route key (sent to every part and summed), m = 0, reads
    shorter than k, and the hazard reads of tests/test_gpu_parity.py;
  * a part holds ~1/nparts of the replicated index's suffix array.
The all-to-all between ranks is emulated in-process here (one rank holds the batch and every part);
tests/test_dist_gloo.py runs the same exchange over a real 2-process group."""
import random

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
import paper_1303_3692_b200 as sa  # noqa: E402

pytestmark = pytest.mark.gpu


def _cuda(a, dt):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a).view(dt)).cuda()


def emulate(parts, words, lens, fixed_len=None):
    """One requester, every part in this process: the exchange of shard.partitioned_match without the
    collective (block g of the send buffer is part g's whole input; its answers come back in place)."""
    w, l = _cuda(words, np.int64), _cuda(lens, np.int32)
    Q = w.shape[0]
    order, ow, ol, offs = parts[0].route(w, l, fixed_len=fixed_len)
    o = offs.cpu().tolist()
    P = len(parts)
    n_short = Q - o[P]
    send = [o[g + 1] - o[g] + n_short for g in range(P)]
    sw, sl = parts[0].part_pack(ow, ol, offs, sum(send))
    back, b0 = [], 0
    for g in range(P):
        rows = sw[b0:b0 + send[g]]
        rl = None if sl is None else sl[b0:b0 + send[g]]
        back.append(parts[g].match(rows, rl, fixed_len=fixed_len) if send[g] else
                    torch.empty((0, 2), dtype=torch.int32, device="cuda"))
        b0 += send[g]
    out = parts[0].part_collect(torch.cat(back), offs, order, Q)
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint32), o


def hazard_reads(text, rng, k, rb):
    n = len(text)
    qs = ["", text[:40], text[-1:] + "T", "A" * 150, "T" * 150]
    for j in range(1, k + 3):
        qs += [text[n - j:], text[n - j:] + "A", text[n - j:] + "T"]
    for m in sorted({1, 2, rb - 1, rb, rb + 1, k - 1, k, k + 1, 31, 32, 33, 100, 150}):
        if m <= 0:
            continue
        qs += ["A" * m, "T" * m, "".join(rng.choice("ACGT") for _ in range(m))]
        if m <= n:
            i = rng.randrange(n - m + 1)
            qs.append(text[i:i + m])
    for _ in range(600):  # many short reads: they are the multi-part case
        m = rng.randint(0, rb + 2)
        i = rng.randrange(n - m + 1)
        qs.append(text[i:i + m] if rng.random() < 0.8 else "".join(rng.choice("ACGT") for _ in range(m)))
    return qs


@pytest.mark.parametrize("layout", ["rec32", "rec16", "plain"])
@pytest.mark.parametrize("nparts", [2, 3, 7])
def test_partitions_equal_oracle(layout, nparts):
    ref = synth.reference(synth.REF_REPEAT, 2_000_000, 91)
    text = ref.tobytes().decode()
    S = oracle.encode(ref)
    sa_ref = oracle.sa_naive(S)
    rb = 8
    parts = [sa.Index(ref, layout=layout, part=(g, nparts, rb)) for g in range(nparts)]
    k = parts[0].k
    T = oracle.kmer_table(S, k)
    infos = [p.part_info() for p in parts]
    assert infos[0]["rank_lo"] == 0 and infos[-1]["rank_hi"] == len(ref)
    for g, (a, p) in enumerate(zip(infos, parts)):
        assert a["part_ranks"] == infos[0]["part_ranks"] and a["part_ranks"][g] == a["rank_lo"]
        if g + 1 < nparts:
            assert a["rank_hi"] == infos[g + 1]["rank_lo"]  # the slices tile the SA
        # the slice's suffix array, built alone, is the oracle's SA over the slice's ranks
        assert np.array_equal(p.export_sa(), sa_ref[a["rank_lo"]:a["rank_hi"]])
        # the table slice: the oracle's table over the part's k-mers, clamped to its ranks
        sh = 2 * (k - rb)
        x0, x1 = a["part_keys"][g] << sh, a["part_keys"][g + 1] << sh
        want_t = np.clip(T[x0:x1 + 1].astype(np.int64), a["rank_lo"], a["rank_hi"]).astype(np.uint32)
        assert np.array_equal(p.export_table(), want_t)
        # balanced: ~1/nparts of the suffixes each
        assert abs((a["rank_hi"] - a["rank_lo"]) - len(ref) / nparts) < 0.2 * len(ref) / nparts
    words, lens = synth.reads(ref, 60_000, 16, 160, 0.1, 0.01, 92)
    rng = random.Random(nparts)
    hw, hl = synth.pack_strings(hazard_reads(text, rng, k, rb), stride=words.shape[1])
    words = np.concatenate([words, hw])
    lens = np.concatenate([lens, hl])
    want = oracle.search_batch(S, sa_ref, words, lens).astype(np.uint32)
    got, offs = emulate(parts, words, lens)
    assert offs[nparts] < len(lens)  # some reads were short (m < rb): the multi-part case ran
    bad = np.nonzero((got != want).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first q={bad[0]} m={lens[bad[0]]}: {got[bad[0]]} vs {want[bad[0]]}"


def test_partition_memory_is_a_slice():
    ref = synth.reference(synth.REF_REPEAT, 3_000_000, 93)
    full = sa.Index(ref, layout="rec32")
    nparts = 4
    parts = [sa.Index(ref, layout="rec32", part=(g, nparts, 8)) for g in range(nparts)]
    text_bytes = ((len(ref) + 31) // 32 + 6) * 8
    full_sa = full.device_bytes - text_bytes - ((1 << (2 * full.k)) + 1) * 4
    for p in parts:
        pi = p.part_info()
        own = (pi["rank_hi"] - pi["rank_lo"]) * 32
        assert own < 0.3 * full_sa
        # text + records slice + table slice + route table + rank boundaries, nothing more
        g = pi["part"]
        table = ((pi["part_keys"][g + 1] - pi["part_keys"][g]) << (2 * (full.k - 8))) + 1
        assert p.device_bytes == text_bytes + own + table * 4 + (4 ** 8 + 1) * 4 + (nparts + 1) * 8


def test_partition_fixed_length_and_dense_words():
    ref = synth.reference(synth.REF_UNIFORM, 300_000, 5)
    S = oracle.encode(ref)
    parts = [sa.Index(ref, part=(g, 2, 4)) for g in range(2)]
    words, lens = synth.reads(ref, 5000, 32, 32, 0.1, 0.0, 6)
    want = oracle.search_batch(S, oracle.sa_naive(S), words, lens).astype(np.uint32)
    got, _ = emulate(parts, words, None, fixed_len=32)
    assert np.array_equal(got, want)
    # fixed length below the route key: every read goes to every part
    w3, l3 = synth.reads(ref, 3000, 3, 3, 0.0, 0.0, 7)
    want3 = oracle.search_batch(S, oracle.sa_naive(S), w3, l3).astype(np.uint32)
    got3, offs3 = emulate(parts, w3, None, fixed_len=3)
    assert offs3[2] == 0 and np.array_equal(got3, want3)


def test_partition_rejects_bad_arguments():
    ref = synth.reference(synth.REF_UNIFORM, 100_000, 5)
    with pytest.raises(sa.SAError):
        sa.Index(ref, part=(0, 1, 4))        # nparts >= 2
    with pytest.raises(sa.SAError):
        sa.Index(ref, k=6, part=(0, 2, 6))   # route_bases < k
    with pytest.raises(sa.SAError):
        sa.Index(ref, part=(0, 2, 13))       # route_bases <= 12
