"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Index: the GPU suffix array must equal the oracle's comparison-sort SA (small / medium sizes) or
pass the oracle's SA check (permutation + strictly increasing adjacent suffixes) at full size; the
k-mer table must equal the oracle's histogram table.  Match: every (lo, hi) must equal the
oracle's textbook search (bit-exact, integers); at full size, a seeded sample is compared with the
oracle's streaming counting oracle (no SA) and every query passes the oracle's certificate.
"""
import itertools
import random

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
import paper_1303_3692_b200 as sa  # noqa: E402

pytestmark = pytest.mark.gpu


def _text(s):
    return s.encode("ascii") if isinstance(s, str) else s


def gpu_match(idx, words, lens=None, fixed_len=None, presort=False, want_stats=False, cooperative=False):
    w = torch.from_numpy(np.ascontiguousarray(words).view(np.int64)).cuda()
    l = None if lens is None else torch.from_numpy(np.ascontiguousarray(lens).view(np.int32)).cuda()
    res = idx.match(w, l, fixed_len=fixed_len, presort=presort, want_stats=want_stats, cooperative=cooperative)
    torch.cuda.synchronize()
    if want_stats:
        return res[0].cpu().numpy().view(np.uint32), res[1].cpu().numpy().view(np.uint32)
    return res.cpu().numpy().view(np.uint32)


LAYOUTS = ["rec16", "rec32", "plain"]


def check_full(text_ascii, queries=None, words=None, lens=None, k=0, check_sa=True, layout="rec16", subtables=False,
               cooperative=(False,)):
    """Build on the GPU; compare SA, table and every interval with the oracle."""
    S = oracle.encode(text_ascii)
    idx = sa.Index(text_ascii, k=k, layout=layout, subtables=subtables)
    sa_ref = oracle.sa_naive(S)
    if check_sa:
        assert np.array_equal(idx.export_sa(), sa_ref)
    if idx.k <= 8:
        assert np.array_equal(idx.export_table(), oracle.kmer_table(S, idx.k))
    if queries is not None:
        words, lens = synth.pack_strings(queries)
    want = oracle.search_batch(S, sa_ref, words, lens).astype(np.uint32)
    for presort in (False, True):
        for coop in cooperative:
            got = gpu_match(idx, words, lens, presort=presort, cooperative=coop)
            bad = np.nonzero((got != want).any(axis=1))[0]
            assert bad.size == 0, f"{bad.size} mismatches (layout={layout}, presort={presort}, cooperative={coop}), " \
                                  f"first q={bad[0]}: got {got[bad[0]]} want {want[bad[0]]}"
    return idx, S, sa_ref, got


def hazard_queries(text, k, rng, extra=200):
    n = len(text)
    qs = ["", text[: min(n, 40)], text[-1:] + "t"]
    for j in range(1, k + 3):
        if j <= n:
            qs.append(text[n - j:])                 # the last j bases
            qs.append(text[n - j:] + "A")           # running past the end
            qs.append(text[n - j:] + "T")
    for m in sorted({1, max(1, k - 1), k, k + 1, 31, 32, 33, 63, 64, 65, 100, 127, 128}):
        qs.append("A" * m)
        qs.append("T" * m)
        if m <= n:
            i = rng.randrange(n - m + 1)
            qs.append(text[i:i + m])
            s = text[i:i + m]
            j = rng.randrange(m)
            qs.append(s[:j] + "ACGT".replace(s[j], "")[rng.randrange(3)] + s[j + 1:])
        qs.append("".join(rng.choice("ACGT") for _ in range(m)))
    for _ in range(extra):
        m = rng.randint(1, 128)
        if m <= n and rng.random() < 0.7:
            i = rng.randrange(n - m + 1)
            qs.append(text[i:i + m])
        else:
            qs.append("".join(rng.choice("ACGT") for _ in range(m)))
    qs += qs[:10]  # duplicates
    return qs


# ---- the paper's worked example --------------------------------------------------------------

def test_paper_example_table1_and_sec4():
    idx = sa.Index("acggtacgtac")
    assert idx.export_sa().tolist() == [9, 0, 5, 10, 1, 6, 2, 7, 3, 8, 4]   # Table I
    words, lens = synth.pack_strings(["a", "c", "ggtac", "tac", "tt", "gg", "acggtacgtac", ""])
    got = gpu_match(idx, words, lens)
    assert got.tolist() == [[0, 3], [3, 6], [6, 7], [9, 11], [11, 11], [6, 7], [1, 2], [0, 11]]
    offs, pos = idx.locate(torch.from_numpy(got.view(np.int32)).cuda())
    assert pos.cpu().numpy()[:3].tolist() == [9, 0, 5]  # "namely 9, 0, 5"


# ---- small adversarial texts: SA, table and intervals bit-exact --------------------------------

@pytest.mark.parametrize("plain", LAYOUTS)  # the SA layout
@pytest.mark.parametrize("n", [1, 2, 5, 31, 32, 33, 63, 64, 65, 1000, 4097])
@pytest.mark.parametrize("k", [0, 1, 3, 6, 16])
def test_random_texts_all_k(n, k, plain):
    rng = random.Random(n * 10 + k)
    text = "".join(rng.choice("ACGT") for _ in range(n))
    check_full(text, hazard_queries(text, k or 6, rng), k=k, layout=plain)


@pytest.mark.parametrize("text", [
    "A" * 5000,
    "AC" * 3000,
    "ACGT" * 1500 + "A",
    "T" * 777 + "A" * 333,
    "ACGTTGCA" * 900,
])
@pytest.mark.parametrize("plain", LAYOUTS)  # the SA layout
def test_periodic_and_homopolymer_texts(text, plain):
    rng = random.Random(len(text))
    check_full(text, hazard_queries(text, 8, rng), k=8, layout=plain)


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("k", [2, 3, 5])
def test_subtables_for_large_buckets(k, layout):
    # small k on a few-kbp text: most buckets exceed 32 suffixes, so the (k+4)-base sub-tables are used
    rng = random.Random(k)
    for n in [3000, 20000]:
        text = "".join(rng.choice("ACGT") for _ in range(n)) + "A" * 300 + "AC" * 200
        check_full(text, hazard_queries(text, k, rng, extra=400), k=k, layout=layout, subtables=True)


@pytest.mark.parametrize("layout", LAYOUTS)
def test_subtables_k16_all_t_bucket(layout):
    # k = 16: the all-T bucket's k-mer is 0xFFFFFFFF.  A poly-T run of 300 bases puts 285 suffixes in it
    # (> 32: it gets a sub-table), next to poly-A (bucket 0) and other large buckets.
    rng = random.Random(16)
    rnd = lambda n: "".join(rng.choice("ACGT") for _ in range(n))
    text = rnd(5000) + "T" * 300 + rnd(3000) + "A" * 200 + rnd(2000) + "TTTTTTTTTTTTTTTTG" * 40 + rnd(1000) + "T" * 60
    qs = hazard_queries(text, 16, rng, extra=300)
    qs += ["T" * m for m in range(14, 320, 3)] + ["T" * m + "G" for m in range(15, 70, 4)]
    qs += ["A" * m for m in range(14, 220, 5)] + ["TTTTTTTTTTTTTTTTG" * r for r in (1, 2, 5, 41)]
    check_full(text, qs, k=16, layout=layout, subtables=True)


@pytest.mark.parametrize("k", [0, 6, 10, 14])
def test_bucket_trees_equal_oracle(k):
    """SA_INDEX_BUCKET_TREE (large buckets' binary-search pivots in line-packed trees) gives the oracle's
    intervals: a repeat-rich reference + homopolymer / periodic runs (buckets of thousands of suffixes),
    reads of 10-300 bases (short, record-decided and long two-phase kernels), the hazard batch."""
    rng = random.Random(k)
    ref = synth.reference(synth.REF_REPEAT, 1_500_000, 57).tobytes().decode()
    ref += "A" * 3000 + "AC" * 2000 + "".join(rng.choice("ACGT") for _ in range(5000)) + "ACGTTGCA" * 700
    words, lens = synth.reads(np.frombuffer(ref.encode(), dtype=np.uint8), 60_000, 10, 300, 0.1, 0.02, 58)
    hw, hl = synth.pack_strings(hazard_queries(ref, k or 12, rng, extra=200) +
                                ["A" * m for m in (12, 40, 100, 200, 300)] + ["AC" * 60, "ACGTTGCA" * 30],
                                stride=words.shape[1])
    words, lens = np.concatenate([words, hw]), np.concatenate([lens, hl])
    idx, S, sa_ref, got = check_full(ref, words=words, lens=lens, k=k, layout="rec32", check_sa=False)
    tree = sa.Index(ref, k=k, layout="rec32", bucket_tree=True)
    assert tree.device_bytes > idx.device_bytes  # some buckets got trees
    want = oracle.search_batch(S, sa_ref, words, lens).astype(np.uint32)
    for presort in (False, True):
        g = gpu_match(tree, words, lens, presort=presort)
        bad = np.nonzero((g != want).any(axis=1))[0]
        assert bad.size == 0, f"{bad.size} mismatches, first {bad[0]} m={lens[bad[0]]}: {g[bad[0]]} vs {want[bad[0]]}"


def test_subtables_repeat_rich():
    ref = synth.reference(synth.REF_REPEAT, 3_000_000, 35)
    words, lens = synth.reads(ref, 200_000, 16, 160, 0.1, 0.01, 36)
    check_full(ref.tobytes(), words=words, lens=lens, layout="rec32", subtables=True)


def test_homopolymer_closed_form():
    n = 3000
    idx = sa.Index("A" * n, k=5)
    assert idx.export_sa().tolist() == list(range(n - 1, -1, -1))
    ks = [1, 2, 4, 5, 6, 100, 2999, 3000]
    words, lens = synth.pack_strings(["A" * kk for kk in ks])
    got = gpu_match(idx, words, lens)
    assert got.tolist() == [[kk - 1, n] for kk in ks]


def de_bruijn(k):
    a = [0] * (4 * k)
    seq = []

    def db(t, p):
        if t > k:
            if k % p == 0:
                seq.extend(a[1:p + 1])
        else:
            a[t] = a[t - p]
            db(t + 1, p)
            for j in range(a[t - p] + 1, 4):
                a[t] = j
                db(t + 1, t)

    db(1, 1)
    s = "".join("ACGT"[i] for i in seq)
    return s + s[:k - 1]


def test_de_bruijn_every_kmer_once():
    kk = 6
    text = de_bruijn(kk)
    kmers = ["".join(p) for p in itertools.product("ACGT", repeat=kk)]
    idx, S, sa_ref, got = check_full(text, kmers, k=4)
    assert np.all(got[:, 1] - got[:, 0] == 1)


@pytest.mark.parametrize("plain", LAYOUTS)  # the SA layout
def test_short_queries_below_k(plain):
    # m < k exercises the widened brackets
    rng = random.Random(7)
    for n in [20, 300, 5000]:
        text = "".join(rng.choice("AC") for _ in range(n)) + "".join(rng.choice("ACGT") for _ in range(n))
        qs = ["".join(p) for m in range(1, 5) for p in itertools.product("ACGT", repeat=m)]
        qs += [text[-j:] for j in range(1, 12)]
        check_full(text, qs, k=10, layout=plain)


def test_long_reads_generic_path():
    # stride > 4 words: the generic (global-memory query) kernel, reads up to 1000 bp with long matches
    ref = synth.reference(synth.REF_REPEAT, 400_000, 21)
    for plain in LAYOUTS:  # the SA layout
        words, lens = synth.reads(ref, 3000, 150, 1000, 0.1, 0.2, 22)
        check_full(ref.tobytes(), words=words, lens=lens, layout=plain, cooperative=(False, True))


@pytest.mark.parametrize("m_max", [160, 256])
def test_reads_of_129_to_256_bases(m_max):
    # strides 5..8 words: the generic (global-memory read) path with records and text past the cache
    ref = synth.reference(synth.REF_REPEAT, 500_000, 31)
    for layout in LAYOUTS:
        words, lens = synth.reads(ref, 4000, 100, m_max, 0.1, 0.1, 32)
        check_full(ref.tobytes(), words=words, lens=lens, layout=layout)


@pytest.mark.parametrize("m_max", [256, 512, 1024, 2048, 3000])
def test_group_kernel_hazards(m_max):
    # strides > 4 words: the one-thread-per-read long-read path and SA_MATCH_COOPERATIVE's group kernel
    # (G = 8 / 16 / 32 lanes per read; 2 words per lane up to 2048 bases, words from memory beyond): the hazard batch (short reads, m < k, the empty
    # read, text tails, reads running past the end) plus long exact, mutated and tail reads of up to m_max
    rng = random.Random(m_max)
    ref = synth.reference(synth.REF_REPEAT, 300_000, 71).tobytes().decode()
    n = len(ref)
    qs = hazard_queries(ref, 16, rng, extra=100)
    for _ in range(300):
        m = rng.randint(129, m_max)
        i = rng.randrange(n - m + 1)
        s = ref[i:i + m]
        r = rng.random()
        if r < 0.4:
            qs.append(s)
        elif r < 0.7:  # one substitution, anywhere (also past the 112 cached bases)
            j = rng.randrange(m)
            qs.append(s[:j] + "ACGT".replace(s[j], "")[rng.randrange(3)] + s[j + 1:])
        elif r < 0.85:  # a text tail running past the end
            qs.append(ref[n - rng.randint(1, m):] + "".join(rng.choice("ACGT") for _ in range(rng.randint(0, 40))))
        else:
            qs.append(ref[n - m:])  # the last m bases: a suffix exactly as long as the read
    qs.append("A" * m_max)
    for layout in LAYOUTS:
        check_full(ref, qs, layout=layout, cooperative=(False, True))


def test_stats_iteration_bound():
    # SA_MATCH_STATS: steps per boundary search never exceed ceil(log2(n+2)); joint lo+hi <= 2x
    ref = synth.reference(synth.REF_REPEAT, 1_000_000, 41)
    words, lens = synth.reads(ref, 50_000, 20, 100, 0.1, 0.0, 42)
    idx = sa.Index(ref)
    got, st = gpu_match(idx, words, lens, want_stats=True)
    S = oracle.encode(ref)
    assert np.array_equal(got, oracle.search_batch(S, oracle.sa_naive(S), words, lens).astype(np.uint32))
    steps = st[0] & 0xFFFF
    import math
    assert steps.max() <= 2 * math.ceil(math.log2(len(ref) + 2))
    # algorithmic bytes: at least the packed read + table pair + result, at most 4 + ceil(m/4) + 1 per step
    ub = st[1].astype(np.int64)
    m = lens.astype(np.int64)
    floor = (m + 3) // 4 + 8
    assert np.all(ub >= floor)
    assert np.all(ub <= floor + 8 + steps * (4 + (m + 3) // 4 + 1))


@pytest.mark.parametrize("key_bases", [0, 8, 16])
def test_order_is_a_sorted_permutation_and_keeps_results(key_bases):
    ref = synth.reference(synth.REF_REPEAT, 2_000_000, 51)
    words, lens = synth.reads(ref, 100_000, 10, 100, 0.1, 0.0, 52)
    idx = sa.Index(ref, k=14)
    w = torch.from_numpy(words.view(np.int64)).cuda()
    l = torch.from_numpy(lens.view(np.int32)).cuda()
    order = idx.order(w, l, key_bases=key_bases).cpu().numpy().view(np.uint32)
    assert np.array_equal(np.sort(order), np.arange(100_000, dtype=np.uint32))
    kb = key_bases or 12
    key = (words[:, 0] >> np.uint64(64 - 2 * kb)).astype(np.uint64)
    m = lens.astype(np.uint64)
    short = m < kb
    key[short] &= ~((np.uint64(1) << (np.uint64(2) * (np.uint64(kb) - m[short]))) - np.uint64(1))
    ks = key[order]
    assert np.all(ks[1:] >= ks[:-1])
    # stable: equal keys keep the reads' input order
    eq = ks[1:] == ks[:-1]
    assert np.all(order[1:][eq] > order[:-1][eq])
    base = idx.match(w, l)
    got = idx.match(w, l, order=torch.from_numpy(order.view(np.int32)).cuda())
    assert torch.equal(got, base)
    # the rows arranged in that order (SA_MATCH_ROWS_ORDERED) give the same intervals at the same places
    ow, ol = torch.empty_like(w), torch.empty_like(l)
    perm = idx.order(w, l, key_bases=key_bases, ordered_words=ow, ordered_lens=ol)
    assert torch.equal(ow, w[perm.long()]) and torch.equal(ol, l[perm.long()])
    got2 = idx.match(ow, ol, order=perm, rows_ordered=True)
    assert torch.equal(got2, base)


@pytest.mark.parametrize("key_bases", [0, 6, 13])
@pytest.mark.parametrize("dense", [False, True])
def test_order_buckets_is_a_key_sorted_permutation(key_bases, dense):
    """SA_ORDER_BUCKETS: the same bucket (key) order as the stable sort, equal keys in any order; the match
    through that order equals the oracle.  Repeat-rich reads (thousands share a key: the warp-aggregated slot
    claims), reads shorter than the key (masked keys), Q not a multiple of the warp, the dense layout."""
    ref = synth.reference(synth.REF_REPEAT, 1_000_000, 61)
    rng = np.random.default_rng(5)
    if dense:  # equal lengths; rebuilt from strings so both layouts hold the same reads
        m = 50
        w0, l0 = synth.reads(ref, 30_000, m, m, 0.1, 0.0, 62)
        qs = [synth.unpack_read(w0[i], m) for i in range(len(l0))] + ["A" * m] * 3000 + [("ACGT" * 20)[:m]] * 500
        qs = [qs[i] for i in rng.permutation(len(qs))]
        words, lens = synth.pack_strings(qs)
        dense_words = synth.pack_dense(qs)
    else:
        words, lens = synth.reads(ref, 77_777, 3, 100, 0.1, 0.0, 62)
        hot, hl = synth.pack_strings(["A" * 40] * 3000 + ["ACGTACGTACGTAC"] * 500, stride=words.shape[1])
        words = np.concatenate([words, hot])
        lens = np.concatenate([lens, hl])
        p = rng.permutation(len(lens))
        words, lens = np.ascontiguousarray(words[p]), np.ascontiguousarray(lens[p])
    Q = len(lens)
    idx = sa.Index(ref, k=12)
    S = oracle.encode(ref)
    want = oracle.search_batch(S, oracle.sa_naive(S), words, lens).astype(np.uint32)
    kb = key_bases or 12
    key = (words[:, 0] >> np.uint64(64 - 2 * kb)).astype(np.uint64)
    mm = lens.astype(np.uint64)
    short = mm < kb
    key[short] &= ~((np.uint64(1) << (np.uint64(2) * (np.uint64(kb) - mm[short]))) - np.uint64(1))
    if dense:
        dw = torch.from_numpy(dense_words.view(np.int64)).cuda()
        order = idx.order(dw, None, fixed_len=m, key_bases=key_bases, n_reads=Q, buckets=True)
        got = idx.match(dw, None, fixed_len=m, order=order, n_reads=Q)
    else:
        w = torch.from_numpy(words.view(np.int64)).cuda()
        l = torch.from_numpy(lens.view(np.int32)).cuda()
        order = idx.order(w, l, key_bases=key_bases, buckets=True)
        got = idx.match(w, l, order=order)
    torch.cuda.synchronize()
    o = order.cpu().numpy().view(np.uint32)
    assert np.array_equal(np.sort(o), np.arange(Q, dtype=np.uint32))
    ks = key[o]
    assert np.all(ks[1:] >= ks[:-1])
    assert np.array_equal(got.cpu().numpy().view(np.uint32), want)


@pytest.mark.parametrize("layout", ["rec16", "rec32"])
@pytest.mark.parametrize("k", [0, 8, 12])
@pytest.mark.parametrize("levels", [1, 5, 8, 12])
def test_smem_tree_equals_oracle(layout, k, levels):
    """SA_MATCH_SMEM_TREE (the per-CTA shared-memory top tree staged by TMA bulk copies) gives the oracle's
    intervals: ordered reads of 10-128 bases (short reads take the plain path), a repeat-rich reference,
    table k below / at / above the order's 12-base key."""
    ref = synth.reference(synth.REF_REPEAT, 2_000_000, 55)
    words, lens = synth.reads(ref, 100_000, 10, 128, 0.1, 0.02, 56)
    rng = random.Random(levels)
    hw, hl = synth.pack_strings(hazard_queries(ref.tobytes().decode(), 12, rng, extra=100), stride=4)
    words, lens = np.concatenate([words, hw]), np.concatenate([lens, hl])
    idx = sa.Index(ref, k=k, layout=layout)
    S = oracle.encode(ref)
    want = oracle.search_batch(S, oracle.sa_naive(S), words, lens).astype(np.uint32)
    w = torch.from_numpy(words.view(np.int64)).cuda()
    l = torch.from_numpy(lens.view(np.int32)).cuda()
    for kb in (8, 12, 16):
        perm = idx.order(w, l, key_bases=kb)
        got = idx.match(w, l, order=perm, smem_tree=levels, tree_key_bases=kb).cpu().numpy().view(np.uint32)
        bad = np.nonzero((got != want).any(axis=1))[0]
        assert bad.size == 0, f"kb={kb}: {bad.size} mismatches, first {bad[0]}: {got[bad[0]]} vs {want[bad[0]]}"


def _stable_key_order(words, lens, kb):
    key = (words[:, 0] >> np.uint64(64 - 2 * kb)).astype(np.uint64)
    m = lens.astype(np.uint64)
    short = m < kb
    key[short] &= ~((np.uint64(1) << (np.uint64(2) * (np.uint64(kb) - m[short]))) - np.uint64(1))
    return np.argsort(key, kind="stable").astype(np.uint32)


_ORDER_INDEX = []


@pytest.mark.parametrize("Q", [1, 31, 65536 * 3 + 17])
@pytest.mark.parametrize("skew", ["random", "one_key", "few_keys"])
@pytest.mark.parametrize("key_bases", [1, 4, 7, 10, 12, 13, 16])
def test_order_equals_stable_argsort(Q, skew, key_bases):
    """sa_match_order = the stable sort of the reads by their first key_bases bases, bit-exact: random,
    one-key and few-key batches, reads shorter than the key (masked), Q across sort-tile sizes."""
    if not _ORDER_INDEX:
        _ORDER_INDEX.append(sa.Index(synth.reference(synth.REF_UNIFORM, 100_000, 71)))
    idx = _ORDER_INDEX[0]
    rng = np.random.default_rng(72 + Q + key_bases)
    words = rng.integers(0, 2**63, size=(Q, 2), dtype=np.int64).view(np.uint64)
    if skew == "one_key":
        words[:, 0] = np.uint64(0x1B1B1B1B1B1B1B1B)
    elif skew == "few_keys":
        words[:, 0] = np.array([0, 0xFFFFFFFFFFFFFFFF, 0x5555555555555555], dtype=np.uint64)[rng.integers(0, 3, Q)]
    lens = rng.integers(0, 65, size=Q).astype(np.uint32)
    w = torch.from_numpy(words.view(np.int64)).cuda()
    l = torch.from_numpy(lens.view(np.int32)).cuda()
    got = idx.order(w, l, key_bases=key_bases).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, _stable_key_order(words, lens, key_bases))


@pytest.mark.parametrize("m", [12, 31, 32, 100, 128, 150, 1000])
def test_dense_layout_matches_strided(m):
    ref = synth.reference(synth.REF_REPEAT, 1_000_000, 61)
    Q = 4096 + 32 * 7
    words, lens = synth.reads(ref, Q, m, m, 0.1, 0.05, 62)
    dense, _ = synth.reads(ref, Q, m, m, 0.1, 0.05, 62, dense=True)
    idx = sa.Index(ref, layout="rec32")
    S = oracle.encode(ref)
    want = oracle.search_batch(S, oracle.sa_naive(S), words, lens).astype(np.uint32)
    d = torch.from_numpy(dense.view(np.int64)).cuda()
    got = idx.match(d, None, fixed_len=m, n_reads=Q).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want)
    perm = idx.order(d, None, fixed_len=m, n_reads=Q)
    got2 = idx.match(d, None, fixed_len=m, n_reads=Q, order=perm).cpu().numpy().view(np.uint32)
    assert np.array_equal(got2, want)
    got3 = idx.match_host(dense, None, fixed_len=m, n_reads=Q, chunk=1000)
    assert np.array_equal(got3, want)


def test_symbol_error_reports_position():
    with pytest.raises(sa.SAError) as e:
        sa.Index("ACGTACGTNACGT")
    assert e.value.code == sa.SA_ESYMBOL and "position 8" in e.value.detail


def test_lowercase_reference():
    text = "acggtacgtac"
    assert sa.Index(text.upper()).export_sa().tolist() == sa.Index(text).export_sa().tolist()


# ---- BASELINE.json configs ----------------------------------------------------------------------

@pytest.mark.parametrize("plain", LAYOUTS)  # the SA layout
def test_c1_full_parity(plain):
    c = synth.CONFIGS["C1"]
    ref = c.reference()
    words, lens = c.reads(ref)
    idx, S, sa_ref, got = check_full(ref.tobytes(), words=words, lens=lens, layout=plain)
    assert idx.k == 10
    # the 10k exact reads all hit
    assert (got[:, 1] > got[:, 0]).sum() >= 10_000 * 0.99
    # same result through the fixed-length path and the host-buffer pipeline
    got_fixed = gpu_match(idx, words, None, fixed_len=32)
    assert np.array_equal(got, got_fixed)
    assert np.array_equal(idx.match_host(words, lens, chunk=3000), got)


@pytest.mark.parametrize("plain", LAYOUTS)  # the SA layout
def test_c2_full_parity(plain):
    c = synth.CONFIGS["C2"]
    ref = c.reference()
    words, lens = c.reads(ref)
    check_full(ref.tobytes(), words=words, lens=lens, layout=plain)


@pytest.mark.parametrize("plain", LAYOUTS)  # the SA layout
@pytest.mark.parametrize("k", [0, 14])
def test_repeat_rich_parity_small(plain, k):
    ref = synth.reference(synth.REF_REPEAT, 3_000_000, 33)
    words, lens = synth.reads(ref, 200_000, 16, 160, 0.1, 0.01, 34)
    check_full(ref.tobytes(), words=words, lens=lens, layout=plain, k=k)


@pytest.mark.parametrize("plain", LAYOUTS)  # the SA layout
def test_locate_parity(plain):
    ref = synth.reference(synth.REF_REPEAT, 500_000, 5)
    words, lens = synth.reads(ref, 20_000, 8, 40, 0.1, 0.0, 6)
    idx, S, sa_ref, got = check_full(ref.tobytes(), words=words, lens=lens, layout=plain)
    offs, pos = idx.locate(torch.from_numpy(got.view(np.int32)).cuda())
    offs = offs.cpu().numpy()
    pos = pos.cpu().numpy().view(np.uint32)
    cnt = (got[:, 1].astype(np.int64) - got[:, 0])
    assert np.array_equal(np.diff(offs), cnt) and offs[0] == 0
    for q in range(0, 20_000, 97):
        assert np.array_equal(pos[offs[q]:offs[q + 1]], oracle.locate(sa_ref, int(got[q, 0]), int(got[q, 1])))


@pytest.mark.parametrize("plain", LAYOUTS)
def test_locate_heavy_reads(plain):
    # reads with > 4096 occurrences take the chunked (block per 4096 positions) path
    text = "A" * 30000 + "ACGT" * 3000 + "".join(random.Random(3).choice("ACGT") for _ in range(5000))
    qs = ["A" * m for m in (1, 3, 7, 100, 5000)] + ["ACGT", "AC", "GTA", "T", "CCCC"]
    idx, S, sa_ref, got = check_full(text, qs, layout=plain, k=6)
    offs, pos = idx.locate(torch.from_numpy(got.view(np.int32)).cuda())
    offs = offs.cpu().numpy()
    pos = pos.cpu().numpy().view(np.uint32)
    assert (got[:, 1].astype(np.int64) - got[:, 0]).max() > 4096
    for q in range(len(qs)):
        assert np.array_equal(pos[offs[q]:offs[q + 1]], oracle.locate(sa_ref, int(got[q, 0]), int(got[q, 1])))


def _full_size_check(cfg, sample=2000, q_count=None, layout="rec32"):
    """The bench configuration (bench.py defaults: rec32 records, auto k, reads ordered by 12 bases)."""
    ref = cfg.reference()
    S = oracle.encode(ref)
    idx = sa.Index(ref, layout=layout)
    sa_gpu = idx.export_sa()
    assert oracle.check_sa(S, sa_gpu) == -1, "GPU suffix array fails the oracle's SA check"
    words, lens = cfg.reads(ref, q_count=q_count)
    w = torch.from_numpy(words.view(np.int64)).cuda()
    l = None if cfg.m_min == cfg.m_max else torch.from_numpy(lens.view(np.int32)).cuda()
    fixed = cfg.m_max if l is None else None
    perm = idx.order(w, l, fixed_len=fixed, key_bases=12)
    got = idx.match(w, l, fixed_len=fixed, order=perm)
    torch.cuda.synchronize()
    got = got.cpu().numpy().view(np.uint32)
    del w, l, perm
    # sampled outputs straight from the definition (no SA)
    rng = np.random.default_rng(cfg.ref_seed)
    qs = np.sort(rng.choice(words.shape[0], size=min(sample, words.shape[0]), replace=False))
    want = oracle.count_batch(S, words[qs], lens[qs]).astype(np.uint32)
    assert np.array_equal(got[qs], want)
    # every read certified against the (verified) suffix array
    nbad, first = oracle.certificate(S, sa_gpu, words, got, lens)
    assert nbad == 0, f"{nbad} reads fail the certificate, first {first}"
    return idx


@pytest.mark.slow
def test_c3_full_size():
    _full_size_check(synth.CONFIGS["C3"])


@pytest.mark.slow
def test_c4_full_size():
    _full_size_check(synth.CONFIGS["C4"], sample=256)


@pytest.mark.slow
@pytest.mark.parametrize("m", [16, 32, 64, 150, 250, 500, 1000])
def test_c5_read_lengths_full_reference(m):
    # C5's reference (= C4's) at a sample of its read lengths; 2M reads per length
    _full_size_check(synth.CONFIGS["C5"].with_m(m), sample=128, q_count=2_000_000)


def test_k16_table_sampled_against_oracle():
    """The bench's k = 16 table (4^16 + 1 entries, 17 GB -- too large for the oracle's histogram table): T[x]
    = #{i : trunc_16(S_i) < x} = lo(x) for the 16-mer x, so sampled entries are checked against the oracle's
    textbook search of x (k-mers of the text, their neighbours, random, the first and last), plus T's
    monotonicity and T[4^16] = n over the whole exported table."""
    ref = synth.reference(synth.REF_REPEAT, 1_000_000, 81)
    idx = sa.Index(ref, k=16, layout="rec32")
    T = idx.export_table()
    assert T.size == (1 << 32) + 1 and T[-1] == len(ref)
    assert np.all(T[1:] >= T[:-1])
    S = oracle.encode(ref)
    sa_ref = oracle.sa_naive(S)
    rng = np.random.default_rng(82)
    pos = rng.integers(0, len(ref) - 16, 3000)
    codes = np.zeros(pos.size, dtype=np.uint64)
    for j in range(16):
        codes = (codes << np.uint64(2)) | S[pos + j].astype(np.uint64)
    xs = np.concatenate([codes, codes + np.uint64(1), codes - np.uint64(1),
                         rng.integers(0, 1 << 32, 2000, dtype=np.uint64),
                         np.array([0, 1, (1 << 32) - 1], dtype=np.uint64)]) & np.uint64((1 << 32) - 1)
    words = (xs << np.uint64(32)).reshape(-1, 1)
    want = oracle.search_batch(S, sa_ref, words, None, fixed_len=16)[:, 0]
    assert np.array_equal(T[xs.astype(np.int64)].astype(np.uint64), want)


@pytest.mark.parametrize("layout", ["rec16", "rec32"])
def test_staged_long_read_verification(layout):
    """The long-read kernel (k_match<0>; with SA_LIB_PATH=variants/libsa_staged.so k_match_staged, whose
    phase (B) windows are staged in shared memory by TMA bulk copies, sa_search_staged.cuh) against the
    oracle: unique loci (one verification), a 2-kb exact
    duplication (hi' - lo' = 2: the per-thread joint search), substitutions at the first staged base, in the
    middle and at the last base, reads running past the end of the text (suffix shorter than the read),
    more candidates per warp than staging slots (m = 3000: 4 slots), and the same batch through a read
    buffer that is only 8-byte aligned (the k_match<0> fallback)."""
    rng = random.Random(7)
    base = synth.reference(synth.REF_REPEAT, 200_000, 91).tobytes().decode()
    dup = base[50_000:52_000]
    ref = base[:120_000] + dup + base[120_000:]  # the 2-kb block twice
    n = len(ref)
    qs = []
    for m in [129, 140, 145, 200, 333, 500, 1000, 1500, 3000]:
        for _ in range(40):
            i = rng.randrange(n - m + 1)
            s = ref[i:i + m]
            r = rng.random()
            if r < 0.4:
                qs.append(s)
            else:
                j = rng.choice([128, 129, 144, m // 2, m - 1, rng.randrange(128, m)])
                j = min(max(j, 0), m - 1)
                qs.append(s[:j] + "ACGT".replace(s[j], "")[rng.randrange(3)] + s[j + 1:])
        if m <= 2000:
            o = 50_000 + rng.randrange(0, 2000 - m + 1)
            qs.append(base[o:o + m])  # inside the duplication: two occurrences
        qs.append(ref[n - m:])                                          # the last m bases
        qs.append(ref[n - m + 10:] + "ACGTACGTAC")                      # runs past the end by 10 bases
        qs.append(ref[n - (m - 5):] + "T" * 5)
    words, lens = synth.pack_strings(qs)
    S = oracle.encode(ref.encode())
    want = oracle.search_batch(S, oracle.sa_naive(S), words, lens).astype(np.uint32)
    idx = sa.Index(ref.encode(), layout=layout)
    for offset in (0, 1):  # 1: the rows start 8 bytes past a 16-byte boundary -> k_match<0>
        Q, stride = words.shape
        buf = torch.zeros(Q * stride + 2, dtype=torch.int64, device="cuda")
        w = buf[offset:offset + Q * stride].view(Q, stride)
        w.copy_(torch.from_numpy(words.view(np.int64)))
        l = torch.from_numpy(lens.view(np.int32)).cuda()
        for presort in (False, True):
            got = idx.match(w, l, presort=presort)
            torch.cuda.synchronize()
            got = got.cpu().numpy().view(np.uint32)
            bad = np.nonzero((got != want).any(axis=1))[0]
            assert bad.size == 0, f"offset {offset} presort {presort}: {bad.size} mismatches, q={bad[0]} m={lens[bad[0]]}"
    assert (want[:, 1] - want[:, 0] == 2).any()  # the duplication was exercised


@pytest.mark.parametrize("layout", LAYOUTS)
@pytest.mark.parametrize("defer", [1, 3, 6])
def test_defer_heavy_reads_equal_oracle(layout, defer):
    """SA_MATCH_DEFER: reads whose k-mer bracket holds more than 2^defer suffixes are searched in a second,
    full-warp pass from their saved bracket.  Repeat-rich reference (big buckets), reads of 3-128 bases
    (m < k: never deferred), the hazard batch, with and without an order, Q not a multiple of the warp;
    every interval equals the oracle's."""
    rng = random.Random(defer)
    ref = synth.reference(synth.REF_REPEAT, 600_000, 81)
    text = ref.tobytes().decode()
    words, lens = synth.reads(ref, 20_003, 3, 128, 0.1, 0.05, 82)
    hw, hl = synth.pack_strings(hazard_queries(text, 12, rng, extra=300) + ["A" * 60] * 100, stride=4)
    words, lens = np.concatenate([words, hw]), np.concatenate([lens, hl])
    S = oracle.encode(ref)
    want = oracle.search_batch(S, oracle.sa_naive(S), words, lens).astype(np.uint32)
    idx = sa.Index(ref, k=12, layout=layout)
    w = torch.from_numpy(words.view(np.int64)).cuda()
    l = torch.from_numpy(lens.view(np.int32)).cuda()
    for order in (None, idx.order(w, l)):
        got = idx.match(w, l, order=order, defer=defer)
        torch.cuda.synchronize()
        got = got.cpu().numpy().view(np.uint32)
        bad = np.nonzero((got != want).any(axis=1))[0]
        assert bad.size == 0, f"{bad.size} mismatches, q={bad[0]} m={lens[bad[0]]}: {got[bad[0]]} vs {want[bad[0]]}"
    with pytest.raises(sa.SAError):
        idx.match(w, l, defer=3, want_stats=True)


@pytest.mark.parametrize("layout", LAYOUTS)
def test_wide_batch_loads_equal_oracle(layout):
    """SA_MATCH_WIDE: the large-batch load hints (L2::64B for the read row and the table pair; automatic from
    2^20 reads) forced on a small batch: every interval equals the oracle's, strided rows of 1 / 2 / 4 words
    (the 128- and 256-bit row loads) and long reads, with and without an order."""
    ref = synth.reference(synth.REF_REPEAT, 700_000, 85)
    S = oracle.encode(ref)
    sa_ref = oracle.sa_naive(S)
    idx = sa.Index(ref, layout=layout)
    for m_lo, m_hi in [(5, 32), (33, 64), (65, 128), (100, 100), (129, 300)]:
        words, lens = synth.reads(ref, 20_000, m_lo, m_hi, 0.1, 0.05, 86 + m_hi)
        want = oracle.search_batch(S, sa_ref, words, lens).astype(np.uint32)
        w = torch.from_numpy(words.view(np.int64)).cuda()
        l = torch.from_numpy(lens.view(np.int32)).cuda()
        for order in (None, idx.order(w, l)):
            got = idx.match(w, l, order=order, wide=True)
            torch.cuda.synchronize()
            assert np.array_equal(got.cpu().numpy().view(np.uint32), want), (m_lo, m_hi, order is None)
