"""Pins for the CPU oracle (oracle/): the paper's worked examples, brute force on
tiny inputs through Python's own string order, closed forms and invariants.

Nothing here retypes the oracle's formulas: the SA pins come from PAPER.md's
tables, from `sorted(range(n), key=lambda i: text[i:])` (Python's built-in
lexicographic string order, where a proper prefix sorts first and 'a'<'c'<'g'<'t'),
and the interval pins from slicing + counting in Python.
"""
import itertools
import os
import random

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                k, v = line.split(":", 1)
                rows.append((k.strip(), v.strip()))
    return rows


def enc(s):
    return oracle.encode(s)


def brute_sa(text):
    return [i for i in sorted(range(len(text)), key=lambda i: text[i:])]


def brute_lohi(text, P):
    m = len(P)
    lo = sum(1 for i in range(len(text)) if text[i:i + m] < P)
    hi = sum(1 for i in range(len(text)) if text[i:i + m] <= P)
    return lo, hi


# ---- paper worked examples -------------------------------------------------------------------

def test_table1_suffix_array():
    g = dict(_golden("paper_table1.txt"))
    sa = oracle.sa_naive(enc(g["text"]))
    assert sa.tolist() == [int(x) for x in g["sa"].split()]


def test_table3_rank_array():
    g = dict(_golden("paper_table3.txt"))
    sa = oracle.sa_naive(enc(g["text"]))
    assert oracle.rank_array(sa).tolist() == [int(x) for x in g["rank"].split()]


def test_table2_dc3_sample_ranks_and_nonsample_order():
    # The SA restricted to the sample positions (i mod 3 != 0) gives Table II's ranks;
    # restricted to i mod 3 == 0 it gives the order S9 <= S0 <= S6 <= S3.
    g = dict(_golden("paper_table2_dc3.txt"))
    sa = oracle.sa_naive(enc(g["text"])).tolist()
    sample = [p for p in sa if p % 3 != 0]
    want = dict((int(a), int(b)) for a, b in (t.split(":") for t in g["sample_rank"].split()))
    assert {p: r + 1 for r, p in enumerate(sample)} == want
    assert [p for p in sa if p % 3 == 0] == [int(x) for x in g["nonsample_order"].split()]


def test_sec4_intervals_and_positions():
    rows = _golden("paper_sec4_intervals.txt")
    text = dict(rows)["text"]
    S = enc(text)
    sa = oracle.sa_naive(S)
    for k, v in rows:
        if k != "query":
            continue
        P, *kv = v.split()
        kv = dict(t.split("=") for t in kv)
        lo, hi = int(kv["lo"]), int(kv["hi"])
        assert oracle.search(S, sa, enc(P)) == (lo, hi)
        assert oracle.count(S, enc(P)) == (lo, hi)
        assert oracle.locate(sa, lo, hi).tolist() == [int(x) for x in kv["positions"].split(",")]


def test_spec_examples_corrected():
    for k, v in _golden("spec_examples.txt"):
        if k == "sa":
            text, *sa = v.split()
            assert oracle.sa_naive(enc(text)).tolist() == [int(x) for x in sa]
            assert brute_sa(text) == [int(x) for x in sa]
        elif k == "query":
            text, P, lo, hi = v.split()
            S = enc(text)
            want = (int(lo.split("=")[1]), int(hi.split("=")[1]))
            assert oracle.search(S, oracle.sa_naive(S), enc(P)) == want
        elif k == "batch":
            text, qs, flat = v.split()
            S = enc(text)
            words, lens = synth.pack_strings(qs.split(","))
            got = oracle.search_batch(S, oracle.sa_naive(S), words, lens)
            assert got.reshape(-1).tolist() == [int(x) for x in flat.split(",")]


def test_literal_alg1_is_wrong_and_corrected_reading_is_right():
    """Reading A4/A6: Alg. 1 read literally (L=0, R=n-1, `midSuffix <= query` moves R) loses the paper's own
    examples; the corrected loops reproduce them.  This pins the direction of the oracle's comparisons."""
    text = "acggtacgtac"
    S = enc(text)
    sa = oracle.sa_naive(S).tolist()

    def literal_lb(P):
        L, R = 0, len(text) - 1
        while R > L + 1:
            p = (L + R) >> 1
            t = text[sa[p]:sa[p] + len(P)]
            if t <= P:  # "if (midSuffix <= querySequence) R = pivot" read literally
                R = p
            else:
                L = p
        return R

    assert literal_lb("c") != 3  # literal reading gives a wrong LB for P=c (P:L161 says 3)
    assert oracle.search(S, np.array(sa, dtype=np.uint32), enc("c"))[0] == 3


# ---- brute force on tiny inputs --------------------------------------------------------------

@pytest.mark.parametrize("alphabet", ["acgt", "ac", "a"])
def test_sa_matches_python_sort(alphabet):
    rng = random.Random(17)
    for _ in range(150):
        n = rng.randint(1, 120)
        text = "".join(rng.choice(alphabet) for _ in range(n))
        assert oracle.sa_naive(enc(text)).tolist() == brute_sa(text)


def _queries_for(text, rng):
    n = len(text)
    qs = ["", text, text + "a", text[-1:] + "t"]
    for _ in range(40):
        i = rng.randrange(n)
        m = rng.randint(1, 12)
        qs.append(text[i:i + m])                                   # occurs (maybe cut at the end)
        qs.append(text[i:i + m] + rng.choice("acgt"))             # may run past the end
        qs.append("".join(rng.choice("acgt") for _ in range(m)))  # random
        j = rng.randrange(len(qs[-3]) or 1)
        s = qs[-3]
        if s:
            qs.append(s[:j] + rng.choice("acgt".replace(s[j], "")) + s[j + 1:])  # one substitution
    for j in range(1, 6):
        qs.append(text[n - j:])             # last j bases
        qs.append(text[n - j:] + "a")       # ... followed by one more base
    return qs


@pytest.mark.parametrize("alphabet", ["acgt", "ag", "a"])
def test_intervals_match_brute_force(alphabet):
    rng = random.Random(23)
    for _ in range(40):
        n = rng.randint(1, 90)
        text = "".join(rng.choice(alphabet) for _ in range(n))
        S = enc(text)
        sa = oracle.sa_naive(S)
        qs = _queries_for(text, rng)
        words, lens = synth.pack_strings(qs, stride=2)
        b_search = oracle.search_batch(S, sa, words, lens)
        b_count = oracle.count_batch(S, words, lens)
        for q, P in enumerate(qs):
            want = brute_lohi(text, P)
            assert oracle.search(S, sa, enc(P)) == want, (text, P)
            assert oracle.count(S, enc(P)) == want, (text, P)
            assert tuple(b_search[q]) == want and tuple(b_count[q]) == want, (text, P)
            # positions = occurrence set, listed in suffix order
            pos = oracle.locate(sa, *want).tolist()
            assert sorted(pos) == [i for i in range(n) if text.startswith(P, i)]
            assert pos == sorted(pos, key=lambda i: text[i:])


def test_cmp_cases_of_sec4():
    # P a prefix of S_i -> 0; P < S_i -> -1; P > S_i -> +1; S_i a proper prefix of P -> +1 (A7)
    S = enc("acggtacgtac")
    assert oracle.cmp(S, 4, enc("tac")) == 0
    assert oracle.cmp(S, 10, enc("c")) == 0
    assert oracle.cmp(S, 9, enc("ggtac")) == 1
    assert oracle.cmp(S, 2, enc("c")) == -1
    assert oracle.cmp(S, 9, enc("acg")) == 1   # suffix "ac" is a proper prefix of "acg"


# ---- closed forms ------------------------------------------------------------------------------

def test_closed_form_homopolymer():
    n = 500
    S = enc("a" * n)
    sa = oracle.sa_naive(S)
    assert sa.tolist() == list(range(n - 1, -1, -1))
    for k in [1, 2, 7, 499, 500, 501, 700]:
        want = (k - 1, n) if k <= n else (n, n)
        assert oracle.search(S, sa, enc("a" * k)) == want
    assert oracle.search(S, sa, enc("c")) == (n, n)
    assert oracle.search(S, sa, enc("")) == (0, n)


def de_bruijn(k, alphabet="acgt"):
    a = [0] * (len(alphabet) * k)
    seq = []

    def db(t, p):
        if t > k:
            if k % p == 0:
                seq.extend(a[1:p + 1])
        else:
            a[t] = a[t - p]
            db(t + 1, p)
            for j in range(a[t - p] + 1, len(alphabet)):
                a[t] = j
                db(t + 1, t)

    db(1, 1)
    s = "".join(alphabet[i] for i in seq)
    return s + s[:k - 1]  # linearised: every k-mer exactly once


@pytest.mark.parametrize("k", [3, 5])
def test_closed_form_de_bruijn(k):
    text = de_bruijn(k)
    assert len(text) == 4 ** k + k - 1
    S = enc(text)
    sa = oracle.sa_naive(S)
    kmers = ["".join(p) for p in itertools.product("acgt", repeat=k)]
    words, lens = synth.pack_strings(kmers)
    res = oracle.search_batch(S, sa, words, lens)
    assert np.all(res[:, 1] - res[:, 0] == 1)
    # and, being in lexicographic order, the k-mers tile the SA except the k-1 short suffixes
    assert np.all(np.diff(res[:, 0].astype(np.int64)) >= 1)


def test_kmer_counts_sum():
    rng = random.Random(5)
    text = "".join(rng.choice("acgt") for _ in range(3000))
    S = enc(text)
    sa = oracle.sa_naive(S)
    k = 4
    kmers = ["".join(p) for p in itertools.product("acgt", repeat=k)]
    words, lens = synth.pack_strings(kmers)
    res = oracle.search_batch(S, sa, words, lens).astype(np.int64)
    assert int((res[:, 1] - res[:, 0]).sum()) == len(text) - k + 1


# ---- k-mer table ------------------------------------------------------------------------------

@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_kmer_table_brute_force(k):
    rng = random.Random(k)
    for n in [1, 2, 3, 5, 17, 200]:
        text = "".join(rng.choice("acgt") for _ in range(n))
        S = enc(text)
        T = oracle.kmer_table(S, k)
        kmers = ["".join(p) for p in itertools.product("acgt", repeat=k)]
        want = [sum(1 for i in range(n) if text[i:i + k] < x) for x in kmers] + [n]
        assert T.tolist() == want
        assert np.all(np.diff(T.astype(np.int64)) >= 0)


# ---- checkers -----------------------------------------------------------------------------------

def test_check_sa_accepts_and_rejects():
    rng = random.Random(9)
    text = "".join(rng.choice("acgt") for _ in range(400))
    S = enc(text)
    sa = oracle.sa_naive(S)
    assert oracle.check_sa(S, sa) == -1
    for r in [0, 17, 398]:
        bad = sa.copy()
        bad[r], bad[r + 1] = bad[r + 1], bad[r]
        assert oracle.check_sa(S, bad) != -1
    dup = sa.copy()
    dup[5] = dup[6]
    assert oracle.check_sa(S, dup) != -1


def test_certificate_sound_against_perturbations():
    rng = random.Random(11)
    text = "".join(rng.choice("acg") for _ in range(300))
    S = enc(text)
    sa = oracle.sa_naive(S)
    qs = _queries_for(text, rng)
    words, lens = synth.pack_strings(qs, stride=2)
    good = oracle.search_batch(S, sa, words, lens).astype(np.uint32)
    assert oracle.certificate(S, sa, words, good, lens) == (0, -1)
    n = len(text)
    for q in range(len(qs)):
        for col in (0, 1):
            for d in (-1, 1):
                v = int(good[q, col]) + d
                if 0 <= v <= n:
                    bad = good.copy()
                    bad[q, col] = v
                    nbad, fb = oracle.certificate(S, sa, words, bad, lens)
                    assert nbad == 1 and fb == q, (qs[q], col, d)


def test_thread_invariance():
    rng = random.Random(3)
    text = "".join(rng.choice("acgt") for _ in range(5000))
    S = enc(text)
    sa = oracle.sa_naive(S)
    qs = _queries_for(text, rng)
    words, lens = synth.pack_strings(qs, stride=2)
    a = oracle.search_batch(S, sa, words, lens, nthreads=1)
    b = oracle.search_batch(S, sa, words, lens, nthreads=4)
    c = oracle.count_batch(S, words, lens, nthreads=3)
    assert np.array_equal(a, b) and np.array_equal(a, c)


def test_encode_rejects_non_acgt():
    assert oracle.encode("AcGt").tolist() == [0, 1, 2, 3]
    with pytest.raises(ValueError, match="position 3"):
        oracle.encode("ACGNT")
