"""the paper's DC3 suffix-array construction on the GPU (SA_INDEX_BUILD_DC3),
pinned to PAPER.md's worked example (Table II sample ranks, the non-sample order of step 2, Table I)
and checked against the oracle's comparison-sort SA and the default prefix-doubling build."""
import os
import random

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
import paper_1303_3692_b200 as sa  # noqa: E402

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = {}
    for line in open(os.path.join(GOLDEN, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            k, v = line.split(":", 1)
            rows[k.strip()] = v.strip()
    return rows


def test_dc3_trace_reproduces_table2_and_step2():
    g = _golden("paper_table2_dc3.txt")
    rank, b0 = sa.dc3_trace(g["text"])
    want = dict((int(a), int(b)) for a, b in (t.split(":") for t in g["sample_rank"].split()))
    assert {i: int(r) for i, r in enumerate(rank) if r} == want          # Table II
    assert b0.tolist() == [int(x) for x in g["nonsample_order"].split()]  # S9 <= S0 <= S6 <= S3


def test_dc3_table1():
    idx = sa.Index("acggtacgtac", build="dc3")
    assert idx.export_sa().tolist() == [9, 0, 5, 10, 1, 6, 2, 7, 3, 8, 4]   # Table I


@pytest.mark.parametrize("alphabet", ["ACGT", "AC", "A"])
def test_dc3_random_texts_all_lengths_mod3(alphabet):
    rng = random.Random(len(alphabet))
    for n in list(range(1, 40)) + [64, 65, 66, 1000, 4097, 20000]:
        text = "".join(rng.choice(alphabet) for _ in range(n))
        got = sa.Index(text, build="dc3", layout="plain").export_sa()
        assert np.array_equal(got, oracle.sa_naive(oracle.encode(text))), (alphabet, n)


@pytest.mark.parametrize("text", ["A" * 30000, "AC" * 20000 + "A", "ACGTTGCA" * 5000, "T" * 777 + "A" * 333])
def test_dc3_deep_recursion(text):
    got = sa.Index(text, build="dc3", layout="plain").export_sa()
    assert np.array_equal(got, oracle.sa_naive(oracle.encode(text)))


def test_dc3_repeat_rich_and_search_parity():
    ref = synth.reference(synth.REF_REPEAT, 3_000_000, 71)
    a = sa.Index(ref, build="dc3")
    b = sa.Index(ref)  # prefix doubling
    assert np.array_equal(a.export_sa(), b.export_sa())
    assert np.array_equal(a.export_sa(), oracle.sa_naive(oracle.encode(ref)))
    words, lens = synth.reads(ref, 50_000, 20, 120, 0.1, 0.0, 72)
    w = torch.from_numpy(words.view(np.int64)).cuda()
    l = torch.from_numpy(lens.view(np.int32)).cuda()
    assert torch.equal(a.match(w, l), b.match(w, l))


@pytest.mark.slow
def test_dc3_equals_doubling_c3():
    ref = synth.CONFIGS["C3"].reference()
    a = sa.Index(ref, build="dc3", layout="plain").export_sa()
    b = sa.Index(ref, layout="plain").export_sa()
    assert np.array_equal(a, b)
