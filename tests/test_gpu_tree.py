"""the flattened suffix tree (sa_tree_*) must give every read exactly the SA
search's interval (and the oracle's), misses included."""
import itertools
import random

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
import paper_1303_3692_b200 as sa  # noqa: E402
from test_gpu_parity import hazard_queries  # noqa: E402

pytestmark = pytest.mark.gpu


def _cuda(words, lens):
    return (torch.from_numpy(np.ascontiguousarray(words).view(np.int64)).cuda(),
            torch.from_numpy(np.ascontiguousarray(lens).view(np.int32)).cuda())


def check_tree(text, words, lens, layout="rec16"):
    idx = sa.Index(text, layout=layout)
    tree = sa.Tree(idx)
    w, l = _cuda(words, lens)
    got = tree.match(w, l).cpu().numpy().view(np.uint32)
    S = oracle.encode(text)
    want = oracle.search_batch(S, oracle.sa_naive(S), words, lens).astype(np.uint32)
    bad = np.nonzero((got != want).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first {bad[0]}: got {got[bad[0]]} want {want[bad[0]]}"
    perm = idx.order(w, l)
    assert np.array_equal(tree.match(w, l, order=perm).cpu().numpy().view(np.uint32), want)
    return tree


def test_tree_paper_example():
    words, lens = synth.pack_strings(["a", "c", "ggtac", "tac", "tt", "gg", "acggtacgtac", "", "acgt", "t"])
    tree = check_tree("acggtacgtac", words, lens)
    assert tree.nodes >= 1


@pytest.mark.parametrize("layout", ["rec16", "rec32", "plain"])
@pytest.mark.parametrize("n", [1, 2, 3, 7, 31, 64, 65, 1000, 5000])
def test_tree_random_texts(n, layout):
    rng = random.Random(n)
    for alphabet in ("ACGT", "AC", "A"):
        text = "".join(rng.choice(alphabet) for _ in range(n))
        words, lens = synth.pack_strings(hazard_queries(text, 8, rng, extra=100))
        check_tree(text, words, lens, layout)


def test_tree_all_kmers_de_bruijn_like():
    rng = random.Random(3)
    text = "".join(rng.choice("ACGT") for _ in range(3000))
    qs = ["".join(p) for m in range(1, 5) for p in itertools.product("ACGT", repeat=m)]
    words, lens = synth.pack_strings(qs)
    check_tree(text, words, lens)


def test_tree_c2_and_repeat_rich():
    c = synth.CONFIGS["C2"]
    ref = c.reference()
    words, lens = c.reads(ref, q_count=200_000)
    check_tree(ref.tobytes(), words, lens)
    ref = synth.reference(synth.REF_REPEAT, 2_000_000, 81)
    words, lens = synth.reads(ref, 200_000, 16, 200, 0.1, 0.01, 82)
    check_tree(ref.tobytes(), words, lens, layout="rec32")
