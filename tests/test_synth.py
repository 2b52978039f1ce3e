"""The seeded input generators (synth/): determinism, thread and shard invariance, recipe properties."""
import numpy as np

import synth


def test_reference_deterministic_and_thread_invariant():
    for kind in (synth.REF_UNIFORM, synth.REF_BACTERIAL, synth.REF_REPEAT):
        a = synth.reference(kind, 300_000, 7, nthreads=1)
        b = synth.reference(kind, 300_000, 7, nthreads=4)
        c = synth.reference(kind, 300_000, 8, nthreads=4)
        assert np.array_equal(a, b)
        assert not np.array_equal(a, c)
        assert set(np.unique(a).tobytes()) <= set(b"ACGT")


def test_reads_shard_invariant_and_packed():
    ref = synth.reference(synth.REF_UNIFORM, 100_000, 3)
    w, l = synth.reads(ref, 5000, 25, 100, 0.1, 0.01, 11, nthreads=4)
    w2, l2 = synth.reads(ref, 2000, 25, 100, 0.1, 0.01, 11, q_begin=1500, nthreads=1)
    assert np.array_equal(w[1500:3500], w2) and np.array_equal(l[1500:3500], l2)
    assert l.min() >= 25 and l.max() <= 100 and w.shape[1] == 4
    # bits past each read's length are zero
    for q in range(200):
        m = int(l[q])
        for j in range(m, 128):
            assert (int(w[q, j >> 5]) >> (62 - 2 * (j & 31))) & 3 == 0


def test_exact_reads_occur_and_random_fraction():
    ref = synth.reference(synth.REF_UNIFORM, 50_000, 5)
    text = ref.tobytes().decode()
    w, l = synth.reads(ref, 2000, 32, 32, 0.25, 0.0, 9)
    hits = sum(synth.unpack_read(w[q], int(l[q])) in text for q in range(2000))
    # 75% are exact copies; a random 32-mer essentially never occurs in 50 kb
    assert abs(hits / 2000 - 0.75) < 0.05


def test_config_recipes_shape():
    c1 = synth.CONFIGS["C1"]
    assert (c1.n, c1.Q, c1.m_min, c1.m_max) == (1_000_000, 11_000, 32, 32)
    c4 = synth.CONFIGS["C4"]
    assert (c4.n, c4.Q, c4.m_max, c4.stride) == (3_100_000_000, 100_000_000, 100, 4)
    assert synth.CONFIGS["C5"].with_m(1000).stride == 32


def test_repeat_reference_has_repeats():
    ref = synth.reference(synth.REF_REPEAT, 2_000_000, 3)
    # the repeat-rich recipe must produce many more repeated 20-mers than an iid text of the same size
    def dup20(r):
        t = r.tobytes()
        seen, d = set(), 0
        for i in range(0, len(t) - 20, 7):
            k = t[i:i + 20]
            d += k in seen
            seen.add(k)
        return d
    iid = synth.reference(synth.REF_UNIFORM, 2_000_000, 3)
    assert dup20(ref) > 50 * max(1, dup20(iid))


def test_dense_layout_equals_packed_strings():
    ref = synth.reference(synth.REF_UNIFORM, 50_000, 2)
    for m in (7, 32, 100):
        w, l = synth.reads(ref, 96, m, m, 0.2, 0.0, 3)
        d1, _ = synth.reads(ref, 96, m, m, 0.2, 0.0, 3, dense=True, nthreads=1)
        d4, _ = synth.reads(ref, 96, m, m, 0.2, 0.0, 3, dense=True, nthreads=4)
        want = synth.pack_dense([synth.unpack_read(w[i], m) for i in range(96)])
        assert np.array_equal(d1, want[: d1.size]) and np.array_equal(d1, d4)


def test_repeat_dup_has_one_exact_100kb_duplication():
    # C3's recipe: the repeat-rich generator plus one exact 100 kb copy (reading B3)
    n = 1_000_000
    a = synth.reference(synth.REF_REPEAT, n, 3)
    b = synth.reference(synth.REF_REPEAT_DUP, n, 3)
    s, d, L = n // 4, 5 * (n // 8), 100_000
    assert np.array_equal(b[d:d + L], b[s:s + L]) and np.array_equal(b[s:s + L], a[s:s + L])
    assert np.array_equal(np.delete(b, np.s_[d:d + L]), np.delete(a, np.s_[d:d + L]))
    assert synth.CONFIGS["C3"].ref_kind == synth.REF_REPEAT_DUP
