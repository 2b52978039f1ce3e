"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds no part of the method's arithmetic (see synth.c's header):
it produces reference bytes and packed reads only.  The recipes for the five
BASELINE.json configurations are stated in DESIGN.md ("Input recipe") and are
collected in ``CONFIGS`` below.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynth.so")
_lib = None

REF_UNIFORM, REF_BACTERIAL, REF_REPEAT, REF_REPEAT_DUP = 0, 1, 2, 3


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(_LIB_PATH)
        lib.synth_reference.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int]
        lib.synth_reference.restype = ctypes.c_int
        lib.synth_reads.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_uint32, ctypes.c_uint32, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p,
                                    ctypes.c_int]
        lib.synth_reads.restype = ctypes.c_int
        _lib = lib
    return _lib


def reference(kind: int, n: int, seed: int, nthreads: int = 0) -> np.ndarray:
    """n upper-case ACGT bytes (numpy uint8)."""
    out = np.empty(n, dtype=np.uint8)
    rc = _load().synth_reference(kind, n, seed, out.ctypes.data, nthreads)
    if rc != 0:
        raise RuntimeError(f"synth_reference failed ({rc})")
    return out


def stride_for(m_max: int) -> int:
    return max(1, (m_max + 31) // 32)


def reads(ref: np.ndarray, q_count: int, m_min: int, m_max: int, p_random: float, p_mut_read: float,
          seed: int, q_begin: int = 0, stride: Optional[int] = None, nthreads: int = 0,
          words_out: Optional[np.ndarray] = None, lens_out: Optional[np.ndarray] = None, dense: bool = False):
    """Reads q_begin..q_begin+q_count-1: (words uint64[q_count, stride], lens uint32[q_count]).

    dense=True (fixed length m only, q_count % 32 == 0): words is one continuous 2-bit stream of
    q_count*m/32 words (include/sa.h "dense layout", stride_words = 0)."""
    if dense:
        assert m_min == m_max and q_count % 32 == 0
        stride = 0
        nwords = q_count // 32 * m_max
        words = words_out if words_out is not None else np.empty(nwords, dtype=np.uint64)
        assert words.dtype == np.uint64 and words.flags.c_contiguous and words.size >= nwords
    else:
        stride = stride or stride_for(m_max)
        words = words_out if words_out is not None else np.empty((q_count, stride), dtype=np.uint64)
        assert words.dtype == np.uint64 and words.flags.c_contiguous and words.size >= q_count * stride
    lens = lens_out if lens_out is not None else np.empty(q_count, dtype=np.uint32)
    assert lens.dtype == np.uint32 and lens.size >= q_count
    ref = np.ascontiguousarray(ref, dtype=np.uint8)
    rc = _load().synth_reads(ref.ctypes.data if ref.size else None, ref.size, q_begin, q_count, m_min, m_max,
                             p_random, p_mut_read, seed, words.ctypes.data, stride, lens.ctypes.data, nthreads)
    if rc != 0:
        raise RuntimeError(f"synth_reads failed ({rc})")
    return words, lens


_CODE = {"A": 0, "C": 1, "G": 2, "T": 3}


def pack_strings(seqs: Sequence[str], stride: Optional[int] = None):
    """Pack hand-written reads (tests, examples) into the include/sa.h layout."""
    m_max = max((len(s) for s in seqs), default=0)
    stride = max(stride or 0, stride_for(m_max))
    words = np.zeros((len(seqs), stride), dtype=np.uint64)
    lens = np.zeros(len(seqs), dtype=np.uint32)
    for q, s in enumerate(seqs):
        s = s.upper()
        lens[q] = len(s)
        for j, ch in enumerate(s):
            words[q, j >> 5] |= np.uint64(_CODE[ch]) << np.uint64(62 - 2 * (j & 31))
    return words, lens


def pack_dense(seqs: Sequence[str]) -> np.ndarray:
    """Pack equal-length reads into the dense layout (one 2-bit stream, read i at bases [i*m, (i+1)*m))."""
    m = len(seqs[0]) if seqs else 0
    assert all(len(x) == m for x in seqs)
    nbases = m * len(seqs)
    words = np.zeros(max(1, (nbases + 31) // 32), dtype=np.uint64)
    for i, x in enumerate(seqs):
        for j, ch in enumerate(x.upper()):
            b = i * m + j
            words[b >> 5] |= np.uint64(_CODE[ch]) << np.uint64(62 - 2 * (b & 31))
    return words


def unpack_read(words_row: np.ndarray, m: int) -> str:
    out = []
    for j in range(m):
        c = (int(words_row[j >> 5]) >> (62 - 2 * (j & 31))) & 3
        out.append("ACGT"[c])
    return "".join(out)


@dataclass(frozen=True)
class Config:
    name: str
    ref_kind: int
    n: int
    ref_seed: int
    Q: int
    m_min: int
    m_max: int
    p_random: float
    p_mut_read: float
    read_seed: int
    description: str = ""
    sweep: tuple = field(default_factory=tuple)

    @property
    def stride(self) -> int:
        return stride_for(self.m_max)

    def reference(self, nthreads: int = 0) -> np.ndarray:
        return reference(self.ref_kind, self.n, self.ref_seed, nthreads)

    def reads(self, ref, q_begin=0, q_count=None, nthreads=0, **kw):
        q_count = self.Q if q_count is None else q_count
        return reads(ref, q_count, self.m_min, self.m_max, self.p_random, self.p_mut_read, self.read_seed,
                     q_begin=q_begin, nthreads=nthreads, **kw)

    def with_m(self, m: int) -> "Config":
        """C5: the read-length sweep point m (seed 5000+m)."""
        return Config(f"{self.name}-m{m}", self.ref_kind, self.n, self.ref_seed, self.Q, m, m, self.p_random,
                      self.p_mut_read, 5000 + m, self.description)


# BASELINE.json configs[0..4]; recipes in DESIGN.md "Input recipe".
CONFIGS = {
    "C1": Config("C1", REF_UNIFORM, 1_000_000, 1, 11_000, 32, 32, 1.0 / 11.0, 0.0, 1,
                 "1 Mbp iid ACGT, 10k exact 32-bp reads + 10% random reads"),
    "C2": Config("C2", REF_BACTERIAL, 5_000_000, 2, 1_000_000, 25, 100, 0.0, 0.01, 2,
                 "5 Mbp E. coli-like, 1M reads of 25-100 bp, 1% of reads with one substitution"),
    "C3": Config("C3", REF_REPEAT_DUP, 100_000_000, 3, 10_000_000, 100, 100, 0.10, 0.0, 3,
                 "100 Mbp repeat-rich (+ one exact 100 kb duplication), 10M 100-bp reads (90% sampled, 10% random)"),
    "C4": Config("C4", REF_REPEAT, 3_100_000_000, 4, 100_000_000, 100, 100, 0.10, 0.0, 4,
                 "3.1 Gbp human-scale repeat-rich, 100M 100-bp reads (90% sampled, 10% random)"),
    "C5": Config("C5", REF_REPEAT, 3_100_000_000, 4, 50_000_000, 100, 100, 0.10, 0.0, 5100,
                 "read-length sweep 16-1000 bp, 50M reads per length, on the C4 reference",
                 sweep=(16, 32, 64, 100, 150, 250, 500, 1000)),
}
