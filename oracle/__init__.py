"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper over oracle/oracle.c (see its header for what is computed
and which PAPER.md passages each function follows).  Only tests/,
``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` leg / ``--impl
reference`` arm may import this package.  It shares no code with the CUDA
library in ``paper_1303_3692_b200/``.

Parity status: every function here is pinned by tests in
tests/test_oracle_pins.py (paper worked examples, brute force, closed forms,
invariants); DESIGN.md "Oracle pins" lists which pin covers which function.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_u32 = ctypes.c_uint32
_int = ctypes.c_int


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `make` (or __graft_entry__.build())")
        lib = ctypes.CDLL(_LIB_PATH)
        sig = {
            "oracle_max_threads": ([], _int),
            "oracle_encode": ([_p, _i64, _p], _i64),
            "oracle_sa_naive": ([_p, _i64, _p], None),
            "oracle_cmp": ([_p, _i64, _i64, _p, _i64], _int),
            "oracle_search": ([_p, _i64, _p, _p, _i64, _p, _p], None),
            "oracle_count": ([_p, _i64, _p, _i64, _p, _p], None),
            "oracle_search_batch": ([_p, _i64, _p, _p, _u32, _p, _u32, _i64, _p, _int], _int),
            "oracle_count_batch": ([_p, _i64, _p, _u32, _p, _u32, _i64, _p, _int], _int),
            "oracle_check_sa": ([_p, _i64, _p, _int], _i64),
            "oracle_certificate": ([_p, _i64, _p, _p, _u32, _p, _u32, _i64, _p, _p, _int], _i64),
            "oracle_kmer_table": ([_p, _i64, _int, _p], None),
        }
        for name, (args, res) in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = res
        _lib = lib
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def max_threads() -> int:
    return _load().oracle_max_threads()


def encode(text) -> np.ndarray:
    """ASCII (str / bytes / uint8 array) -> codes a=0 c=1 g=2 t=3; ValueError with the position of a bad byte."""
    if isinstance(text, str):
        text = text.encode("ascii")
    a = np.frombuffer(text, dtype=np.uint8) if isinstance(text, (bytes, bytearray)) else np.ascontiguousarray(text, dtype=np.uint8)
    out = np.empty(a.size, dtype=np.uint8)
    bad = _load().oracle_encode(_ptr(a), a.size, _ptr(out))
    if bad >= 0:
        raise ValueError(f"non-ACGT symbol {chr(a[bad])!r} at position {bad}")
    return out


def sa_naive(S: np.ndarray) -> np.ndarray:
    S = np.ascontiguousarray(S, dtype=np.uint8)
    sa = np.empty(S.size, dtype=np.uint32)
    _load().oracle_sa_naive(_ptr(S), S.size, _ptr(sa))
    return sa


def cmp(S: np.ndarray, s: int, P: np.ndarray) -> int:
    P = np.ascontiguousarray(P, dtype=np.uint8)
    return _load().oracle_cmp(_ptr(S), S.size, s, _ptr(P), P.size)


def search(S: np.ndarray, sa: np.ndarray, P: np.ndarray):
    P = np.ascontiguousarray(P, dtype=np.uint8)
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    _load().oracle_search(_ptr(S), S.size, _ptr(sa), _ptr(P), P.size, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


def count(S: np.ndarray, P: np.ndarray):
    P = np.ascontiguousarray(P, dtype=np.uint8)
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    _load().oracle_count(_ptr(S), S.size, _ptr(P), P.size, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


def _qargs(words, lens, fixed_len):
    words = np.ascontiguousarray(words, dtype=np.uint64)
    if words.ndim == 1:
        words = words.reshape(-1, 1)
    lens = None if lens is None else np.ascontiguousarray(lens, dtype=np.uint32)
    return words, words.shape[1], lens, (0 if fixed_len is None else int(fixed_len))


def search_batch(S, sa, words, lens=None, fixed_len=None, nthreads=0) -> np.ndarray:
    """Textbook binary search for every packed query -> uint64 [Q, 2] (lo, hi)."""
    words, stride, lens, fixed = _qargs(words, lens, fixed_len)
    Q = words.shape[0]
    out = np.empty((Q, 2), dtype=np.uint64)
    rc = _load().oracle_search_batch(_ptr(S), S.size, _ptr(sa), _ptr(words), stride, _ptr(lens), fixed, Q,
                                     _ptr(out), nthreads)
    if rc != 0:
        raise MemoryError("oracle_search_batch")
    return out


def count_batch(S, words, lens=None, fixed_len=None, nthreads=0) -> np.ndarray:
    """Streaming counting oracle (no suffix array) -> uint64 [Q, 2] (lo, hi)."""
    words, stride, lens, fixed = _qargs(words, lens, fixed_len)
    Q = words.shape[0]
    out = np.empty((Q, 2), dtype=np.uint64)
    rc = _load().oracle_count_batch(_ptr(S), S.size, _ptr(words), stride, _ptr(lens), fixed, Q, _ptr(out), nthreads)
    if rc != 0:
        raise MemoryError("oracle_count_batch")
    return out


def check_sa(S, sa, nthreads=0) -> int:
    """-1 if sa is the suffix array of S, else the first bad index found."""
    sa = np.ascontiguousarray(sa, dtype=np.uint32)
    if sa.size != S.size:
        return 0
    return _load().oracle_check_sa(_ptr(S), S.size, _ptr(sa), nthreads)


def certificate(S, sa, words, lohi, lens=None, fixed_len=None, nthreads=0):
    """(number of failing queries, first failing query or -1) for uint32 [Q, 2] intervals."""
    words, stride, lens, fixed = _qargs(words, lens, fixed_len)
    lohi = np.ascontiguousarray(lohi, dtype=np.uint32)
    Q = words.shape[0]
    fb = ctypes.c_int64()
    nbad = _load().oracle_certificate(_ptr(S), S.size, _ptr(sa), _ptr(words), stride, _ptr(lens), fixed, Q,
                                      _ptr(lohi), ctypes.byref(fb), nthreads)
    return nbad, fb.value


def kmer_table(S, k: int) -> np.ndarray:
    """T[x] = #{i : trunc_k(S_i) < x}, x in [0, 4^k]."""
    T = np.empty((1 << (2 * k)) + 1, dtype=np.uint32)
    _load().oracle_kmer_table(_ptr(S), S.size, k, _ptr(T))
    return T


def locate(sa: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """Positions of an interval in SA order (P=a -> 9, 0, 5)."""
    return np.asarray(sa[lo:hi])


def rank_array(sa: np.ndarray) -> np.ndarray:
    """1-based rank of every suffix, i.e. inverse SA + 1 (Table III)."""
    r = np.empty(sa.size, dtype=np.int64)
    r[sa.astype(np.int64)] = np.arange(1, sa.size + 1)
    return r
