"""paper_1303_3692_b200 -- B200-native suffix-array exact matching (arXiv 1303.3692's hot path).

A thin ctypes binding over the C ABI in ``include/sa.h`` (``libsa.so``, built in-tree by
``make``).  The binding only marshals arguments: every step of the path (pack, suffix-array
build, bracket table, search, locate) runs in the library's CUDA kernels.  PyTorch is used for
device memory and streams.  There is no CPU fallback: if ``libsa.so`` is missing or no CUDA
device is present, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np

__all__ = ["SAError", "Index", "Tree", "lib", "random_gather", "dc3_trace", "LIB_PATH", "EXPORTED_SYMBOLS"]

_HERE = os.path.dirname(os.path.abspath(__file__))
# SA_LIB_PATH selects another build of the same library (A/B measurements of build variants)
LIB_PATH = os.environ.get("SA_LIB_PATH") or os.path.join(_HERE, "libsa.so")

SA_OK, SA_EINVAL, SA_ESYMBOL, SA_ETOOLONG, SA_ENOMEM, SA_ECUDA, SA_EEMPTY = 0, -1, -2, -3, -4, -5, -6
SA_INDEX_PLAIN = 1          # sa_index_opts.flags: plain uint32 SA instead of 16-byte records
SA_INDEX_REC32 = 2          # sa_index_opts.flags: 32-byte records caching 112 bases
SA_MATCH_STATS = 1          # sa_match_batch flags: per-query steps | text windows << 16 into the workspace
SA_MATCH_PRESORT = 4        # sa_match_batch flags: order reads by their first 12 bases before the search
SA_MATCH_ROWS_ORDERED = 8   # sa_match_batch flags: rows already arranged in `order` order
SA_MATCH_COOPERATIVE = 32   # sa_match_batch flags: reads over 128 bases searched by 8/16/32-lane groups
SA_MATCH_SMEM_TREE = 64     # sa_match_batch flags: shared-memory top tree per CTA (needs an order)
SA_ORDER_BUCKETS = 0x100    # sa_match_order key_bases flag: bucket placement (not stable), for L2-sized batches
SA_MATCH_DEFER = 1 << 17    # sa_match_batch flags: reads in big k-mer buckets deferred to a second full-warp pass
SA_MATCH_WIDE = 1 << 24     # sa_match_batch flags: the large-batch load hints at any batch size
SA_INDEX_BUILD_DC3 = 4      # sa_index_opts.flags: build the SA with DC3 (the paper's algorithm)
SA_INDEX_SUBTABLE = 8       # sa_index_opts.flags: (k+4)-base sub-tables for buckets of > 32 suffixes
SA_INDEX_BUCKET_TREE = 16   # sa_index_opts.flags: line-packed binary-search trees for buckets of >= 32 suffixes
LAYOUTS = {"rec16": 0, "rec32": SA_INDEX_REC32, "plain": SA_INDEX_PLAIN}
_NAMES = {0: "SA_OK", -1: "SA_EINVAL", -2: "SA_ESYMBOL", -3: "SA_ETOOLONG", -4: "SA_ENOMEM", -5: "SA_ECUDA",
          -6: "SA_EEMPTY"}

_p, _u64, _u32, _i32, _sz = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32, ctypes.c_size_t


class _Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("kmer_k", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32)]


# name -> (argtypes, restype); mirrors include/sa.h
_SIGS = {
    "sa_index_create": ([_p, _u64, ctypes.POINTER(_Opts), ctypes.POINTER(_p)], ctypes.c_int),
    "sa_index_destroy": ([_p], None),
    "sa_index_info": ([_p, ctypes.POINTER(_u64), ctypes.POINTER(_u32), ctypes.POINTER(_u64), ctypes.POINTER(_i32)],
                      ctypes.c_int),
    "sa_index_export_sa": ([_p, _p], ctypes.c_int),
    "sa_index_export_table": ([_p, _p], ctypes.c_int),
    "sa_index_export_text": ([_p, _p], ctypes.c_int),
    "sa_match_workspace_size": ([_p, _u64, _u32, _u32, ctypes.POINTER(_sz)], ctypes.c_int),
    "sa_match_batch": ([_p, _p, _p, _u32, _u32, _u64, _p, _p, _p, _sz, _u32, _p], ctypes.c_int),
    "sa_match_order_workspace_size": ([_u64, ctypes.POINTER(_sz)], ctypes.c_int),
    "sa_match_order_workspace_size_ex": ([_u64, _u32, ctypes.POINTER(_sz)], ctypes.c_int),
    "sa_match_order": ([_p, _p, _p, _u32, _u32, _u64, _u32, _p, _p, _p, _p, _sz, _p], ctypes.c_int),
    "sa_match_batch_host": ([_p, _p, _p, _u32, _u32, _u64, _p, _u64], ctypes.c_int),
    "sa_locate_workspace_size": ([_u64, ctypes.POINTER(_sz)], ctypes.c_int),
    "sa_locate_offsets": ([_p, _p, _u64, _p, _p, _sz, _p], ctypes.c_int),
    "sa_locate": ([_p, _p, _p, _u64, _p, _p], ctypes.c_int),
    "sa_tool_random_gather": ([_i32, _u64, _u32, _u64, _u32, _i32, ctypes.POINTER(ctypes.c_float)], ctypes.c_int),
    "sa_dc3_trace": ([_p, _u64, _p, _p], ctypes.c_int),
    "sa_index_create_part": ([_p, _u64, ctypes.POINTER(_Opts), _u32, _u32, _u32, ctypes.POINTER(_p)], ctypes.c_int),
    "sa_index_part_info": ([_p, ctypes.POINTER(_u32), ctypes.POINTER(_u32), ctypes.POINTER(_u32),
                            ctypes.POINTER(_u64), ctypes.POINTER(_u64), _p, _p], ctypes.c_int),
    "sa_match_route": ([_p, _p, _p, _u32, _u32, _u64, _p, _p, _p, _p, _p, _sz, _p], ctypes.c_int),
    "sa_part_pack": ([_p, _p, _p, _u32, _p, _u64, _u64, _p, _p, _p], ctypes.c_int),
    "sa_part_collect": ([_p, _p, _p, _u64, _p, _p, _p], ctypes.c_int),
    "sa_scatter_results": ([_p, _p, _u64, _p, _p], ctypes.c_int),
    "sa_tree_create": ([_p, ctypes.POINTER(_p)], ctypes.c_int),
    "sa_tree_destroy": ([_p], None),
    "sa_tree_info": ([_p, ctypes.POINTER(_u64), ctypes.POINTER(_u64)], ctypes.c_int),
    "sa_tree_match": ([_p, _p, _p, _u32, _u32, _u64, _p, _p, _p], ctypes.c_int),
    "sa_last_error": ([], ctypes.c_char_p),
    "sa_version": ([], ctypes.c_int32),
}
EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def lib():
    """Load libsa.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `make` or __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


class SAError(RuntimeError):
    def __init__(self, code: int, where: str):
        detail = lib().sa_last_error().decode(errors="replace")
        super().__init__(f"{where}: {_NAMES.get(code, code)}: {detail}")
        self.code = code
        self.detail = detail


def _check(code: int, where: str):
    if code != SA_OK:
        raise SAError(code, where)


def _stream_ptr(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream or None


def _empty(shape, dtype, device, stream=None):
    """torch.empty on `stream` when one is given: the caching allocator then ties the block to the stream
    the library works on, so a transient freed on return is not handed out again while that stream's
    kernels still use it."""
    import torch
    if stream is None:
        return torch.empty(shape, dtype=dtype, device=device)
    with torch.cuda.stream(stream):
        return torch.empty(shape, dtype=dtype, device=device)


def _dptr(t) -> Optional[int]:
    return None if t is None else (t.data_ptr() or None)


def _rows(words, n_reads):
    """(Q, stride_words): a 2-D [Q, stride] array is the strided layout; a 1-D stream with
    n_reads given is the dense layout (stride_words = 0)."""
    if n_reads is not None:
        assert words.dim() == 1 if hasattr(words, "dim") else words.ndim == 1
        return int(n_reads), 0
    return int(words.shape[0]), int(words.shape[1])


class Index:
    """Suffix-array index of one reference on one GPU (``sa_index_create``).

    ref: str / bytes / numpy uint8 array of ACGT (case-insensitive).  k: bracket-table k (0 = auto).
    layout: "rec16" (default, 16-byte records caching 48 bases), "rec32" (32-byte records, 112 bases)
    or "plain" (uint32 SA; every step reads the packed text).
    build: "doubling" (default, prefix doubling) or "dc3" (the paper's DC3, SA_INDEX_BUILD_DC3).
    """

    def __init__(self, ref, k: int = 0, device: Optional[int] = None, layout: str = "rec16", build: str = "doubling",
                 part: Optional[Tuple[int, int, int]] = None, subtables: bool = False, bucket_tree: bool = False):
        if isinstance(ref, str):
            ref = ref.encode("ascii")
        arr = np.frombuffer(ref, dtype=np.uint8) if isinstance(ref, (bytes, bytearray)) else \
            np.ascontiguousarray(ref, dtype=np.uint8)
        if build not in ("doubling", "dc3"):
            raise ValueError("build must be 'doubling' or 'dc3'")
        flags = LAYOUTS[layout] | (SA_INDEX_BUILD_DC3 if build == "dc3" else 0) | (SA_INDEX_SUBTABLE if subtables else 0) | \
            (SA_INDEX_BUCKET_TREE if bucket_tree else 0)
        opts = _Opts(-1 if device is None else int(device), int(k), flags, 0)
        self.layout = layout
        h = _p()
        ptr = arr.ctypes.data if arr.size else None
        if part is None:
            _check(lib().sa_index_create(ptr, arr.size, ctypes.byref(opts), ctypes.byref(h)), "sa_index_create")
        else:  # (part, nparts, route_bases): a partition of the index
            _check(lib().sa_index_create_part(ptr, arr.size, ctypes.byref(opts), int(part[0]), int(part[1]),
                                              int(part[2]), ctypes.byref(h)), "sa_index_create_part")
        self._h = h
        self._part = part is not None
        n, kk, nb, dev = _u64(), _u32(), _u64(), _i32()
        _check(lib().sa_index_info(h, ctypes.byref(n), ctypes.byref(kk), ctypes.byref(nb), ctypes.byref(dev)),
               "sa_index_info")
        self.n, self.k, self.device_bytes, self.device = n.value, kk.value, nb.value, dev.value

    def part_info(self) -> dict:
        p, np_, rb, lo, hi = _u32(), _u32(), _u32(), _u64(), _u64()
        _check(lib().sa_index_part_info(self._h, ctypes.byref(p), ctypes.byref(np_), ctypes.byref(rb),
                                        ctypes.byref(lo), ctypes.byref(hi), None, None), "sa_index_part_info")
        keys = np.empty(np_.value + 1, dtype=np.uint32)
        ranks = np.empty(np_.value + 1, dtype=np.uint64)
        _check(lib().sa_index_part_info(self._h, None, None, None, None, None, keys.ctypes.data, ranks.ctypes.data),
               "sa_index_part_info")
        return {"part": p.value, "nparts": np_.value, "route_bases": rb.value, "rank_lo": lo.value,
                "rank_hi": hi.value, "part_keys": keys.tolist(), "part_ranks": ranks.tolist()}

    def route(self, words, lens=None, fixed_len: Optional[int] = None, stream=None):
        """sa_match_route: (order int32[Q], ordered words, ordered lens or None, dest offsets int64[nparts+1]);
        ordered rows [offs[g], offs[g+1]) go to part g, rows [offs[nparts], Q) (reads shorter than the route key)
        to every part."""
        import torch
        Q, stride = words.shape
        need = _sz()
        _check(lib().sa_match_order_workspace_size(Q, ctypes.byref(need)), "sa_match_order_workspace_size")
        ws = _empty(max(1, need.value), torch.uint8, words.device, stream)
        order = _empty(Q, torch.int32, words.device, stream)
        ow = _empty(tuple(words.shape), words.dtype, words.device, stream)
        ol = None if lens is None else _empty(tuple(lens.shape), lens.dtype, lens.device, stream)
        nparts = self.part_info()["nparts"]
        offs = _empty(nparts + 1, torch.int64, words.device, stream)
        _check(lib().sa_match_route(self._h, _dptr(words), _dptr(lens), int(fixed_len or 0), stride, Q, _dptr(order),
                                    _dptr(ow), _dptr(ol), _dptr(offs), _dptr(ws), need.value, _stream_ptr(stream)),
               "sa_match_route")
        return order, ow, ol, offs

    def part_pack(self, ordered_words, ordered_lens, offs, send_rows: int, stream=None):
        """sa_part_pack: the all-to-all send buffer (block g = rows routed to part g + all short rows)."""
        import torch
        Q, stride = ordered_words.shape
        sw = _empty((send_rows, stride), ordered_words.dtype, ordered_words.device, stream)
        sl = None if ordered_lens is None else _empty(send_rows, ordered_lens.dtype, ordered_lens.device, stream)
        _check(lib().sa_part_pack(self._h, _dptr(ordered_words), _dptr(ordered_lens), stride, _dptr(offs), Q, send_rows,
                                  _dptr(sw), _dptr(sl), _stream_ptr(stream)), "sa_part_pack")
        return sw, sl

    def part_collect(self, back, offs, order, Q: int, out=None, stream=None):
        """sa_part_collect: every read's global interval from the parts' answers, at the read's own index."""
        import torch
        if out is None:
            out = _empty((Q, 2), torch.int32, back.device, stream)
        _check(lib().sa_part_collect(self._h, _dptr(back), _dptr(offs), Q, _dptr(order), _dptr(out),
                                     _stream_ptr(stream)), "sa_part_collect")
        return out

    # ---- lifetime ----
    def close(self):
        if getattr(self, "_h", None):
            lib().sa_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- exports (for checking against the oracle) ----
    def _slice(self):
        """(SA entries, table entries) held by this index: all of them, or a partition's slice."""
        if not getattr(self, "_part", None):
            return self.n, (1 << (2 * self.k)) + 1
        pi = self.part_info()
        g, rb = pi["part"], pi["route_bases"]
        keys = pi["part_keys"]
        return pi["rank_hi"] - pi["rank_lo"], (keys[g + 1] - keys[g]) * (1 << (2 * (self.k - rb))) + 1

    def export_sa(self) -> np.ndarray:
        """The suffix array (a partition: its slice SA[rank_lo .. rank_hi))."""
        out = np.empty(self._slice()[0], dtype=np.uint32)
        _check(lib().sa_index_export_sa(self._h, out.ctypes.data), "sa_index_export_sa")
        return out

    def export_table(self) -> np.ndarray:
        """The k-mer bracket table (a partition: the entries of its route keys, clamped to its ranks)."""
        out = np.empty(self._slice()[1], dtype=np.uint32)
        _check(lib().sa_index_export_table(self._h, out.ctypes.data), "sa_index_export_table")
        return out

    def export_text(self) -> np.ndarray:
        out = np.empty((self.n + 31) // 32, dtype=np.uint64)
        _check(lib().sa_index_export_text(self._h, out.ctypes.data), "sa_index_export_text")
        return out

    # ---- the hot path ----
    def workspace_size(self, Q: int, stride: int, flags: int) -> int:
        ws = _sz()
        _check(lib().sa_match_workspace_size(self._h, Q, stride, flags, ctypes.byref(ws)), "sa_match_workspace_size")
        return ws.value

    def order_workspace_size(self, Q: int, key_bases: int = 0, buckets: bool = False) -> int:
        ws = _sz()
        kb = int(key_bases) | (SA_ORDER_BUCKETS if buckets else 0)
        _check(lib().sa_match_order_workspace_size_ex(Q, kb, ctypes.byref(ws)), "sa_match_order_workspace_size_ex")
        return ws.value

    def order(self, words, lens=None, fixed_len: Optional[int] = None, out=None, stream=None, workspace=None,
              key_bases: int = 0, ordered_words=None, ordered_lens=None, n_reads: Optional[int] = None,
              buckets: bool = False):
        """sa_match_order: a permutation of the reads sorted by their first key_bases bases (0 = 12);
        optionally also the rows / lengths arranged in that order (for match(..., rows_ordered=True)).
        n_reads: give it (with a 1-D `words` stream and fixed_len) for the dense layout.
        buckets: SA_ORDER_BUCKETS (bucket placement; equal keys in no fixed order)."""
        import torch
        Q, stride = _rows(words, n_reads)
        kb = int(key_bases) | (SA_ORDER_BUCKETS if buckets else 0)
        need = _sz()
        _check(lib().sa_match_order_workspace_size_ex(Q, kb, ctypes.byref(need)), "sa_match_order_workspace_size_ex")
        if workspace is None or workspace.numel() < need.value:
            workspace = _empty(max(1, need.value), torch.uint8, words.device, stream)
        if out is None:
            out = _empty(Q, torch.int32, words.device, stream)
        _check(lib().sa_match_order(self._h, _dptr(words), _dptr(lens), int(fixed_len or 0), stride, Q, kb,
                                    _dptr(out), _dptr(ordered_words), _dptr(ordered_lens), _dptr(workspace),
                                    workspace.numel(), _stream_ptr(stream)), "sa_match_order")
        return out

    def match(self, words, lens=None, fixed_len: Optional[int] = None, out=None, stream=None, want_stats=False,
              presort: bool = False, workspace=None, order=None, rows_ordered: bool = False,
              n_reads: Optional[int] = None, cooperative: bool = False, smem_tree: int = 0, tree_key_bases: int = 0,
              defer: int = 0, wide: bool = False):
        """sa_match_batch on device tensors.

        words: CUDA int64 tensor [Q, stride] (uint64 bit patterns, include/sa.h layout).
        lens:  CUDA int32 tensor [Q] (uint32 lengths) or None with fixed_len.
        presort: SA_MATCH_PRESORT (include/sa.h): order the reads inside the call.
        order: optional CUDA int32 [Q] permutation from order() (thread slot t takes read order[t]).
        rows_ordered: words/lens are order()'s ordered_words/ordered_lens (row t is read order[t]).
        n_reads: with a 1-D `words` stream and fixed_len: the dense layout (include/sa.h).
        cooperative: SA_MATCH_COOPERATIVE (reads over 128 bases: 8/16/32 lanes per read).
        smem_tree: L > 0 selects SA_MATCH_SMEM_TREE with L levels (tree_key_bases: the order's key length).
        defer: b > 0 selects SA_MATCH_DEFER: reads whose k-mer bracket holds more than 2^b suffixes go to a
        second pass.
        wide: SA_MATCH_WIDE (the large-batch load hints, automatic from 2^20 reads, at any batch size).
        workspace: optional CUDA uint8 tensor of >= workspace_size() bytes (allocated if None).
        Returns a CUDA int32 tensor [Q, 2] holding uint32 (lo, hi) -- view it as uint32 on the host --
        and, with want_stats, also an int32 tensor [2, Q]: row 0 steps | text windows << 16, row 1 the
        read's algorithmic bytes (SA_MATCH_STATS).
        """
        import torch
        assert words.is_cuda and words.dtype == torch.int64 and words.is_contiguous()
        Q, stride = _rows(words, n_reads)
        if lens is None and fixed_len is None:
            raise ValueError("give lens or fixed_len")
        if lens is not None:
            assert lens.is_cuda and lens.dtype == torch.int32 and lens.numel() == Q and lens.is_contiguous()
        if out is None:
            out = _empty((Q, 2), torch.int32, words.device, stream)
        assert out.is_cuda and out.dtype == torch.int32 and out.numel() == 2 * Q and out.is_contiguous()
        flags = (SA_MATCH_STATS if want_stats else 0) | (SA_MATCH_PRESORT if presort else 0) | \
                (SA_MATCH_ROWS_ORDERED if rows_ordered else 0) | (SA_MATCH_COOPERATIVE if cooperative else 0)
        if smem_tree:  # levels of the shared-memory top tree (include/sa.h SA_MATCH_SMEM_TREE)
            flags |= SA_MATCH_SMEM_TREE | ((int(smem_tree) & 15) << 8) | ((int(tree_key_bases) & 31) << 12)
        if defer:
            flags |= SA_MATCH_DEFER | ((int(defer) & 15) << 18)
        if wide:
            flags |= SA_MATCH_WIDE
        need = self.workspace_size(Q, stride, flags) \
            if flags & (SA_MATCH_STATS | SA_MATCH_PRESORT | SA_MATCH_DEFER) else 0
        if need and (workspace is None or workspace.numel() < need):
            workspace = _empty(need, torch.uint8, words.device, stream)
        ws_ptr, ws_bytes = (_dptr(workspace), workspace.numel()) if workspace is not None else (None, 0)
        _check(lib().sa_match_batch(self._h, _dptr(words), _dptr(lens), int(fixed_len or 0), stride, Q, _dptr(order),
                                    _dptr(out), ws_ptr, ws_bytes, flags, _stream_ptr(stream)),
               "sa_match_batch")
        if want_stats:  # [2, Q]: row 0 steps | text windows << 16, row 1 algorithmic bytes (include/sa.h)
            return out, workspace[: 8 * Q].view(torch.int32).view(2, Q)
        return out

    def match_host(self, words: np.ndarray, lens: Optional[np.ndarray] = None, fixed_len: Optional[int] = None,
                   out: Optional[np.ndarray] = None, chunk: int = 0, n_reads: Optional[int] = None) -> np.ndarray:
        """sa_match_batch_host: host buffers in (pinned recommended), intervals out; synchronous.

        words/lens/out may be numpy arrays or pinned CPU torch tensors (anything with .ctypes or .data_ptr())."""
        def hptr(a):
            if a is None:
                return None
            return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
        Q, stride = _rows(words, n_reads)
        if out is None:
            out = np.empty((Q, 2), dtype=np.uint32)
        _check(lib().sa_match_batch_host(self._h, hptr(words), hptr(lens), int(fixed_len or 0), stride, Q, hptr(out),
                                         int(chunk)), "sa_match_batch_host")
        return out

    def locate_offsets(self, lohi, stream=None):
        """sa_locate_offsets: exclusive prefix sum of the counts (CUDA int64 [Q+1]); offsets[Q] = total."""
        import torch
        Q = lohi.shape[0]
        offsets = _empty(Q + 1, torch.int64, lohi.device, stream)
        ws = _sz()
        _check(lib().sa_locate_workspace_size(Q, ctypes.byref(ws)), "sa_locate_workspace_size")
        wsb = _empty(max(1, ws.value), torch.uint8, lohi.device, stream)
        _check(lib().sa_locate_offsets(self._h, _dptr(lohi), Q, _dptr(offsets), _dptr(wsb), ws.value,
                                       _stream_ptr(stream)), "sa_locate_offsets")
        return offsets

    def locate_positions(self, lohi, offsets, n_reads: Optional[int] = None, stream=None, out=None):
        """sa_locate over the first n_reads reads (default all): positions SA[lo..hi) in SA order, int32 [total].
        out: optional preallocated int32 tensor of >= offsets[n_reads] entries."""
        import torch
        Q = lohi.shape[0] if n_reads is None else int(n_reads)
        if out is None:
            if stream is not None:  # offsets were written on `stream`: wait for it before reading the total
                stream.synchronize()
            out = _empty(int(offsets[Q].item()), torch.int32, lohi.device, stream)
        positions = out
        _check(lib().sa_locate(self._h, _dptr(lohi), _dptr(offsets), Q, _dptr(positions), _stream_ptr(stream)),
               "sa_locate")
        return positions

    def locate(self, lohi, stream=None) -> Tuple["object", "object"]:
        """Positions SA[lo..hi) of every read (SA order).  Returns (offsets int64 [Q+1], positions int32 [total])."""
        offsets = self.locate_offsets(lohi, stream)
        return offsets, self.locate_positions(lohi, offsets, stream=stream)


class Tree:
    """Flattened suffix tree of an Index (sa_tree_create); keeps the index alive while it lives."""

    def __init__(self, index: "Index"):
        h = _p()
        _check(lib().sa_tree_create(index._h, ctypes.byref(h)), "sa_tree_create")
        self._h, self.index = h, index
        nodes, nb = _u64(), _u64()
        _check(lib().sa_tree_info(h, ctypes.byref(nodes), ctypes.byref(nb)), "sa_tree_info")
        self.nodes, self.device_bytes = nodes.value, nb.value

    def close(self):
        if getattr(self, "_h", None):
            lib().sa_tree_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def match(self, words, lens=None, fixed_len: Optional[int] = None, out=None, stream=None, order=None):
        """sa_tree_match: the same [lo, hi) per read as Index.match, by walking the tree."""
        import torch
        Q, stride = words.shape
        if out is None:
            out = _empty((Q, 2), torch.int32, words.device, stream)
        _check(lib().sa_tree_match(self._h, _dptr(words), _dptr(lens), int(fixed_len or 0), stride, Q, _dptr(order),
                                   _dptr(out), _stream_ptr(stream)), "sa_tree_match")
        return out


def scatter_results(order, in_lohi, out=None, stream=None):
    """sa_scatter_results: out[order[t]] = in_lohi[t]."""
    import torch
    Q = in_lohi.shape[0]
    if out is None:
        out = torch.empty_like(in_lohi)
    _check(lib().sa_scatter_results(_dptr(order), _dptr(in_lohi), Q, _dptr(out), _stream_ptr(stream)),
           "sa_scatter_results")
    return out


def dc3_trace(ref):
    """sa_dc3_trace: (sample_rank uint32[n], nonsample uint32[ceil(n/3)]) of the paper's DC3 steps 1-2."""
    if isinstance(ref, str):
        ref = ref.encode("ascii")
    arr = np.frombuffer(ref, dtype=np.uint8) if isinstance(ref, (bytes, bytearray)) else \
        np.ascontiguousarray(ref, dtype=np.uint8)
    n = arr.size
    rank = np.empty(n, dtype=np.uint32)
    b0 = np.empty((n + 2) // 3, dtype=np.uint32)
    _check(lib().sa_dc3_trace(arr.ctypes.data, n, rank.ctypes.data, b0.ctypes.data), "sa_dc3_trace")
    return rank, b0


def random_gather(device: int = 0, buffer_bytes: int = 16 << 30, access_bytes: int = 32, n_threads: int = 148 * 2048 * 4,
                  loads: int = 64, dependent: int = 0) -> dict:
    """Random-access microbenchmark: dependent=0 independent loads, 1 pointer-chased loads, 2 stores,
    10-13 PTX cache operators, 20 TMA bulk copies, 21 cp.async (LDGSTS), 22 the L2::64B hint (32-B accesses)."""
    ms = ctypes.c_float()
    _check(lib().sa_tool_random_gather(device, buffer_bytes, access_bytes, n_threads, loads, int(dependent),
                                       ctypes.byref(ms)), "sa_tool_random_gather")
    accesses = n_threads * loads
    return {"ms": ms.value, "accesses": accesses, "access_bytes": access_bytes,
            "GBps": accesses * access_bytes / (ms.value * 1e-3) / 1e9,
            "Gaccess_per_s": accesses / (ms.value * 1e-3) / 1e9}
