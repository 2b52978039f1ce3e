"""A/B of libsa builds on one box, one process: the reference and every read batch are generated once;
for each library the index is built (rec32, auto k), then for each read length the batch is ordered
(sa_match_order, 12 bases) and matched (sa_match_batch) 8 times, the last 5 timed with CUDA events.

  python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_x.so --m 100 1000 [--q N]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--libs", nargs="+", required=True)
ap.add_argument("--m", nargs="+", type=int, default=[100])
ap.add_argument("--q", type=int, default=50_000_000)
ap.add_argument("--layout", type=int, default=2, help="sa_index_opts.flags (2 = rec32, 1 = plain, 0 = rec16)")
ap.add_argument("--k", type=int, default=0)
ap.add_argument("--reps", type=int, default=3, help="interleaved repetitions of the whole lib loop")
args = ap.parse_args()

_p, _u32, _u64, _sz = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_size_t


class Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("kmer_k", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32)]


def load(so):
    L = ctypes.CDLL(os.path.abspath(so))
    L.sa_index_create.argtypes = [_p, _u64, ctypes.POINTER(Opts), ctypes.POINTER(_p)]
    L.sa_index_destroy.argtypes = [_p]
    L.sa_match_order_workspace_size.argtypes = [_u64, ctypes.POINTER(_sz)]
    L.sa_match_order.argtypes = [_p, _p, _p, _u32, _u32, _u64, _u32, _p, _p, _p, _p, _sz, _p]
    L.sa_match_batch.argtypes = [_p, _p, _p, _u32, _u32, _u64, _p, _p, _p, _sz, _u32, _p]
    return L


cfg0 = synth.CONFIGS["C5"]
ref = cfg0.reference()
torch.cuda.init()
batches = {}
for m in args.m:
    cfg = cfg0.with_m(m) if m != 100 else synth.CONFIGS["C4"]
    stride = (m + 31) // 32
    w = torch.empty((args.q, stride), dtype=torch.int64, pin_memory=True)
    cfg.reads(ref, q_count=args.q, words_out=w.numpy().view(np.uint64))
    batches[m] = w
libs = [load(so) for so in args.libs]
s = torch.cuda.current_stream().cuda_stream
for rep in range(args.reps):
    for so, L in zip(args.libs, libs):
        h = _p()
        assert L.sa_index_create(ref.ctypes.data, len(ref), ctypes.byref(Opts(0, args.k, args.layout, 0)),
                                 ctypes.byref(h)) == 0
        for m in args.m:
            wh = batches[m]
            Q, stride = wh.shape
            w = wh.cuda()
            sz = _sz()
            L.sa_match_order_workspace_size(Q, ctypes.byref(sz))
            ws = torch.empty(sz.value, dtype=torch.uint8, device="cuda")
            perm = torch.empty(Q, dtype=torch.int32, device="cuda")
            out = torch.empty((Q, 2), dtype=torch.int32, device="cuda")
            ts, to = [], []
            for i in range(8):
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                e[0].record()
                assert L.sa_match_order(h, w.data_ptr(), None, m, stride, Q, 12, perm.data_ptr(), None, None,
                                        ws.data_ptr(), sz.value, s) == 0
                e[1].record()
                assert L.sa_match_batch(h, w.data_ptr(), None, m, stride, Q, perm.data_ptr(), out.data_ptr(), None, 0,
                                        0, s) == 0
                e[2].record()
                torch.cuda.synchronize()
                if i >= 3:
                    to.append(e[0].elapsed_time(e[1]))
                    ts.append(e[1].elapsed_time(e[2]))
            print(json.dumps({"rep": rep, "lib": os.path.basename(so), "m": m, "Q": Q, "match_ms": float(np.median(ts)),
                              "order_ms": float(np.median(to)),
                              "checksum": int((out[:, 1].long() - out[:, 0].long()).sum())}), flush=True)
            del w, ws, perm, out
        L.sa_index_destroy(h)
        torch.cuda.empty_cache()
