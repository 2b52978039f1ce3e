"""A/B of two libsa builds (possibly of different commits) through the stable part of the C ABI:
sa_index_create (rec32) + sa_match_order + sa_match_batch on one C4/C5 read batch, match timed with
CUDA events.  python tools/lib_ab.py <lib.so> <m> [Q]"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

so, m = sys.argv[1], int(sys.argv[2])
Q = int(sys.argv[3]) if len(sys.argv) > 3 else 50_000_000
L = ctypes.CDLL(so)
_p, _u32, _u64, _sz = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_size_t


class Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("kmer_k", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32)]


L.sa_index_create.argtypes = [_p, _u64, ctypes.POINTER(Opts), ctypes.POINTER(_p)]
L.sa_match_order_workspace_size.argtypes = [_u64, ctypes.POINTER(_sz)]
L.sa_match_order.argtypes = [_p, _p, _p, _u32, _u32, _u64, _u32, _p, _p, _p, _p, _sz, _p]
L.sa_match_batch.argtypes = [_p, _p, _p, _u32, _u32, _u64, _p, _p, _p, _sz, _u32, _p]

cfg = synth.CONFIGS["C5"].with_m(m)
ref = cfg.reference()
h = _p()
torch.cuda.init()
assert L.sa_index_create(ref.ctypes.data, len(ref), ctypes.byref(Opts(0, 0, 2, 0)), ctypes.byref(h)) == 0
stride = (m + 31) // 32
w = torch.empty((Q, stride), dtype=torch.int64)
cfg.reads(ref, q_count=Q, words_out=w.numpy().view(np.uint64))
w = w.cuda()
sz = _sz()
L.sa_match_order_workspace_size(Q, ctypes.byref(sz))
ws = torch.empty(sz.value, dtype=torch.uint8, device="cuda")
perm = torch.empty(Q, dtype=torch.int32, device="cuda")
out = torch.empty((Q, 2), dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
assert L.sa_match_order(h, w.data_ptr(), None, m, stride, Q, 12, perm.data_ptr(), None, None, ws.data_ptr(),
                        sz.value, s) == 0
ts = []
for i in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    assert L.sa_match_batch(h, w.data_ptr(), None, m, stride, Q, perm.data_ptr(), out.data_ptr(), None, 0, 0, s) == 0
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
print(json.dumps({"lib": os.path.basename(so), "m": m, "Q": Q, "match_ms": float(np.median(ts)),
                  "checksum": int((out[:, 1].long() - out[:, 0].long()).sum())}))
