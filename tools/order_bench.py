"""Time sa_match_order alone (the index does not matter for the ordering: a small one is built) on a C4
read batch: python tools/order_bench.py [Q] [lib.so ...]"""
import ctypes, json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

Q = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
libs = sys.argv[2:] or ["paper_1303_3692_b200/libsa.so"]
_p, _u32, _u64, _sz = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_size_t


class Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("kmer_k", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32)]


cfg = synth.CONFIGS["C4"]
small = synth.reference(synth.REF_UNIFORM, 100_000, 1)
big = cfg.reference()
w = torch.empty((Q, 4), dtype=torch.int64)
cfg.reads(big, q_count=Q, words_out=w.numpy().view(np.uint64))
w = w.cuda()
for so in libs:
    L = ctypes.CDLL(os.path.abspath(so))
    L.sa_index_create.argtypes = [_p, _u64, ctypes.POINTER(Opts), ctypes.POINTER(_p)]
    L.sa_match_order_workspace_size.argtypes = [_u64, ctypes.POINTER(_sz)]
    L.sa_match_order.argtypes = [_p, _p, _p, _u32, _u32, _u64, _u32, _p, _p, _p, _p, _sz, _p]
    h = _p()
    assert L.sa_index_create(small.ctypes.data, len(small), ctypes.byref(Opts(0, 0, 0, 0)), ctypes.byref(h)) == 0
    sz = _sz()
    L.sa_match_order_workspace_size(Q, ctypes.byref(sz))
    ws = torch.empty(sz.value, dtype=torch.uint8, device="cuda")
    perm = torch.empty(Q, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    ts = []
    for i in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        assert L.sa_match_order(h, w.data_ptr(), None, 100, 4, Q, 12, perm.data_ptr(), None, None, ws.data_ptr(),
                                sz.value, s) == 0
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    print(json.dumps({"lib": os.path.basename(so), "Q": Q, "order_ms": float(np.median(ts)),
                      "perm_checksum": int((perm.long() * torch.arange(Q, device="cuda")).sum())}), flush=True)
