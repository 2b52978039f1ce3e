"""Experiment: k_match with one full 32-byte sector written per read (variants/libsa_outpad.so, out
buffer of 8 uint32 per read) against the standard 8-byte result, C4, 100 M reads, ordered."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1303_3692_b200 as sa  # noqa: E402

pad = "outpad" in os.environ.get("SA_LIB_PATH", "")
cfg = synth.CONFIGS["C4"]
ref = cfg.reference()
idx = sa.Index(ref, layout="rec32")
Q = cfg.Q
w = torch.empty((Q, 4), dtype=torch.int64, pin_memory=True)
cfg.reads(ref, words_out=w.numpy().view(np.uint64))
w = w.cuda()
perm = idx.order(w, None, fixed_len=100)
out = torch.empty((Q, 8 if pad else 2), dtype=torch.int32, device="cuda")
# the binding checks out's shape: call the C ABI directly through the binding's low-level helper
ws = torch.empty(max(1, idx.workspace_size(Q, 4, 0)), dtype=torch.uint8, device="cuda")
lib = sa.lib()
import ctypes
def run():
    st = lib.sa_match_batch(idx._h, ctypes.c_void_p(w.data_ptr()), None, 100, 4, Q, ctypes.c_void_p(perm.data_ptr()),
                            ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(), 0,
                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0, st
for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
lohi = out[:, :2].contiguous()
chk = idx.match(w, None, fixed_len=100, order=perm) if not pad else None
print(json.dumps({"pad": pad, "match_ms_median": float(np.median(ts)), "min": min(ts),
                  "checksum": int((lohi[:, 1].long() - lohi[:, 0].long()).sum())}))
