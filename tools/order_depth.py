"""How much does the depth of the read ordering matter to k_match at C4?  The rows are put in order
(no permutation in the kernel) by the first 12 bases (the bench's ordering), the first 32 bases, or
all bases, and the in-order kernel is timed on each."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1303_3692_b200 as sa  # noqa: E402

SIGN = -0x8000000000000000  # int64 xor flips unsigned order into signed order


def timed(idx, w, reps=5):
    out = torch.empty((w.shape[0], 2), dtype=torch.int32, device=w.device)
    idx.match(w, None, fixed_len=100, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        idx.match(w, None, fixed_len=100, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), out


def lex_order(w, words):
    perm = torch.arange(w.shape[0], device=w.device)
    for j in reversed(range(words)):
        col = (w[perm, j] ^ SIGN)
        _, p = torch.sort(col, stable=True)
        perm = perm[p]
    return perm


cfg = synth.CONFIGS["C4"]
ref = cfg.reference()
idx = sa.Index(ref, layout="rec32")
Q = int(os.environ.get("Q", 50_000_000))
words, _ = cfg.reads(ref, q_count=Q)
w = torch.from_numpy(words.view(np.int64)).cuda()
del words
res = {"Q": Q}
perm12 = idx.order(w, None, fixed_len=100).long()
ms, o12 = timed(idx, w[perm12].contiguous())
res["order12_ms"] = ms
for name, nw in [("order32", 1), ("order64", 2), ("order_all", 4)]:
    p = lex_order(w, nw)
    ms, o = timed(idx, w[p].contiguous())
    res[name + "_ms"] = ms
    # same intervals per read regardless of order
    a = torch.empty_like(o); a[p] = o
    b = torch.empty_like(o12); b[perm12] = o12
    res[name + "_same"] = bool(torch.equal(a, b))
print(json.dumps(res))
