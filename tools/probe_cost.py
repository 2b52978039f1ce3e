"""Where k_match's time goes at C4 by probe count: the reads are ordered and split by their probe count
(SA_MATCH_STATS); each class is matched alone (rows already in order, no permutation) and timed."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1303_3692_b200 as sa  # noqa: E402


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
    return float(np.median(ts))


cfg = synth.CONFIGS["C4"]
ref = cfg.reference()
idx = sa.Index(ref, layout="rec32")
Q = int(os.environ.get("Q", 50_000_000))
words, _ = cfg.reads(ref, q_count=Q)
w = torch.from_numpy(words.view(np.int64)).cuda()
del words
perm = idx.order(w, None, fixed_len=100)
ws = w[perm.long()].contiguous()          # rows in order
_, st = idx.match(ws, None, fixed_len=100, want_stats=True)
st = st[0]
steps = (st.view(torch.int32).to(torch.int64) & 0xFFFF)
res = {"Q": Q, "all_ms": timed(idx, ws), "classes": []}
for lo, hi in [(0, 0), (1, 1), (2, 2), (3, 4), (5, 8), (9, 16), (17, 64)]:
    sel = ((steps >= lo) & (steps <= hi)).nonzero().squeeze(1)
    if sel.numel() == 0:
        continue
    sub = ws[sel].contiguous()
    ms = timed(idx, sub)
    res["classes"].append({"probes": [lo, hi], "reads": int(sel.numel()), "frac_reads": sel.numel() / Q,
                           "ms": ms, "ns_per_read": ms * 1e6 / sel.numel(),
                           "probes_sum": int(steps[sel].sum())})
res["sum_class_ms"] = sum(c["ms"] for c in res["classes"])
print(json.dumps(res))
