"""Histogram of search probes per read at C4 (SA_MATCH_STATS): where the record lines go."""
import json, sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1303_3692_b200 as sa

cfg = synth.CONFIGS["C4"]
ref = cfg.reference()
idx = sa.Index(ref, layout="rec32")
words, lens = cfg.reads(ref, q_count=20_000_000)
w = torch.from_numpy(words.view(np.int64)).cuda()
perm = idx.order(w, None, fixed_len=100)
out, st = idx.match(w, None, fixed_len=100, order=perm, want_stats=True)
st = st[0]
steps = (st.cpu().numpy().view(np.uint32) & 0xFFFF).astype(np.int64)
lohi = out.cpu().numpy().view(np.uint32).astype(np.int64)
cnt = lohi[:, 1] - lohi[:, 0]
h = np.bincount(steps, minlength=48)
res = {"reads": int(steps.size), "mean_steps": float(steps.mean()),
       "hist": h.tolist(),
       "share_of_probes_from_reads_with_gt8": float(steps[steps > 8].sum() / steps.sum()),
       "frac_reads_gt8": float((steps > 8).mean()),
       "count_hist_log2": np.bincount(np.log2(np.maximum(cnt, 1)).astype(int)).tolist(),
       "miss_frac": float((cnt == 0).mean())}
print(json.dumps(res))
