#!/bin/bash
# compute-sanitizer memcheck over the f2-f4 features and the sub-tables
CS=/usr/local/cuda/bin/compute-sanitizer
cat > /tmp/sanitize_run2.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth, paper_1303_3692_b200 as sa
ref = synth.reference(synth.REF_REPEAT, 100_000, 7)
w, l = synth.reads(ref, 4096, 20, 200, 0.1, 0.05, 8)
wt = torch.from_numpy(w.view(np.int64)).cuda(); lt = torch.from_numpy(l.view(np.int32)).cuda()
full = sa.Index(ref, layout="rec32", k=6, subtables=True)
base = full.match(wt, lt)
tree = sa.Tree(full)
assert torch.equal(tree.match(wt, lt), base)
dc = sa.Index(ref, build="dc3", layout="plain")
assert torch.equal(dc.match(wt, lt), sa.Index(ref, layout="plain").match(wt, lt))
rank, b0 = sa.dc3_trace("acggtacgtac")
parts = [sa.Index(ref, layout="rec16", part=(g, 3, 4)) for g in range(3)]
order, ow, ol, offs = parts[0].route(wt, lt)
offs = offs.cpu().tolist()
res = torch.empty_like(base)
for g in range(3):
    if offs[g + 1] > offs[g]:
        res[offs[g]:offs[g + 1]] = parts[g].match(ow[offs[g]:offs[g + 1]], ol[offs[g]:offs[g + 1]])
got = sa.scatter_results(order, res)
assert torch.equal(got, base)  # all reads are >= k of the parts
torch.cuda.synchronize()
print("ok")
PY
$CS --tool memcheck --error-exitcode 9 --print-limit 20 python /tmp/sanitize_run2.py > gpurun_out/sanitize2_memcheck.txt 2>&1
echo "memcheck rc=$? $(tail -1 gpurun_out/sanitize2_memcheck.txt)"
