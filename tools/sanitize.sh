#!/bin/bash
# compute-sanitizer memcheck / racecheck / initcheck over a small end-to-end run of the C ABI
CS=/usr/local/cuda/bin/compute-sanitizer
cat > /tmp/sanitize_run.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth, paper_1303_3692_b200 as sa
ref = synth.reference(synth.REF_REPEAT, 200_000, 3)
for layout in ("rec16", "rec32", "plain"):
    for build in ("doubling", "dc3"):
        idx = sa.Index(ref, layout=layout, build=build)
        w, l = synth.reads(ref, 4096, 1, 200, 0.1, 0.05, 4)
        wt = torch.from_numpy(w.view(np.int64)).cuda(); lt = torch.from_numpy(l.view(np.int32)).cuda()
        perm = idx.order(wt, lt)
        out = idx.match(wt, lt, order=perm)
        out2 = idx.match(wt, lt, want_stats=True)[0]
        d, _ = synth.reads(ref, 4096, 100, 100, 0.1, 0.0, 5, dense=True)
        dd = torch.from_numpy(d.view(np.int64)).cuda()
        idx.match(dd, None, fixed_len=100, n_reads=4096)
        idx.match_host(d, None, fixed_len=100, n_reads=4096, chunk=1000)
        offs, pos = idx.locate(out)
        torch.cuda.synchronize()
        assert torch.equal(out, out2)
print("ok")
PY
for tool in memcheck racecheck initcheck; do
  $CS --tool $tool --error-exitcode 9 --print-limit 20 python /tmp/sanitize_run.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitize_$tool.txt)"
done
