#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over the kernels added late in round 2: the long-read
# split shortcut (k_match<0>), the bucket ordering (k_bucket_count / k_bucket_place, SA_ORDER_BUCKETS) and,
# with SA_LIB_PATH=variants/libsa_staged.so, the TMA-staged long-read kernel (k_match_staged).
CS=/usr/local/cuda/bin/compute-sanitizer
out=${1:-gpurun_out/sanitize_r02b}; mkdir -p $out
cat > /tmp/sanitize_r02b.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth, oracle, paper_1303_3692_b200 as sa
ref = synth.reference(synth.REF_REPEAT, 150_000, 11)
S = oracle.encode(ref); SA = oracle.sa_naive(S)
w, l = synth.reads(ref, 3000, 100, 1200, 0.1, 0.05, 12)
want = oracle.search_batch(S, SA, w, l).astype(np.uint32)
wt = torch.from_numpy(w.view(np.int64)).cuda(); lt = torch.from_numpy(l.view(np.int32)).cuda()
for layout in ("rec16", "rec32"):
    idx = sa.Index(ref, layout=layout)
    assert np.array_equal(idx.match(wt, lt).cpu().numpy().view(np.uint32), want)
    perm = idx.order(wt, lt, buckets=True)
    assert np.array_equal(idx.match(wt, lt, order=perm).cpu().numpy().view(np.uint32), want)
    idx.close()
print("ok")
PY
for lib in "" variants/libsa_staged.so; do
  tag=${lib:+staged}; tag=${tag:-default}
  for tool in memcheck racecheck synccheck; do
    SA_LIB_PATH=$lib $CS --tool $tool --error-exitcode 9 --print-limit 20 python /tmp/sanitize_r02b.py > $out/${tag}_$tool.txt 2>&1
    echo "$tag $tool rc=$? $(tail -1 $out/${tag}_$tool.txt)" | tee -a $out/summary.txt
  done
done
