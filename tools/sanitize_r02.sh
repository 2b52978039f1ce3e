#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over the round-2 kernels: long reads in two phases
# (k_match<0>), the shared-memory top tree (k_match_tree: TMA bulk copies + mbarrier), the bucket trees,
# the partitioned index (slice build, route / pack / collect) and the sub-table hash.
CS=/usr/local/cuda/bin/compute-sanitizer
out=${1:-gpurun_out/sanitize_r02}; mkdir -p $out
cat > /tmp/sanitize_r02.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth, paper_1303_3692_b200 as sa
ref = synth.reference(synth.REF_REPEAT, 150_000, 11)
w, l = synth.reads(ref, 3000, 0, 400, 0.1, 0.05, 12)
wt = torch.from_numpy(w.view(np.int64)).cuda(); lt = torch.from_numpy(l.view(np.int32)).cuda()
ws, ls = synth.reads(ref, 3000, 0, 128, 0.1, 0.05, 13)
wst = torch.from_numpy(ws.view(np.int64)).cuda(); lst = torch.from_numpy(ls.view(np.int32)).cuda()
base = sa.Index(ref, layout="rec32")
want = base.match(wt, lt)
want_s = base.match(wst, lst)
perm = base.order(wst, lst)
for lv in (3, 8):
    assert torch.equal(base.match(wst, lst, order=perm, smem_tree=lv), want_s)
bt = sa.Index(ref, layout="rec32", k=6, bucket_tree=True)
assert torch.equal(bt.match(wt, lt), want) and torch.equal(bt.match(wst, lst), want_s)
st = sa.Index(ref, layout="rec32", k=16, subtables=True)
assert torch.equal(st.match(wt, lt), want)
parts = [sa.Index(ref, layout="rec32", part=(g, 3, 5)) for g in range(3)]
order, ow, ol, offs = parts[0].route(wt, lt)
o = offs.cpu().tolist(); Q = wt.shape[0]; ns = Q - o[3]
send = [o[g + 1] - o[g] + ns for g in range(3)]
sw, sl = parts[0].part_pack(ow, ol, offs, sum(send))
back, b0 = [], 0
for g in range(3):
    back.append(parts[g].match(sw[b0:b0 + send[g]], sl[b0:b0 + send[g]])); b0 += send[g]
got = parts[0].part_collect(torch.cat(back), offs, order, Q)
torch.cuda.synchronize()
assert torch.equal(got, want)
print("ok")
PY
for tool in memcheck racecheck synccheck; do
  $CS --tool $tool --error-exitcode 9 --print-limit 20 python /tmp/sanitize_r02.py > $out/$tool.txt 2>&1
  echo "$tool rc=$? $(tail -1 $out/$tool.txt)" | tee -a $out/summary.txt
done
