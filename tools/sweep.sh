#!/bin/bash
# A/B sweep of match-kernel variants on one GPU: bash tools/sweep.sh <tag> <config> "<variant args>"...
tag=$1; cfg=$2; shift 2
for v in "$@"; do
  name=$(echo "$v" | tr -d ' -' )
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu $v \
     > gpurun_out/sweep_${tag}_${cfg}_${name:-default}.json 2> gpurun_out/sweep_${tag}_${cfg}_${name:-default}.log
  python - "$v" gpurun_out/sweep_${tag}_${cfg}_${name:-default}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:32s} {d['value']/1e9:7.3f} Gq/s  {d['ms_per_step']:8.3f} ms  frac={d['roofline']['frac']:.3f}  "
          f"steps={d['search_stats']['mean_steps']:.2f} texts={d['search_stats']['mean_text_windows']:.2f} "
          f"k={d['config']['kmer_k']} idxGB={d['index_bytes']/1e9:.1f}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
