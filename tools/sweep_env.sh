#!/bin/bash
# like sweep.sh but each variant is "ENV=VAL|bench args": bash tools/sweep_env.sh <tag> <config> "SA_MATCH_MINBLOCKS=6|--layout rec32" ...
tag=$1; cfg=$2; shift 2
for v in "$@"; do
  envs=${v%%|*}; args=${v#*|}
  name=$(echo "$envs$args" | tr -c 'A-Za-z0-9' '_' )
  env $envs timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu $args \
     > gpurun_out/sweep_${tag}_${cfg}_${name:-default}.json 2> gpurun_out/sweep_${tag}_${cfg}_${name:-default}.log
  python - "$v" gpurun_out/sweep_${tag}_${cfg}_${name:-default}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:44s} {d['value']/1e9:7.3f} Gq/s  step {d['ms_per_step']:7.3f} ms  match {d['launch_ms']['median']:7.3f} ms  "
          f"steps={d['search_stats']['mean_steps']:.2f} texts={d['search_stats']['mean_text_windows']:.2f} k={d['config']['kmer_k']}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
