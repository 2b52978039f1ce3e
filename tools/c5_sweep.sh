#!/bin/bash
# C5: read-length sweep on the C4 reference (50M reads per length), one bench line per m
for m in ${C5_MS:-16 32 64 100 150 250 500 1000}; do
  timeout 900 python bench.py --config C5 --m $m --steps 5 --warmup 3 --no-e2e --no-cpu "$@" \
     > gpurun_out/c5_m${m}.json 2> gpurun_out/c5_m${m}.log
  python - $m gpurun_out/c5_m${m}.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"m={sys.argv[1]:5s} {d['value']/1e9:7.3f} Gq/s  step {d['ms_per_step']:8.3f} ms  match {d['launch_ms']['median']:8.3f} ms "
          f"steps={d['search_stats']['mean_steps']:.2f} texts={d['search_stats']['mean_text_windows']:.2f} "
          f"hits={d['shards'][0][0]} locate={d.get('locate')}")
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
