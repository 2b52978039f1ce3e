#!/bin/bash
# A/B of the group-cooperative long-read kernel (C5) and of the staged result write (C4); parity first
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "group or staged or long_reads or 129_to_256 or order_is or dense_layout" \
  > gpurun_out/ab_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_pytest.txt
tail -2 gpurun_out/ab_pytest.txt
bash tools/gather_async.sh > gpurun_out/gather_async.txt 2>&1; cat gpurun_out/gather_async.txt
for v in "X=0|" "X=0|--staged-write"; do
  bash tools/sweep_env.sh ab C4 "$v"
done
for m in 150 250 500 1000; do
  for e in X=0 SA_MATCH_NO_GROUP=1; do
    env $e timeout 600 python bench.py --config C5 --m $m --steps 5 --warmup 3 --no-e2e --no-cpu --no-locate \
      > gpurun_out/c5g_${e}_m${m}.json 2> gpurun_out/c5g_${e}_m${m}.log
    python -c "
import json,sys
d=json.loads(open('gpurun_out/c5g_${e}_m${m}.json').read().strip().splitlines()[-1])
print('$e m=$m', round(d['value']/1e9,3), 'Gq/s step', round(d['ms_per_step'],3), 'match', round(d['launch_ms']['median'],3), 'steps', d['search_stats']['mean_steps'], 'texts', d['search_stats']['mean_text_windows'])" || tail -3 gpurun_out/c5g_${e}_m${m}.log
  done
done
