#!/bin/bash
# parity of the long-read paths, then C5 A/B: 4-word chunked compare (this build) vs the previous
# word-at-a-time thread path (variants/libsa_prev.so with SA_MATCH_NO_GROUP=1) vs the cooperative kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "group or long_reads or 129_to_256 or dense_layout or order_is" \
  > gpurun_out/lr_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/lr_pytest.txt
tail -2 gpurun_out/lr_pytest.txt
bash tools/sweep_env.sh lr C4 "X=0|"
for m in ${LR_MS:-150 250 500 1000}; do
  for v in "X=0|" "SA_LIB_PATH=variants/libsa_prev.so SA_MATCH_NO_GROUP=1|" "X=0|--cooperative"; do
    envs=${v%%|*}; args=${v#*|}
    name=$(echo "$envs$args" | tr -c 'A-Za-z0-9' '_')
    env $envs timeout 600 python bench.py --config C5 --m $m --steps 5 --warmup 3 --no-e2e --no-cpu --no-locate $args \
      > gpurun_out/lr_m${m}_${name}.json 2> gpurun_out/lr_m${m}_${name}.log
    python -c "
import json
d=json.loads(open('gpurun_out/lr_m${m}_${name}.json').read().strip().splitlines()[-1])
print('m=$m %-60s' % '$v', round(d['value']/1e9,3), 'Gq/s step', round(d['ms_per_step'],3), 'match', round(d['launch_ms']['median'],3), 'texts', round(d['search_stats']['mean_text_windows'],3))" || tail -3 gpurun_out/lr_m${m}_${name}.log
  done
done
