#!/bin/bash
# repeated A/B of the ordering key length (noise: ~3% between runs)
for rep in 1 2 3; do
  for kb in 8 10 12; do
    python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-locate --order-bases $kb > gpurun_out/order_ab_${kb}_${rep}.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/order_ab_${kb}_${rep}.json').read().strip().splitlines()[-1])
print('bases=$kb rep=$rep', round(d['value']/1e9,3), 'step', round(d['ms_per_step'],3), 'match', round(d['launch_ms']['median'],3))"
  done
done
