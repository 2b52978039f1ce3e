for v in "" variants/libsa_t256_m5.so variants/libsa_head1.so variants/libsa_head1_m5.so; do
  for m in 150 250 1000; do
    SA_LIB_PATH=$v timeout 600 python bench.py --config C5 --m $m --steps 5 --warmup 3 --no-e2e --no-cpu --no-locate > gpurun_out/c5ab.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/c5ab.json').read().strip().splitlines()[-1]); print('${v:-default}', $m, round(d['value']/1e9,3), round(d['launch_ms']['median'],3))"
  done
done
