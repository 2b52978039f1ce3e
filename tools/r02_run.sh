#!/bin/bash
# one gpurun call: tests (fast tier), the default bench line, the per-GPU batch curve, C5 m=1000
# usage: bash tools/r02_run.sh <tag> [pytest selection]
tag=$1; sel=${2:-"gpu and not slow"}
out=gpurun_out/$tag; mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $out/gpu.txt 2>&1
nproc > $out/host.txt; grep -m1 "model name" /proc/cpuinfo >> $out/host.txt; free -g >> $out/host.txt
timeout 1500 python -m pytest tests -m "$sel" -x -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
timeout 900 python bench.py > $out/bench_c4.json 2> $out/bench_c4.log
for q in 50000000 25000000 12500000; do
  timeout 600 python bench.py --q $q --no-e2e --no-cpu --no-locate --steps 20 > $out/bench_c4_q$q.json 2> $out/bench_c4_q$q.log
done
timeout 600 python bench.py --config C5 --m 1000 --no-e2e --no-cpu --no-locate --steps 10 > $out/bench_c5_m1000.json 2> $out/bench_c5_m1000.log
