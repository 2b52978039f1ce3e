out=gpurun_out/r02y; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "defer or order or c1_full or c2_full" > $out/pytest_defer.txt 2>&1; echo "rc=$?" >> $out/pytest_defer.txt
for d in 0 2 3 4 5 6; do
  timeout 900 python bench.py --defer $d --no-cpu --no-e2e --no-locate > $out/bench_100M_d$d.json 2> $out/bench_100M_d$d.log
done
for d in 0 3 4 5; do
  timeout 900 python bench.py --q 12500000 --defer $d --no-cpu --no-e2e --no-locate > $out/bench_12M_d$d.json 2> $out/bench_12M_d$d.log
done
