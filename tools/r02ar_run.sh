out=gpurun_out/r02ar; mkdir -p $out
timeout 1800 python -m pytest tests -m "gpu and not slow" -x -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
timeout 900 python bench.py > $out/bench_c4.json 2> $out/bench_c4.log
for q in 50000000 25000000 12500000; do
  timeout 900 python bench.py --q $q --no-cpu --no-e2e --no-locate > $out/bench_c4_q$q.json 2> $out/bench_c4_q$q.log
done
timeout 1500 bash tools/prof_c4.sh r02ar_c4q12M --no-locate --q 12500000
timeout 2400 python -m pytest tests -m "slow" -x -q -k "c4" > $out/pytest_slow_c4.txt 2>&1; echo "rc=$?" >> $out/pytest_slow_c4.txt
