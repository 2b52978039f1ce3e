out=gpurun_out/r02f; mkdir -p $out
timeout 900 python bench.py > $out/bench_c4.json 2> $out/bench_c4.log
for m in 16 32 64 100 150 250 500 1000; do
  timeout 600 python bench.py --config C5 --m $m --no-e2e --no-cpu --no-locate --steps 10 > $out/bench_c5_m$m.json 2> $out/bench_c5_m$m.log
done
timeout 1500 bash tools/prof_c4.sh r02f_c4 --no-locate
timeout 1500 bash tools/prof_c4.sh r02f_c5m1000 --config C5 --m 1000 --no-locate
timeout 2400 python -m pytest tests -m "slow" -x -q > $out/pytest_slow.txt 2>&1; echo "rc=$?" >> $out/pytest_slow.txt
