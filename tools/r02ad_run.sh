out=gpurun_out/r02ad; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ctab or c1_full or order_is or k16" > $out/pytest_ctab.txt 2>&1; echo "rc=$?" >> $out/pytest_ctab.txt
for q in 100000000 50000000 25000000 12500000; do
  for c in off on; do
    timeout 900 python bench.py --q $q --ctab $c --no-cpu --no-e2e --no-locate > $out/bench_${q}_$c.json 2> $out/bench_${q}_$c.log
  done
done
