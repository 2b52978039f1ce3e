out=gpurun_out/r02v; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi.py -m gpu -x -q -k "order or dense or staged" > $out/pytest_order.txt 2>&1; echo "rc=$?" >> $out/pytest_order.txt
for q in 12500000 25000000 50000000 100000000; do
  for meth in sort buckets; do
    timeout 900 python bench.py --q $q --order-method $meth --no-cpu --no-e2e --no-locate > $out/bench_${q}_${meth}.json 2> $out/bench_${q}_${meth}.log
  done
done
timeout 900 python bench.py --q 12500000 --order-method buckets --order-bases 11 --no-cpu --no-e2e --no-locate > $out/bench_12500000_buckets11.json 2> $out/bench_12500000_buckets11.log
timeout 900 python bench.py --q 12500000 --order-method buckets --order-bases 13 --no-cpu --no-e2e --no-locate > $out/bench_12500000_buckets13.json 2> $out/bench_12500000_buckets13.log
