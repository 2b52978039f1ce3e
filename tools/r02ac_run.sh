out=gpurun_out/r02ac; mkdir -p $out
SA_LIB_PATH=variants/libsa_skeys.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "order or c1_full or c2_full or stats or dense or repeat_rich" > $out/pytest_skeys.txt 2>&1; echo "rc=$?" >> $out/pytest_skeys.txt
for q in 100000000 12500000; do
  for lib in "" variants/libsa_skeys.so; do
    tag=${lib:+skeys}; tag=${tag:-default}
    SA_LIB_PATH=$lib timeout 900 python bench.py --q $q --no-cpu --no-e2e --no-locate > $out/bench_${q}_$tag.json 2> $out/bench_${q}_$tag.log
  done
done
SA_LIB_PATH=variants/libsa_skeys.so timeout 900 python bench.py --no-cpu --no-e2e --no-locate > $out/bench_100000000_skeys2.json 2> $out/bench_100000000_skeys2.log
timeout 900 python bench.py --no-cpu --no-e2e --no-locate > $out/bench_100000000_default2.json 2> $out/bench_100000000_default2.log
