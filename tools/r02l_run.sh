out=gpurun_out/r02l; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "k16_table_sampled" -x -q > $out/pytest_k16table.txt 2>&1; echo "rc=$?" >> $out/pytest_k16table.txt
for v in "--q 12500000 --k 15" "--q 12500000 --k 14" "--q 12500000" "--q 25000000 --k 15" "--q 50000000 --k 15" "--k 15" "--layout plain" "--layout rec16"; do
  name=$(echo "$v" | tr -d ' -'); timeout 600 python bench.py --no-e2e --no-cpu --no-locate --steps 20 $v > $out/bench_${name:-default}.json 2> $out/bench_${name:-default}.log
done
