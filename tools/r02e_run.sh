out=gpurun_out/r02e; mkdir -p $out
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
timeout 1200 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_longwarp.so variants/libsa_r01.so --m 100 150 250 500 1000 --reps 2 > $out/ab_long.jsonl 2> $out/ab_long.log
for v in "" "--bucket-tree" "--q 12500000" "--q 12500000 --bucket-tree"; do
  name=$(echo "$v" | tr -d ' -'); timeout 600 python bench.py --no-e2e --no-cpu --no-locate --steps 10 $v > $out/bench_${name:-default}.json 2> $out/bench_${name:-default}.log
done
