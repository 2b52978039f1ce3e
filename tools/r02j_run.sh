out=gpurun_out/r02j; mkdir -p $out
bash tools/sanitize_r02.sh $out/sanitize
for v in "" "--graph" "--q 12500000" "--q 12500000 --graph" "--q 25000000 --graph" "--q 50000000 --graph"; do
  name=$(echo "$v" | tr -d ' -'); timeout 600 python bench.py --no-e2e --no-cpu --no-locate --steps 20 $v > $out/bench_${name:-default}.json 2> $out/bench_${name:-default}.log
done
for c in 1048576 2097152 8388608 16777216; do
  timeout 600 python bench.py --no-cpu --no-locate --steps 5 --e2e-chunk $c > $out/bench_e2e_chunk$c.json 2> $out/bench_e2e_chunk$c.log
done
