# final HEAD verification of round 2 (64-thread k_match blocks): GPU tests (incl. the full-size slow tier), smoke,
# bench lines (C4, C4 at the 2/4/8-GPU per-rank batches, the C5 sweep), launch lists + ncu --set full of k_match (C4, C5 m=1000)
out=gpurun_out/r02ao; mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
timeout 1800 python -m pytest tests -m "gpu and not slow" -x -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
timeout 900 python bench.py > $out/bench_c4.json 2> $out/bench_c4.log
for q in 50000000 25000000 12500000; do
  timeout 900 python bench.py --q $q --no-cpu --no-e2e --no-locate > $out/bench_c4_q$q.json 2> $out/bench_c4_q$q.log
done
for m in 16 32 64 100 150 250 500 1000; do
  timeout 600 python bench.py --config C5 --m $m --no-e2e --no-cpu --no-locate --steps 10 > $out/bench_c5_m$m.json 2> $out/bench_c5_m$m.log
done
timeout 1500 bash tools/prof_c4.sh r02ao_c4 --no-locate
timeout 1500 bash tools/prof_c4.sh r02ao_c5m1000 --config C5 --m 1000 --no-locate
timeout 2400 python -m pytest tests -m "slow" -x -q > $out/pytest_slow.txt 2>&1; echo "rc=$?" >> $out/pytest_slow.txt
