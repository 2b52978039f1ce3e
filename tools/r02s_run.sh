out=gpurun_out/r02s; mkdir -p $out
nvidia-smi > $out/nvidia-smi.txt 2>&1
timeout 1800 python -m pytest tests -m "gpu and not slow" -x -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
timeout 900 python bench.py > $out/bench_c4.json 2> $out/bench_c4.log
timeout 900 python bench.py --q 12500000 --no-cpu > $out/bench_c4_12M.json 2> $out/bench_c4_12M.log
