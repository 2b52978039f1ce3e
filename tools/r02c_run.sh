out=gpurun_out/r02c; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q > $out/pytest_partition.txt 2>&1; echo "rc=$?" >> $out/pytest_partition.txt
timeout 1500 bash tools/prof_c4.sh r02c_c4 --no-locate
timeout 1500 bash tools/prof_c4.sh r02c_c5m1000 --config C5 --m 1000 --no-locate
