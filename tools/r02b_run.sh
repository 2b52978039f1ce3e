out=gpurun_out/r02b; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_partition.py -x -q > $out/pytest_partition.txt 2>&1; echo "rc=$?" >> $out/pytest_partition.txt
timeout 1200 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_nopf.so variants/libsa_rowpf.so variants/libsa_r01.so --m 100 150 500 1000 --reps 2 > $out/ab_long.jsonl 2> $out/ab_long.log
timeout 600 python bench.py --no-cpu --no-locate --steps 10 > $out/bench_c4_e2e_order.json 2> $out/bench_c4_e2e_order.log
SA_LIB_PATH=variants/libsa_hostnoorder.so timeout 600 python bench.py --no-cpu --no-locate --steps 10 > $out/bench_c4_e2e_noorder.json 2> $out/bench_c4_e2e_noorder.log
