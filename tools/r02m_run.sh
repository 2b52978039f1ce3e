out=gpurun_out/r02m; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -k "order or dense or c1_full or c2_full or smem_tree" -x -q > $out/pytest_order.txt 2>&1; echo "rc=$?" >> $out/pytest_order.txt
timeout 900 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_cubsort.so --m 100 --q 100000000 --reps 2 > $out/ab_sort_100M.jsonl 2> $out/ab_sort_100M.log
timeout 900 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_cubsort.so --m 100 --q 12500000 --reps 2 > $out/ab_sort_12M.jsonl 2> $out/ab_sort_12M.log
