out=gpurun_out/r02ag; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wide or c1_full or c2_full or dense or long_reads" > $out/pytest.txt 2>&1; echo "rc=$?" >> $out/pytest.txt
L="paper_1303_3692_b200/libsa.so variants/libsa_nowide.so"
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 100000000 --reps 2 > $out/ab_100M.jsonl 2> $out/ab_100M.log
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 50000000 --reps 2 > $out/ab_50M.jsonl 2> $out/ab_50M.log
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 12500000 --reps 2 > $out/ab_12M.jsonl 2> $out/ab_12M.log
timeout 900 python bench.py > $out/bench_c4.json 2> $out/bench_c4.log
