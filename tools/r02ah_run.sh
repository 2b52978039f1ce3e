out=gpurun_out/r02ah; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wide or c1_full or short_queries or random_texts" > $out/pytest.txt 2>&1; echo "rc=$?" >> $out/pytest.txt
L="paper_1303_3692_b200/libsa.so variants/libsa_nowide.so"
timeout 1500 python tools/ab_libs.py --libs $L --m 16 32 64 100 150 --q 50000000 --reps 2 > $out/ab_c5.jsonl 2> $out/ab_c5.log
