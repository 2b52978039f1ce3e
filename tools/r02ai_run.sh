out=gpurun_out/r02ai; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "wide or long or 129 or group_kernel or dense or staged" > $out/pytest.txt 2>&1; echo "rc=$?" >> $out/pytest.txt
L="paper_1303_3692_b200/libsa.so variants/libsa_nowide.so"
timeout 1500 python tools/ab_libs.py --libs $L --m 150 250 500 1000 --q 50000000 --reps 2 > $out/ab_long.jsonl 2> $out/ab_long.log
