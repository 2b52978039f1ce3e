out=gpurun_out/r02u; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "staged or long_reads or group_kernel or dense" > $out/pytest_long.txt 2>&1; echo "rc=$?" >> $out/pytest_long.txt
timeout 1500 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_nostaged.so variants/libsa_stagedwarp.so --m 150 250 500 1000 --q 50000000 --reps 1 > $out/ab_staged.jsonl 2> $out/ab_staged.log
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_match_staged -c 1 -o $out/prof_staged_m150 -f python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so --m 150 --q 20000000 --reps 1 > $out/ncu150.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_match_staged -c 1 -o $out/prof_staged_m1000 -f python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so --m 1000 --q 20000000 --reps 1 > $out/ncu1000.log 2>&1
