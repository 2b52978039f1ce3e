out=gpurun_out/r02an; mkdir -p $out
L="paper_1303_3692_b200/libsa.so variants/libsa_t128.so variants/libsa_t64.so"
timeout 1500 python tools/ab_libs.py --libs $L --m 16 100 150 500 1000 --q 50000000 --reps 1 > $out/ab_c5.jsonl 2> $out/ab_c5.log
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 25000000 --reps 2 > $out/ab_25M.jsonl 2> $out/ab_25M.log
