out=gpurun_out/r02am; mkdir -p $out
L="paper_1303_3692_b200/libsa.so variants/libsa_t128.so variants/libsa_t64.so variants/libsa_t256_m6.so"
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 100000000 --reps 2 > $out/ab_100M.jsonl 2> $out/ab_100M.log
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 12500000 --reps 2 > $out/ab_12M.jsonl 2> $out/ab_12M.log
