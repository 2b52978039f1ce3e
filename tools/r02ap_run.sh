out=gpurun_out/r02ap; mkdir -p $out
L="paper_1303_3692_b200/libsa.so variants/libsa_t32_m32.so variants/libsa_t96_m13.so variants/libsa_t64_m24.so variants/libsa_t256_m5b.so"
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 100000000 --reps 2 > $out/ab_100M.jsonl 2> $out/ab_100M.log
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 12500000 --reps 2 > $out/ab_12M.jsonl 2> $out/ab_12M.log
timeout 1500 python tools/ab_libs.py --libs $L --m 150 500 --q 50000000 --reps 1 > $out/ab_c5.jsonl 2> $out/ab_c5.log
