out=gpurun_out/r02aq; mkdir -p $out
L="paper_1303_3692_b200/libsa.so variants/libsa_allwide.so variants/libsa_nowide.so"
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 12500000 --reps 3 > $out/ab_12M.jsonl 2> $out/ab_12M.log
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 25000000 --reps 2 > $out/ab_25M.jsonl 2> $out/ab_25M.log
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 100000000 --reps 1 > $out/ab_100M.jsonl 2> $out/ab_100M.log
