out=gpurun_out/r02g; mkdir -p $out
timeout 1800 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_bulkpf.so variants/libsa_m3.so variants/libsa_pfm3.so variants/libsa_chunk2m3.so --m 150 250 500 1000 --reps 2 > $out/ab_long.jsonl 2> $out/ab_long.log
