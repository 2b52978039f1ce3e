out=gpurun_out/r02af; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1_full or c2_full or repeat_rich or paper or random_texts" > $out/pytest_default.txt 2>&1; echo "rc=$?" >> $out/pytest_default.txt
for v in rec64 idx64; do
  SA_LIB_PATH=variants/libsa_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1_full or c2_full or repeat_rich" > $out/pytest_$v.txt 2>&1; echo "rc=$?" >> $out/pytest_$v.txt
done
L="paper_1303_3692_b200/libsa.so variants/libsa_row0.so variants/libsa_rec64.so variants/libsa_tab64.so variants/libsa_idx64.so"
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 100000000 --reps 2 > $out/ab_100M.jsonl 2> $out/ab_100M.log
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 12500000 --reps 2 > $out/ab_12M.jsonl 2> $out/ab_12M.log
timeout 1500 python tools/ab_libs.py --libs $L --m 100 --q 25000000 --reps 1 > $out/ab_25M.jsonl 2> $out/ab_25M.log
