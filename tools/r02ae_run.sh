out=gpurun_out/r02ae; mkdir -p $out
for v in row64 row64na rowna; do
  SA_LIB_PATH=variants/libsa_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c1_full or c2_full or repeat_rich" > $out/pytest_$v.txt 2>&1; echo "rc=$?" >> $out/pytest_$v.txt
done
timeout 1500 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_row64.so variants/libsa_row64na.so variants/libsa_rowna.so --m 100 --q 100000000 --reps 2 > $out/ab_row_100M.jsonl 2> $out/ab_row_100M.log
timeout 1500 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_row64.so variants/libsa_row64na.so variants/libsa_rowna.so --m 100 --q 12500000 --reps 2 > $out/ab_row_12M.jsonl 2> $out/ab_row_12M.log
