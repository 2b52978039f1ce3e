out=gpurun_out/r02i; mkdir -p $out
SA_LIB_PATH=variants/libsa_dual3.so timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q > $out/pytest_dual3.txt 2>&1; echo "rc=$?" >> $out/pytest_dual3.txt
timeout 900 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_dual.so variants/libsa_dual3.so --m 100 --q 100000000 --reps 2 > $out/ab_dual_100M.jsonl 2> $out/ab_dual_100M.log
timeout 900 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_dual.so variants/libsa_dual3.so --m 16 64 100 --q 12500000 --reps 2 > $out/ab_dual_12M.jsonl 2> $out/ab_dual_12M.log
