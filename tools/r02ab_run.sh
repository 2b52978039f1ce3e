out=gpurun_out/r02ab; mkdir -p $out
SA_LIB_PATH=variants/libsa_lpf.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "long or group_kernel or staged or dense" > $out/pytest_lpf.txt 2>&1; echo "rc=$?" >> $out/pytest_lpf.txt
timeout 1500 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_lpf.so --m 150 250 500 1000 --q 50000000 --reps 2 > $out/ab_lpf.jsonl 2> $out/ab_lpf.log
