out=gpurun_out/r02w; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "staged or long or 129 or group_kernel or dense or stats or bucket" > $out/pytest_long.txt 2>&1; echo "rc=$?" >> $out/pytest_long.txt
timeout 1500 python tools/ab_libs.py --libs paper_1303_3692_b200/libsa.so variants/libsa_nosplit.so --m 150 250 500 1000 --q 50000000 --reps 2 > $out/ab_split.jsonl 2> $out/ab_split.log
