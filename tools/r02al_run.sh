out=gpurun_out/r02al; mkdir -p $out
timeout 600 python tools/order_bench.py 12500000 paper_1303_3692_b200/libsa.so variants/libsa_i32.so > $out/order_12M.jsonl 2>&1
timeout 600 python tools/order_bench.py 25000000 paper_1303_3692_b200/libsa.so variants/libsa_i32.so > $out/order_25M.jsonl 2>&1
timeout 600 python tools/order_bench.py 100000000 paper_1303_3692_b200/libsa.so variants/libsa_i32.so > $out/order_100M.jsonl 2>&1
