out=gpurun_out/r02p; mkdir -p $out
python tools/order_bench.py 100000000 paper_1303_3692_b200/libsa.so variants/libsa_cubsort.so variants/libsa_os_fix_t256i16.so variants/libsa_os_fix_t256i32.so variants/libsa_os_fix_t512i8.so variants/libsa_os_fix_t256i8.so > $out/order_100M.jsonl 2>&1
python tools/order_bench.py 12500000 paper_1303_3692_b200/libsa.so variants/libsa_cubsort.so variants/libsa_os_fix_t256i16.so variants/libsa_os_fix_t256i8.so > $out/order_12M.jsonl 2>&1
