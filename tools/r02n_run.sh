out=gpurun_out/r02n; mkdir -p $out
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum --clock-control none -k regex:"k_order|k_onesweep|Onesweep|k_presort|Histogram" --csv --log-file $out/order_launches.csv python tools/order_bench.py 100000000 paper_1303_3692_b200/libsa.so variants/libsa_cubsort.so > $out/order_ncu.log 2>&1
python tools/order_bench.py 100000000 paper_1303_3692_b200/libsa.so variants/libsa_cubsort.so > $out/order_time.jsonl 2>&1
