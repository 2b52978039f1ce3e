out=gpurun_out/r02ak; mkdir -p $out
timeout 1500 bash tools/prof_c4.sh r02ak_c4q12M --no-locate --q 12500000
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_write.sum --clock-control none -k regex:"Onesweep|k_presort|Histogram" --csv --log-file $out/order_100M.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-locate > $out/order_100M.json 2> $out/order_100M.log
