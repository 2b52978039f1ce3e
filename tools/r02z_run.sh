out=gpurun_out/r02z; mkdir -p $out
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/launches_12M.csv python bench.py --q 12500000 --steps 3 --warmup 1 --no-e2e --no-cpu --no-locate > $out/launches_12M.json 2> $out/launches_12M.log
