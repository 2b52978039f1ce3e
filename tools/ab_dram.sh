#!/bin/bash
# DRAM bytes + duration of one k_match launch at C4 for the default and the 128-bit-load build
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
$NCU --metrics $M --clock-control none -k regex:k_match -s 1 -c 1 --csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-locate 2>/dev/null | grep -E "k_match" > gpurun_out/ab_dram_default.csv
SA_LIB_PATH=variants/libsa_load128.so $NCU --metrics $M --clock-control none -k regex:k_match -s 1 -c 1 --csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-locate 2>/dev/null | grep -E "k_match" > gpurun_out/ab_dram_load128.csv
cat gpurun_out/ab_dram_default.csv gpurun_out/ab_dram_load128.csv | awk -F'","' '{print $5, $(NF-2), $(NF-1), $NF}'
