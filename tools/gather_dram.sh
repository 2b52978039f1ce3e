#!/bin/bash
# DRAM bytes moved per random 32-B load / store (ncu on the microbenchmark kernels)
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__sectors_read.sum
$NCU --metrics $M --clock-control none -k regex:k_gather -s 1 -c 1 --csv python -c "
import sys; sys.path.insert(0, '.')
import paper_1303_3692_b200 as sa
print(sa.random_gather(0, buffer_bytes=16 << 30, access_bytes=32, n_threads=148 * 2048 * 4, loads=64))
" 2>/dev/null | grep -E '^"[0-9]' > gpurun_out/gather_dram.csv
$NCU --metrics $M --clock-control none -k regex:k_scatter -s 1 -c 1 --csv python -c "
import sys; sys.path.insert(0, '.')
import paper_1303_3692_b200 as sa
print(sa.random_gather(0, buffer_bytes=800 << 20, access_bytes=8, n_threads=148 * 2048 * 4, loads=64, dependent=2))
" 2>/dev/null | grep -E '^"[0-9]' > gpurun_out/scatter_dram.csv
echo "accesses per launch: $((148*2048*4*64))"
cat gpurun_out/gather_dram.csv gpurun_out/scatter_dram.csv | awk -F'","' '{print $5, $(NF-2), $NF}'
