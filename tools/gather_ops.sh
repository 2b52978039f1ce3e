#!/bin/bash
# DRAM sectors per random access for each cache operator / access size / L2 fetch limit (ncu)
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__sectors_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
for fetch in none 32; do
 for acc in 32 8; do
  for mode in 10 11 12 13; do
    if [ $fetch = none ]; then envp="X=0"; else envp="SA_L2_FETCH_BYTES=$fetch"; fi
    out=$(env $envp $NCU --metrics $M --clock-control none -k regex:k_gather -c 1 --csv python -c "
import sys; sys.path.insert(0, '.')
import paper_1303_3692_b200 as sa
sa.random_gather(0, buffer_bytes=16 << 30, access_bytes=$acc, n_threads=148 * 2048 * 4, loads=64, dependent=$mode)
" 2>/dev/null | grep -E '^"[0-9]' | awk -F'","' '{gsub(/"/,"",$NF); printf "%s=%s ", $(NF-2), $NF}')
    echo "fetch=$fetch acc=$acc mode=$mode accesses=$((148*2048*4*64)) $out"
  done
 done
done
