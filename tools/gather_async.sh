#!/bin/bash
# DRAM sectors per random 32-B access through the LSU (10), TMA bulk copy (20), LDGSTS (21) and the
# L2::64B prefetch hint (22): ncu counters plus the uninstrumented rate
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__sectors_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_op_read.sum
for mode in 10 20 21 22; do
  out=$($NCU --metrics $M --clock-control none -k regex:k_gather -c 1 --csv python -c "
import sys; sys.path.insert(0, '.')
import paper_1303_3692_b200 as sa
sa.random_gather(0, buffer_bytes=16 << 30, access_bytes=32, n_threads=148 * 2048 * 4, loads=64, dependent=$mode)
" 2>/dev/null | grep -E '^"[0-9]' | awk -F'","' '{gsub(/"/,"",$NF); printf "%s=%s ", $(NF-2), $NF}')
  rate=$(python -c "
import sys; sys.path.insert(0, '.')
import paper_1303_3692_b200 as sa
r = sa.random_gather(0, buffer_bytes=16 << 30, access_bytes=32, n_threads=148 * 2048 * 4, loads=64, dependent=$mode)
print('Gaccess_per_s=%.2f' % r['Gaccess_per_s'])")
  echo "mode=$mode accesses=$((148*2048*4*64)) $rate $out"
done
