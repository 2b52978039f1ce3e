#!/bin/bash
# A/B: the L2::64B fetch-size hint on every search load (variants/*.so) at C4; launch list of the staged write
mkdir -p gpurun_out
bash tools/sweep_env.sh l2 C4 "X=0|" "SA_LIB_PATH=variants/libsa_l2_64.so|" "SA_LIB_PATH=variants/libsa_l2_64na.so|" "X=0|"
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__sectors_read.sum,dram__sectors_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum
for v in "X=0" "SA_LIB_PATH=variants/libsa_l2_64.so"; do
  env $v $NCU --metrics $M --clock-control none -k regex:k_match -c 2 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-locate \
    2>/dev/null | grep -E '^"[0-9]' | awk -F'","' -v v="$v" '{gsub(/"/,"",$NF); printf "%s %s %s=%s\n", v, $5, $(NF-2), $NF}' | sed 's/(const sa_search::MatchArgs)//'
done > gpurun_out/l2hint_ncu.txt
cat gpurun_out/l2hint_ncu.txt
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_staged.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-locate --staged-write > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_staged.csv "k_match|k_unpartition|Onesweep|Histogram|presort|Exclusive" | tail -25
