#!/bin/bash
# ncu evidence for the f2 (DC3 build) and f3 (tree walk) rows at C3
NCU=/usr/local/cuda/bin/ncu
# DC3 build launch list (C3) vs prefix doubling
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_dc3_c3.csv \
  python -c "
import sys; sys.path.insert(0, '.')
import synth, paper_1303_3692_b200 as sa
ref = synth.CONFIGS['C3'].reference()
sa.Index(ref, build='dc3', layout='plain')
" > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_doubling_c3.csv \
  python -c "
import sys; sys.path.insert(0, '.')
import synth, paper_1303_3692_b200 as sa
ref = synth.CONFIGS['C3'].reference()
sa.Index(ref, layout='plain')
" > /dev/null 2>&1
# the tree walk kernel at C3 (full set, one launch)
$NCU --set full --clock-control none --import-source on -k regex:k_tree_match -s 1 -c 1 -o gpurun_out/prof_tree_c3 -f \
  python bench.py --config C3 --tree --steps 2 --warmup 1 --no-e2e --no-cpu --no-locate > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on -k regex:k_match -s 1 -c 1 -o gpurun_out/prof_match_c3 -f \
  python bench.py --config C3 --steps 2 --warmup 1 --no-e2e --no-cpu --no-locate > /dev/null 2>&1
ls -la gpurun_out/*c3*
