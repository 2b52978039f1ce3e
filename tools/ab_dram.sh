#!/bin/bash
# DRAM bytes + L2 sectors + duration of one k_match launch at C4 for each given libsa build
# usage: bash tools/ab_dram.sh <tag> [lib ...]   ("default" = the in-tree libsa.so)
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum
tag=$1; shift
for lib in "$@"; do
  name=$(basename $lib .so)
  if [ "$lib" = default ]; then envp=""; else envp="SA_LIB_PATH=$lib"; fi
  env $envp $NCU --metrics $M --clock-control none -k regex:k_match -s 1 -c 1 --csv \
      python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-locate 2>/dev/null | grep -E '^"[0-9]' > gpurun_out/ab_${tag}_${name}.csv
  python - $name gpurun_out/ab_${tag}_${name}.csv <<'PY'
import csv, sys
vals = {r[-3]: r[-1] for r in csv.reader(open(sys.argv[2])) if len(r) > 3}
print(sys.argv[1].ljust(20), " ".join(f"{k.split('.')[0]}={v}" for k, v in sorted(vals.items())))
PY
done
