out=gpurun_out/r02aa; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "l2_out or c1_full" > $out/pytest.txt 2>&1; echo "rc=$?" >> $out/pytest.txt
python -c "
import torch; p=torch.cuda.get_device_properties(0); print(p)
from cuda.bindings import runtime as rt
print(rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0))
print(rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0))
" > $out/props.txt 2>&1
for q in 12500000 25000000 100000000; do
  for f in "" "--l2-out"; do
    timeout 900 python bench.py --q $q $f --no-cpu --no-e2e --no-locate > $out/bench_${q}${f}.json 2> $out/bench_${q}${f}.log
  done
done
