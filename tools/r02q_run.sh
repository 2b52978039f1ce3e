out=gpurun_out/r02q; mkdir -p $out
/usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:k_onesweep -s 4 -c 1 -o $out/prof_onesweep -f python tools/order_bench.py 100000000 > $out/prof.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none -k regex:OnesweepKernel -s 4 -c 1 -o $out/prof_cubonesweep -f python tools/order_bench.py 100000000 variants/libsa_cubsort.so > $out/prof_cub.log 2>&1
