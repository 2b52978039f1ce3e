#!/bin/bash
# Build an A/B variant of libsa with extra defines on the match path only:
#   bash tools/variant.sh <name> "<-DFOO=1 ...>"   ->  variants/libsa_<name>.so
# (sa_match.cu -- the translation unit holding the search kernel -- is recompiled with the defines; the
# other objects come from the default build in build/.)
set -e
name=$1; defs=$2
cd "$(dirname "$0")/.."
make -s -j8 all
mkdir -p variants
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3,-Wall -Xptxas -v --expt-relaxed-constexpr"
$NV $defs -Iinclude -c -o build/var_${name}_sa_match.o paper_1303_3692_b200/csrc/sa_match.cu 2> build/ptxas_var_${name}.log || (cat build/ptxas_var_${name}.log; false)
objs=$(ls build/*.o | grep -v "build/var_" | grep -v "build/sa_match.o")
$NV -shared -o variants/libsa_${name}.so build/var_${name}_sa_match.o $objs -lcudart
echo variants/libsa_${name}.so
