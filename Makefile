# Build everything in-tree (the .so files travel to the GPU box with gpurun).
NVCC      ?= /usr/local/cuda/bin/nvcc
CC        := gcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3,-Wall -Xptxas -v --expt-relaxed-constexpr
CFLAGS    := -O2 -fPIC -fopenmp -Wall -Wextra

PKG       := paper_1303_3692_b200
CSRC      := $(PKG)/csrc
CU_SRCS   := $(wildcard $(CSRC)/*.cu)
CU_HDRS   := $(wildcard $(CSRC)/*.cuh) include/sa.h

all: synth/libsynth.so oracle/liboracle.so $(PKG)/libsa.so

synth/libsynth.so: synth/synth.c
	$(CC) $(CFLAGS) -shared -o $@ $< -lm

oracle/liboracle.so: oracle/oracle.c
	$(CC) $(CFLAGS) -shared -o $@ $<

# one object per translation unit (make -j compiles them in parallel), then one shared library
CU_OBJS   := $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS))

build/%.o: $(CSRC)/%.cu $(CU_HDRS)
	$(NVCC) $(NVFLAGS) -Iinclude -c -o $@ $< 2> build/ptxas_$*.log || (cat build/ptxas_$*.log; false)

$(PKG)/libsa.so: $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -lcudart
	cat build/ptxas_sa_*.log > build/ptxas.log

$(shell mkdir -p build)

# A/B build variants (variants/*.so; bench.py / tests / tools/ab_libs.py load one with SA_LIB_PATH=... or
# --libs): sa_match.cu (the search kernels) recompiled with the defines, linked with the default objects
VARIANTS := ldcg ldnoalloc ldca l2_64 l2_64na t128 t64 t128_m12 t64_m32 t256_m6 t64_m24 t128_m10 t64_m20 \
            t256_m1 outpad t256_m5 head1 head2 head3 head1_m5 bulkpf chunk2m3 m3 longwarp dual dual3 hostnoorder \
            packed onesweep staged stagedwarp nowide t32_m32 t96_m13 t256_m5b allwide
DEFS_onesweep := -DSA_ORDER_ONESWEEP
DEFS_staged := -DSA_MATCH_STAGED
DEFS_nowide := -DSA_NO_WIDE
DEFS_allwide := -DSA_WIDE_Q_LOG2=0
DEFS_t32_m32 := -DSA_MATCH_THREADS=32 -DSA_MATCH_MINB=32
DEFS_t96_m13 := -DSA_MATCH_THREADS=96 -DSA_MATCH_MINB=13
DEFS_t256_m5b := -DSA_MATCH_THREADS=256 -DSA_MATCH_MINB=5
DEFS_stagedwarp := -DSA_MATCH_STAGED -DSA_STAGED_WARPCMP
DEFS_ldcg := -DSA_LD_MODE=1
DEFS_ldnoalloc := -DSA_LD_MODE=2
DEFS_ldca := -DSA_LD_MODE=3
DEFS_l2_64 := -DSA_LD_MODE=4
DEFS_l2_64na := -DSA_LD_MODE=5
DEFS_t128 := -DSA_MATCH_THREADS=128
DEFS_t64 := -DSA_MATCH_THREADS=64
DEFS_t128_m12 := -DSA_MATCH_THREADS=128 -DSA_MATCH_MINB=12
DEFS_t64_m32 := -DSA_MATCH_THREADS=64 -DSA_MATCH_MINB=32
DEFS_t64_m24 := -DSA_MATCH_THREADS=64 -DSA_MATCH_MINB=24
DEFS_t256_m6 := -DSA_MATCH_THREADS=256 -DSA_MATCH_MINB=6
DEFS_t128_m10 := -DSA_MATCH_THREADS=128 -DSA_MATCH_MINB=10
DEFS_t64_m20 := -DSA_MATCH_THREADS=64 -DSA_MATCH_MINB=20
DEFS_t256_m1 := -DSA_MATCH_THREADS=256 -DSA_MATCH_MINB=1
DEFS_outpad := -DSA_OUT_PAD=1
DEFS_t256_m5 := -DSA_MATCH_THREADS=256 -DSA_MATCH_MINB=5
DEFS_head1 := -DSA_QW0_HEAD=1
DEFS_head2 := -DSA_QW0_HEAD=2
DEFS_head3 := -DSA_QW0_HEAD=3
DEFS_head1_m5 := -DSA_QW0_HEAD=1 -DSA_MATCH_MINB=5
DEFS_bulkpf := -DSA_BULK_PREFETCH
DEFS_chunk2m3 := -DSA_CHUNK2 -DSA_MATCH_MINB_LONG=3
DEFS_m3 := -DSA_MATCH_MINB_LONG=3
DEFS_longwarp := -DSA_LONG_WARP
DEFS_dual := -DSA_MATCH_DUAL
DEFS_dual3 := -DSA_MATCH_DUAL -DSA_DUAL_MINB=3
DEFS_hostnoorder := -DSA_HOST_NO_ORDER
DEFS_packed := -DSA_ORDER_PACKED
variants: $(addprefix variants/libsa_,$(addsuffix .so,$(VARIANTS)))
variants/libsa_%.so: $(CU_OBJS) $(CU_HDRS)
	bash tools/variant.sh $* "$(DEFS_$*)"

clean:
	rm -f synth/libsynth.so oracle/liboracle.so $(PKG)/libsa.so

.PHONY: all clean variants
