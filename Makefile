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

# A/B build variants (variants/*.so; bench.py / tests load one with SA_LIB_PATH=...)
VARIANTS := variants/libsa_ldcg.so variants/libsa_ldnoalloc.so variants/libsa_ldca.so variants/libsa_l2_64.so \
            variants/libsa_l2_64na.so variants/libsa_t128.so variants/libsa_t64.so variants/libsa_t128_m12.so \
            variants/libsa_t64_m32.so variants/libsa_t256_m6.so variants/libsa_t64_m24.so variants/libsa_t128_m10.so \
            variants/libsa_t64_m20.so variants/libsa_t256_m1.so variants/libsa_outpad.so variants/libsa_t256_m5.so \
            variants/libsa_head1.so variants/libsa_head2.so variants/libsa_head3.so variants/libsa_head1_m5.so \
            variants/libsa_bulkpf.so
variants/libsa_ldcg.so: DEFS := -DSA_LD_MODE=1
variants/libsa_ldnoalloc.so: DEFS := -DSA_LD_MODE=2
variants/libsa_ldca.so: DEFS := -DSA_LD_MODE=3
variants/libsa_l2_64.so: DEFS := -DSA_LD_MODE=4
variants/libsa_l2_64na.so: DEFS := -DSA_LD_MODE=5
variants/libsa_t128.so: DEFS := -DSA_MATCH_THREADS=128
variants/libsa_t64.so: DEFS := -DSA_MATCH_THREADS=64
variants/libsa_t128_m12.so: DEFS := -DSA_MATCH_THREADS=128 -DSA_MATCH_MINB=12
variants/libsa_t64_m32.so: DEFS := -DSA_MATCH_THREADS=64 -DSA_MATCH_MINB=32
variants/libsa_t64_m24.so: DEFS := -DSA_MATCH_THREADS=64 -DSA_MATCH_MINB=24
variants/libsa_t256_m6.so: DEFS := -DSA_MATCH_THREADS=256 -DSA_MATCH_MINB=6
variants/libsa_t128_m10.so: DEFS := -DSA_MATCH_THREADS=128 -DSA_MATCH_MINB=10
variants/libsa_t64_m20.so: DEFS := -DSA_MATCH_THREADS=64 -DSA_MATCH_MINB=20
variants/libsa_t256_m1.so: DEFS := -DSA_MATCH_THREADS=256 -DSA_MATCH_MINB=1
variants/libsa_outpad.so: DEFS := -DSA_OUT_PAD=1
variants/libsa_t256_m5.so: DEFS := -DSA_MATCH_THREADS=256 -DSA_MATCH_MINB=5
variants/libsa_head1.so: DEFS := -DSA_QW0_HEAD=1
variants/libsa_head2.so: DEFS := -DSA_QW0_HEAD=2
variants/libsa_head3.so: DEFS := -DSA_QW0_HEAD=3
variants/libsa_head1_m5.so: DEFS := -DSA_QW0_HEAD=1 -DSA_MATCH_MINB=5
variants/libsa_bulkpf.so: DEFS := -DSA_BULK_PREFETCH
variants: $(VARIANTS)
variants/%.so: $(CU_SRCS) $(CU_HDRS)
	mkdir -p variants && $(NVCC) $(NVFLAGS) $(DEFS) -Iinclude -shared -o $@ $(CU_SRCS) -lcudart 2> build/ptxas_$(notdir $@).log || (cat build/ptxas_$(notdir $@).log; false)

clean:
	rm -f synth/libsynth.so oracle/liboracle.so $(PKG)/libsa.so

.PHONY: all clean variants
