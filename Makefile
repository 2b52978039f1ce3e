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

$(PKG)/libsa.so: $(CU_SRCS) $(CU_HDRS)
	$(NVCC) $(NVFLAGS) -Iinclude -shared -o $@ $(CU_SRCS) -lcudart 2> build/ptxas.log || (cat build/ptxas.log; false)

$(shell mkdir -p build)

# A/B build variant: 128-bit instead of 256-bit record / read-row loads
variants/libsa_load128.so: $(CU_SRCS) $(CU_HDRS)
	mkdir -p variants && $(NVCC) $(NVFLAGS) -DSA_LOAD128 -Iinclude -shared -o $@ $(CU_SRCS) -lcudart 2> build/ptxas_load128.log || (cat build/ptxas_load128.log; false)

clean:
	rm -f synth/libsynth.so oracle/liboracle.so $(PKG)/libsa.so

.PHONY: all clean
