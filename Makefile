# Build for the B200-native TSDF path (sm_100a only; no other targets).
#   paper_1611_03631_b200/libvxg.so                 : product (CUDA kernels + C ABI)
#   paper_1611_03631_b200/workload/libworkload.so   : seeded synthetic scans (bench/test input)
#   oracle/liboracle.so, oracle/_ref/*              : CPU checker (oracle/Makefile)
NVCC      ?= nvcc
CC_OMP    ?= /usr/bin/gcc
CUDA_HOME ?= /usr/local/cuda
PKG       := paper_1611_03631_b200
ARCH      := -gencode arch=compute_100a,code=sm_100a
# --fmad=false + IEEE div/sqrt (nvcc defaults): parity with the reference's
# non-contracted fp32/fp64 arithmetic. No -use_fast_math.
NVFLAGS   := $(ARCH) -O3 -lineinfo --fmad=false -prec-div=true -prec-sqrt=true -std=c++17 \
             -Xcompiler -fPIC,-ffp-contract=off -Xptxas -warn-spills
CSRC      := $(PKG)/csrc
LIB       := $(PKG)/libvxg.so
OBJDIR    := build/obj

.PHONY: all lib workload oracle clean ptxas
all: lib workload oracle

lib: $(LIB)
workload: $(PKG)/workload/libworkload.so
oracle:
	$(MAKE) -C oracle

$(OBJDIR)/vxg_tsdf.o: $(CSRC)/vxg_tsdf.cu $(CSRC)/vxg_kernels.cuh $(CSRC)/vxg_device.cuh $(CSRC)/vxg_sort.cuh $(CSRC)/vxg_esdf.cuh include/vxg.h include/vxg_types.h
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(OBJDIR)/bucket_schedule.o: $(CSRC)/bucket_schedule.cpp
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -x cu -c -o $@ $<

$(OBJDIR)/vxg_io.o: $(CSRC)/vxg_io.cu include/vxg.h include/vxg_types.h
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(LIB): $(OBJDIR)/vxg_tsdf.o $(OBJDIR)/bucket_schedule.o $(OBJDIR)/vxg_io.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -lcudart_static -Xcompiler -fPIC

$(PKG)/workload/libworkload.so: $(PKG)/workload/workload.c
	$(CC_OMP) -O2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -o $@ $< -lm

ptxas:
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /dev/null $(CSRC)/vxg_tsdf.cu 2>&1 | grep -E "Function properties|registers|spill" | paste - - - | sed 's/ptxas info    ://g'

clean:
	rm -rf build $(LIB) $(PKG)/workload/libworkload.so
	$(MAKE) -C oracle clean
