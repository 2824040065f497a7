# Builds every native artefact in-tree (they travel to the GPU box with gpurun).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude
# make DEV=1: development build that reads the GC_* tuning knobs from the environment
ifeq ($(DEV),1)
NVFLAGS += -DGC_DEV_KNOBS
endif
# make CHECKS=1: device invariant checks (GC_CHECK) compiled in
ifeq ($(CHECKS),1)
NVFLAGS += -DGC_CHECKS
endif
# make MINB=n: resident CTAs per SM the k_solve register budget is sized for (A/B builds)
ifneq ($(MINB),)
NVFLAGS += -DGC_MINB=$(MINB)
endif
PKG := paper_1008_0502_b200

all: $(PKG)/libgc.so synth/libsynth.so oracle/liboracle.so

$(PKG)/libgc.so: $(PKG)/csrc/gc_solver.cu $(PKG)/csrc/gc_saliency.cu $(wildcard $(PKG)/csrc/*.cuh) include/gc.h Makefile
	$(NVCC) $(NVFLAGS) -Xptxas -v -Xptxas -dlcm=cg -c -o $(PKG)/csrc/gc_solver.o $(PKG)/csrc/gc_solver.cu 2> build_gc_ptxas.log || (cat build_gc_ptxas.log; false)
	$(NVCC) $(NVFLAGS) -fmad=false -c -o $(PKG)/csrc/gc_saliency.o $(PKG)/csrc/gc_saliency.cu
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(PKG)/csrc/gc_solver.o $(PKG)/csrc/gc_saliency.o

synth/libsynth.so: synth/synth_host.c synth/synth_cuda.cu synth/synth.h
	gcc -O2 -fPIC -c synth/synth_host.c -o synth/synth_host.o
	$(NVCC) $(ARCH) -O3 -Xcompiler -fPIC -c synth/synth_cuda.cu -o synth/synth_cuda.o
	$(NVCC) $(ARCH) -shared -cudart static -o $@ synth/synth_host.o synth/synth_cuda.o

oracle/liboracle.so: oracle/oracle.cpp
	g++ -O2 -std=c++17 -fPIC -shared -pthread -o $@ oracle/oracle.cpp

clean:
	rm -f $(PKG)/libgc.so $(PKG)/csrc/*.o synth/libsynth.so synth/*.o oracle/liboracle.so build_gc_ptxas.log

.PHONY: all clean
