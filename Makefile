# Build everything in-tree (the .so files travel to the GPU box with the gpurun snapshot).
#   make oracle  -> oracle/liboracle.so            (plain C, CPU, test infrastructure)
#   make gen     -> jacobi_gen/libjacobigen.so     (input generator, host + device twin)
#   make lib     -> paper_1403_5805_b200/libjacobi.so  (the product: C-ABI + sm_100a kernels)
#   make probe   -> probes/bwprobe                 (read-only HBM ceiling probe)
PY        ?= python
NVCC      ?= /usr/local/cuda/bin/nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v
NCCL_DIR  := $(shell $(PY) -c "import nvidia.nccl, os; print(list(nvidia.nccl.__path__)[0])" 2>/dev/null)
PKG       := paper_1403_5805_b200

LIB_SRCS  := $(PKG)/csrc/sweep.cu $(PKG)/csrc/cluster.cu $(PKG)/csrc/plan.cu $(PKG)/csrc/dist.cu
LIB_HDRS  := include/jacobi.h $(PKG)/csrc/internal.h

all: oracle gen lib lib-check probe

oracle: oracle/liboracle.so
oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -pthread -o $@ $< -lm

gen: jacobi_gen/libjacobigen.so
jacobi_gen/libjacobigen.so: jacobi_gen/gen_host.cpp jacobi_gen/gen_dev.cu jacobi_gen/gen_common.h jacobi_gen/jacobi_gen.h
	$(NVCC) -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC,-ffp-contract=off -shared -o $@ \
	    jacobi_gen/gen_host.cpp jacobi_gen/gen_dev.cu -lpthread

lib: $(PKG)/libjacobi.so
$(PKG)/libjacobi.so: $(LIB_SRCS) $(LIB_HDRS)
	$(NVCC) $(NVFLAGS) -Iinclude -I$(NCCL_DIR)/include -shared -o $@ $(LIB_SRCS) \
	    -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib 2> build_lib.log || (cat build_lib.log; false)

# Bounds-checked build of the product (device-side checks of every tile's A / x ranges; debug aid).
lib-check: $(PKG)/libjacobi_check.so
$(PKG)/libjacobi_check.so: $(LIB_SRCS) $(LIB_HDRS)
	$(NVCC) $(NVFLAGS) -DJACOBI_BOUNDS_CHECK -Iinclude -I$(NCCL_DIR)/include -shared -o $@ $(LIB_SRCS) \
	    -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib 2> build_lib_check.log || (cat build_lib_check.log; false)

probe: probes/bwprobe
probes/bwprobe: probes/bwprobe.cu
	$(NVCC) -O3 -std=c++17 $(ARCH) -lineinfo -o $@ $<

clean:
	rm -f oracle/liboracle.so jacobi_gen/libjacobigen.so $(PKG)/libjacobi.so $(PKG)/libjacobi_check.so probes/bwprobe build_lib.log build_lib_check.log

.PHONY: all oracle gen lib lib-check probe clean
