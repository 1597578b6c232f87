# Top-level build: the product library (sm_100a only) and the CPU checker.
#   make            -> paper_1508_03619_b200/lib/libgk_bfs.so + oracle/
#   make lib        -> only the CUDA library
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_1508_03619_b200
CSRC := $(PKG)/csrc
LIB := $(PKG)/lib/libgk_bfs.so
SRCS := $(CSRC)/gk_bfs_small.cu $(CSRC)/gk_bfs_kernel.cu $(CSRC)/gk_bfs_resume.cu $(CSRC)/gk_bfs_kernel_c.cu $(CSRC)/gk_bfs_resume_c.cu $(CSRC)/gk_bfs_cluster.cu $(CSRC)/gk_bfs_sharded.cu $(CSRC)/gk_bc.cu $(CSRC)/gk_aux.cu $(CSRC)/gk_graph_build.cu $(CSRC)/gk_capi.cu $(CSRC)/gk_shard.cu $(CSRC)/gk_sg.cu $(CSRC)/gk_pack.cu
HDRS := $(CSRC)/gk_bfs_grid.cuh $(CSRC)/gk_internal.cuh $(CSRC)/gk_persistent.cuh $(CSRC)/gk_bfs_steps.cuh include/gk_bfs.h
NVFLAGS := -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
           -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -cudart static \
           -Xptxas -v -Iinclude
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS)) build/gk_expand.o

all: lib oracle host

lib: $(LIB)

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -dc -o $@ $< 2> build/$*.ptxas.txt || (cat build/$*.ptxas.txt; false)

# host expansion of the compact result transfer (AVX-512 by run-time dispatch)
build/gk_expand.o: $(CSRC)/gk_expand.cpp
	@mkdir -p build
	g++ -O3 -std=c++17 -fPIC -fvisibility=hidden -pthread -c -o $@ $<

$(LIB): $(OBJS)
	@mkdir -p $(PKG)/lib
	$(NVCC) -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
	    -Xcompiler -fPIC -o $@ $(OBJS)

oracle:
	$(MAKE) -C oracle

host: $(LIB)
	$(MAKE) -C $(PKG)/host

clean:
	rm -rf build $(PKG)/lib
	$(MAKE) -C oracle clean

.PHONY: all lib oracle host clean
