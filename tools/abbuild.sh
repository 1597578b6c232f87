#!/bin/bash
# usage: abbuild.sh NAME "-DFOO=1 ..."   -> ablib/NAME.so
set -e
cd /root/repo
NAME=$1; shift
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -cudart static -Iinclude"
mkdir -p build/ab ablib
nvcc $F "$@" -dc -o build/ab/k_$NAME.o paper_1508_03619_b200/csrc/gk_bfs_kernel.cu
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -fPIC -o ablib/$NAME.so build/ab/k_$NAME.o build/gk_bfs_sharded.o build/gk_bc.o build/gk_aux.o build/gk_graph_build.o build/gk_capi.o build/gk_shard.o build/gk_sg.o
echo built ablib/$NAME.so
