#!/bin/bash
# usage: [SRC=gk_bfs_cluster] abbuild.sh NAME "-DFOO=1 ..."   -> ablib/NAME.so
# Rebuilds csrc/$SRC.cu (default gk_bfs_kernel) with the extra flags and links
# it with the other objects of the last `make lib`.
set -e
cd /root/repo
NAME=$1; shift
SRC=${SRC:-gk_bfs_kernel}
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -cudart static -Iinclude"
mkdir -p build/ab ablib
nvcc $F "$@" -dc -o build/ab/${SRC}_$NAME.o paper_1508_03619_b200/csrc/$SRC.cu
OTHERS=$(ls build/*.o | grep -v "build/$SRC.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -fPIC -o ablib/$NAME.so build/ab/${SRC}_$NAME.o $OTHERS
echo built ablib/$NAME.so
