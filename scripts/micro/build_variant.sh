#!/bin/bash
# usage: build_variant.sh <persist.cu variant> <out .so>   (other objects from build/nmfb200)
set -e
cd /root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I paper_2101_08431_b200/csrc -I include -c "$1" -o /tmp/variant_persist.o
objs=$(ls build/nmfb200/*.o | grep -v persist.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$2" $objs /tmp/variant_persist.o -lcudart
