#!/bin/bash
# usage: build_variant.sh <variant .cu> <object name it replaces, e.g. persist.o> <out .so>
set -e
cd /root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I paper_2101_08431_b200/csrc -I include -c "$1" -o /tmp/variant_obj.o
objs=$(ls build/nmfb200/*.o | grep -v "/$2\$")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$3" $objs /tmp/variant_obj.o -lcudart
