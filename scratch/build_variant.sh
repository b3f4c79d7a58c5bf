#!/bin/bash
# usage: scratch/build_variant.sh NAME "-DFLAG=.. -DFLAG2"  -> scratch/var/NAME/libedl_b200.so
set -e
name=$1; flags=$2
src=/root/repo/paper_1909_11985_b200/csrc
tmp=/tmp/var_$name
rm -rf $tmp; mkdir -p $tmp/pkg/csrc; cp $src/*.cu $src/*.cuh $src/*.cpp $src/*.hpp $src/Makefile $tmp/pkg/csrc/
mkdir -p $tmp/include; cp /root/repo/include/*.h $tmp/include/
cd $tmp/pkg/csrc && make -j8 NVCC="/usr/local/cuda/bin/nvcc -ccbin /usr/bin/g++ $flags" OUT=$tmp/libedl_b200.so >/dev/null 2>&1 || { echo "build $name failed"; exit 1; }
mkdir -p /root/repo/scratch/var/$name && cp $tmp/libedl_b200.so /root/repo/scratch/var/$name/
echo "built $name"
