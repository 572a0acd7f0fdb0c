#!/bin/bash
# build_variant.sh <name> <git-rev> <file.cu> [extra nvcc flags]: libdsp_<name>.so = current objects
# with <file.cu> taken from <git-rev> (same-box A/B timing via DSP_LIB_OVERRIDE)
set -e
name=$1; rev=$2; f=$3; shift 3
mkdir -p /tmp/variants
git show $rev:paper_2403_10266_b200/csrc/$f > /tmp/variants/$f
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
     -Ipaper_2403_10266_b200/csrc "$@" -c /tmp/variants/$f -o /tmp/variants/$name.o
objs=$(ls build/dsp/*.o | grep -v "/${f}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2403_10266_b200/libdsp_$name.so $objs /tmp/variants/$name.o -cudart static -ldl -lpthread
echo built paper_2403_10266_b200/libdsp_$name.so
