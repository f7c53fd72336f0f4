#!/bin/bash
# Build a variant of libgi.so into tools/ab/libgi_<name>.so with extra nvcc flags.
# usage: bash tools/ab_build.sh NAME [-DFLAG=1 ...]
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
CS=$R/paper_1911_07260_b200/csrc
T=$(mktemp -d)
NV="nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -I $R/include $*"
$NV -DGI_BLOCK=512 -DGI_VARIANT=v512 -DGI_PRIMARY=1 -c $CS/gi_kernels.cu -o $T/k512.o
$NV -DGI_BLOCK=1024 -DGI_VARIANT=v1024 -DGI_PRIMARY=0 -c $CS/gi_kernels.cu -o $T/k1024.o
$NV -c $CS/gi_capi.cu -o $T/capi.o
$NV -c $CS/gi_kcore.cu -o $T/kcore.o
mkdir -p $R/tools/ab
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $R/tools/ab/libgi_$name.so $T/*.o
rm -rf $T
