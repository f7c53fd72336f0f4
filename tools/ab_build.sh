#!/bin/bash
# Like ab_build.sh with separate flags per CTA width.
# usage: bash tools/ab_build.sh NAME "FLAGS_512" "FLAGS_1024" ["FLAGS_HOST"]
set -e
name=$1
R=$(cd "$(dirname "$0")/.." && pwd)
CS=$R/paper_1911_07260_b200/csrc
T=$(mktemp -d)
NV="nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -I $R/include"
$NV $2 -DGI_BLOCK=512 -DGI_VARIANT=v512 -DGI_PRIMARY=1 -c $CS/gi_kernels.cu -o $T/k512.o
$NV $3 -DGI_BLOCK=1024 -DGI_VARIANT=v1024 -DGI_PRIMARY=0 -c $CS/gi_kernels.cu -o $T/k1024.o
$NV $4 -c $CS/gi_capi.cu -o $T/capi.o
$NV $4 -c $CS/gi_kcore.cu -o $T/kcore.o
$NV $4 -c $CS/gi_probe.cu -o $T/probe.o
mkdir -p ${AB_OUT:-$R/tools/ab}
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ${AB_OUT:-$R/tools/ab}/libgi_$name.so $T/*.o
rm -rf $T
