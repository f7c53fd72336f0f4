#!/bin/bash
# registers / spills of the persistent kernels per CTA width: bash tools/ptxas_summary.sh [extra nvcc flags]
R=$(cd "$(dirname "$0")/.." && pwd)
for B in 512 1024; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xptxas=-v -Xcompiler -fPIC -I $R/include \
    -DGI_BLOCK=$B -DGI_VARIANT=v$B -DGI_PRIMARY=$([ $B = 512 ] && echo 1 || echo 0) "$@" -c $R/paper_1911_07260_b200/csrc/gi_kernels.cu -o /tmp/ps_$B.o 2>&1 |
  awk -v B=$B '/Compiling entry function/ {f=$0; sub(/.*sssp_persistentILi/, "", f); sub(/E.*/, "", f); if ($0 !~ /sssp_persistent/) f=""}
       /spill stores/ && f!="" {sp=$5" "$6" "$9" "$10}
       /Used [0-9]+ registers/ && f!="" {print "block " B " kind " f ": " $5 " regs, spill st/ld " sp; f=""}'
done
