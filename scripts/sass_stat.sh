#!/bin/bash
# static SASS statistics of one kernel source (cross-compiled for sm_100a): size, moves, spills
f=${1:-paper_1804_10541_b200/csrc/hv_fast.cu}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Xptxas -O3,-v \
  --expt-relaxed-constexpr -c $f -o /tmp/sass_stat.o 2>&1 | grep -E "spill|Used" | sed 's/ptxas info    ://'
cuobjdump -sass /tmp/sass_stat.o | grep -E "^\s+/\*[0-9a-f]{4}\*/" > /tmp/sass_stat.txt
echo "instr $(wc -l < /tmp/sass_stat.txt)  mov $(grep -cE 'MOV' /tmp/sass_stat.txt)  dfp $(grep -cE 'DADD|DMUL|DFMA' /tmp/sass_stat.txt)  lds $(grep -c 'LDS' /tmp/sass_stat.txt)  shfl $(grep -c SHFL /tmp/sass_stat.txt)"
