#!/bin/bash
# ncu --set full of the fused kernels + k_warp_fast at a given size (one launch each)
# usage: scripts/prof_full.sh OUTNAME MX MY MZ
out=${1:-full}; shift
ncu --set full --import-source on --clock-control none -k regex:"k_fused|k_hv2|k_ev2|k_warp_fast|k_nodal" -s 8 -c 5 \
    -o gpurun_out/$out -f python scripts/kbench.py ${@:-128 128 128} --iters 2 > gpurun_out/$out.log 2>&1
