#!/bin/bash
# ncu --set full of one Hv launch (k_hv2) at a given size
out=$1; shift
ncu --set full --import-source on --clock-control none -k regex:"k_hv2|k_fused" -s 2 -c 2 \
    -o gpurun_out/$out -f python scripts/kbench.py $@ --iters 1 > gpurun_out/$out.log 2>&1
