#!/bin/bash
# per-kernel device times (ncu launch list) of one bench step: k_warp*, k_fused*, k_nodal*
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_warp|k_nodal|k_fused" -c ${1:-10} python bench.py --steps 2 --warmup 2 --no-gn --no-cpu 2>/dev/null | grep -E "^  [a-z]|k_warp|k_nodal|k_fused|gpu__time" | grep -E "k_|gpu__time" | paste - - | sed -E 's/\(.*gpu__time_duration.sum//' | awk '{print $1, $2, $NF}'
