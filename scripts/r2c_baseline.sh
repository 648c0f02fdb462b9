#!/bin/bash
# Round-2 session-3 baseline: GPU tests on the restored tree, kernel times at C4, source-level
# ncu of one k_hv2 and one k_ev2 launch (512x512x256, h=0.7) for the per-line instruction counts
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python scripts/kbench.py 512 512 900 --h 0.7 0.7 0.7 --iters 8 > gpurun_out/kb_c4.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_hv2|k_ev2|k_warp_z" -s 3 -c 3 \
    -o gpurun_out/src256 -f python scripts/kbench.py 512 512 256 --h 0.7 0.7 0.7 --iters 1 > gpurun_out/ncu_src.log 2>&1
tail -2 gpurun_out/ncu_src.log
