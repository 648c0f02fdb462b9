#!/bin/bash
# hv3 bring-up: kernel-variant tests, C4 timings (hv3 tile heights vs hv2), ncu of one k_hv3 launch
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fast32.py -x -q > gpurun_out/t_kern.log 2>&1; tail -3 gpurun_out/t_kern.log
for v in "" "MFREG_LIB_VARIANT=oy8" "MFREG_NO_HV3=1"; do
  echo "== $v"; env $v timeout 300 python scripts/kbench.py 512 512 900 --h 0.7 0.7 0.7 --iters 8 2>&1 | tail -1
done
MFREG_LIB_VARIANT=oy8 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_hv3" -s 1 -c 1 \
    -o gpurun_out/hv3 -f python scripts/kbench.py 512 512 256 --h 0.7 0.7 0.7 --iters 1 > gpurun_out/ncu_hv3.log 2>&1
tail -1 gpurun_out/ncu_hv3.log
