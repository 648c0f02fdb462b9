#!/bin/bash
# uniform-warp Hv pass on the stored coefficients (MFREG_HV4=1): correctness, C4 timings vs k_hv2, ncu
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fast32.py -x -q > gpurun_out/t_hv4.log 2>&1; tail -3 gpurun_out/t_hv4.log
for v in "MFREG_HV4=1" "MFREG_HV4=0"; do
  echo "== $v"; env $v timeout 300 python scripts/kbench.py 512 512 900 --h 0.7 0.7 0.7 --iters 8 2>&1 | tail -1
  env $v timeout 300 python scripts/kbench.py 512 512 900 --h 0.7 0.7 0.7 --iters 8 --mode fast32 2>&1 | tail -1
done
MFREG_HV4=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_hv3" -s 1 -c 1 \
    -o gpurun_out/hv4 -f python scripts/kbench.py 512 512 256 --h 0.7 0.7 0.7 --iters 1 > gpurun_out/ncu_hv4.log 2>&1
tail -1 gpurun_out/ncu_hv4.log
