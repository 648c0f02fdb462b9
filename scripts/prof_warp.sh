#!/bin/bash
# fast P y in the z-marching warp: correctness (fast / FAST32 / parity tests) and C4 eval timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fast32.py tests/test_gpu_parity.py tests/test_gpu_slab_parity.py -x -q > gpurun_out/t_warp.log 2>&1; tail -3 gpurun_out/t_warp.log
for v in "" "MFREG_LIB_VARIANT=minb4" "MFREG_EXACT_PY=1"; do
  echo "== $v"; env $v timeout 300 python scripts/kbench.py 512 512 900 --h 0.7 0.7 0.7 --iters 8 2>&1 | tail -1
done
timeout 300 python scripts/kbench.py 512 512 900 --h 0.7 0.7 0.7 --iters 8 --mode fast32 2>&1 | tail -1
