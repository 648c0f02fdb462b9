#!/bin/bash
# one build -> measure iteration: kernel tests (fast / FAST32 / parity / slabs) + C4 kernel times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fast32.py tests/test_gpu_parity.py -x -q > gpurun_out/it_tests.log 2>&1; echo "rc=$?" >> gpurun_out/it_tests.log
tail -3 gpurun_out/it_tests.log
for v in "" $MFREG_VARIANTS; do
  echo "== variant '$v'"; MFREG_LIB_VARIANT=$v timeout 300 python scripts/kbench.py 512 512 900 --h 0.7 0.7 0.7 --iters 8 2>&1 | tail -1
  MFREG_LIB_VARIANT=$v timeout 300 python scripts/kbench.py 512 512 900 --h 0.7 0.7 0.7 --iters 8 --mode fast32 2>&1 | tail -1
done
if [ -n "$NCU_K" ]; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$NCU_K" -s 1 -c 1 \
      -o gpurun_out/it_src -f python scripts/kbench.py 512 512 256 --h 0.7 0.7 0.7 --iters 1 > gpurun_out/it_ncu.log 2>&1
  tail -1 gpurun_out/it_ncu.log
fi
