#!/bin/bash
# Round-2 evidence on one B200: gpu tests, bench (ours + reference arm), ncu launch list of the
# bench step and ncu --set full of the three image passes at C4, fp64 peak, C5 sweep, C4 GN trace
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 12 -c 24 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 2 --no-gn --no-cpu --no-fast32 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_hv2|k_ev2|k_warp_z" -s 3 -c 6 \
    -o gpurun_out/full_c4 -f python bench.py --steps 1 --warmup 1 --no-gn --no-cpu --no-fast32 > gpurun_out/ncu_full.log 2>&1
./scripts/probe/fp64_peak > gpurun_out/fp64_peak.json 2>&1 || (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak scripts/probe/fp64_peak.cu && /tmp/fp64_peak > gpurun_out/fp64_peak.json)
timeout 600 python scripts/c5_sweep.py > gpurun_out/c5.txt 2>&1
MFREG_TRACE_TIME=1 timeout 600 python scripts/c4_reg.py > gpurun_out/c4_trace.txt 2>&1
