#!/bin/bash
# Round evidence on one B200: gpu tests, bench (ours + reference arm), ncu launch list, ncu --set full
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 60 -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-gn --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_hv2|k_ev2|k_warp_fast|k_nodal" -s 10 -c 5 \
    -o gpurun_out/full -f python bench.py --steps 2 --warmup 3 --no-gn --no-cpu > /dev/null 2>&1
# C4 finest-level launch list (one eval + a 4-iteration CG) and the C5 1024^3 derivative sweep
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/c4_launches.py > /dev/null 2>&1
timeout 600 python scripts/c5_sweep.py > gpurun_out/c5.txt 2>&1
MFREG_TRACE_TIME=1 timeout 600 python scripts/c4_reg.py > gpurun_out/c4_trace.txt 2>&1
