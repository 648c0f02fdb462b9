#!/bin/bash
# Round-2 C4 evidence: bench (ours, reference arm), ncu launch list of the bench step, ncu --set full of the image passes
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 12 -c 24 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 2 --no-gn --no-cpu --no-fast32 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_hv2|k_ev2|k_warp_z" -s 3 -c 6 \
    -o gpurun_out/full_c4 -f python bench.py --steps 1 --warmup 1 --no-gn --no-cpu --no-fast32 > gpurun_out/ncu_full.log 2>&1
