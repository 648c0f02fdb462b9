#!/bin/bash
# Round-2 session-4 evidence, one B200: ncu capture of the C4 bench step for the current sources
# (-> profiles/traffic.json), SASS mixes, GPU tests, bench (ours + reference arm), C4 launch list,
# host-pipeline timeline, C5 sweep, C4 GN trace
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_hv2|k_ev2|k_warp_z" -s 3 -c 3 \
    -o gpurun_out/full_c4 -f python bench.py --steps 1 --warmup 1 --no-gn --no-cpu --no-fast32 > gpurun_out/ncu_full.log 2>&1
python scripts/ncu_traffic.py c4 gpurun_out/full_c4.ncu-rep > gpurun_out/traffic.txt 2>&1; cp profiles/traffic.json gpurun_out/ 2>/dev/null
for k in k_warp_z k_ev2 k_hv2; do
  ncu -i gpurun_out/full_c4.ncu-rep -k regex:$k --page source --csv --print-source sass > gpurun_out/src_$k.csv 2>/dev/null
  python scripts/sass_mix.py gpurun_out/src_$k.csv 235929600 > gpurun_out/mix_$k.txt 2>&1
done
ncu -i gpurun_out/full_c4.ncu-rep --page raw --csv > gpurun_out/full_raw.csv 2>/dev/null
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 12 -c 24 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 2 --no-gn --no-cpu --no-fast32 > /dev/null 2>&1
MFREG_PIPE_TRACE=1 timeout 300 python scripts/pipe_probe.py > gpurun_out/pipe_probe.txt 2>&1
timeout 900 python scripts/c5_sweep.py > gpurun_out/c5.txt 2>&1
MFREG_TRACE_TIME=1 timeout 900 python scripts/c4_reg.py > gpurun_out/c4_trace.txt 2>&1
tail -2 gpurun_out/gpu_tests.log; tail -1 gpurun_out/bench.log | cut -c1-300
