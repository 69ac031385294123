#!/bin/bash
# profiles/capture.sh — the commands that produced this round's profiles (run on a B200 box:
#   gpurun --timeout 2400 -- "bash profiles/capture.sh"), outputs land in gpurun_out/.
mkdir -p gpurun_out
B="python bench.py --batch 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra-configs"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"blur_level2|detect_count|detect_emit|refine_kernel" -c 44 --csv $B > gpurun_out/k12_traffic.csv 2> gpurun_out/k12.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --batch 8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/all_launch.csv 2> gpurun_out/all.err
ncu --set full --import-source on --clock-control none -k regex:describe_stream -c 1 -o gpurun_out/r01_describe_stream_final $B > gpurun_out/ncu_desc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"detect_count" -c 1 -o gpurun_out/r01_detect_count_tma $B > gpurun_out/ncu_det.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err
ls -la gpurun_out
