#!/bin/bash
# profiles/capture_r02.sh — round-2 profile captures (run on a B200 box:
#   gpurun --timeout 2400 -- "bash profiles/capture_r02.sh"); outputs land in gpurun_out/.
mkdir -p gpurun_out
B2="python bench.py --batch 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra-configs"
B32="python bench.py --batch 32 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra-configs"
# DRAM traffic of K1/K2/K3 at the benched batch (32): one step = 8 octaves
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum --clock-control none \
    -k regex:"blur_level2|detect_count|detect_emit|refine_kernel" --launch-skip 0 -c 200 --csv $B32 > gpurun_out/k12_traffic_b32.csv 2> gpurun_out/k12_b32.err
# launch list of one bench step at batch 8
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --batch 8 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra-configs > gpurun_out/all_launch.csv 2> gpurun_out/all.err
# full captures with source: the descriptor and the largest level blur
ncu --set full --import-source on --clock-control none -k regex:describe_stream -c 1 -o gpurun_out/r02_describe_stream $B2 > gpurun_out/ncu_desc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:blur_level2 --launch-skip 2 -c 1 -o gpurun_out/r02_blur_level $B2 > gpurun_out/ncu_blur.log 2>&1
ls -la gpurun_out
