#!/bin/bash
# profiles/capture_r02b.sh — round-2 evidence on the final kernels (run on a B200 box:
#   gpurun --timeout 3000 -- "bash profiles/capture_r02b.sh"); outputs land in gpurun_out/.
mkdir -p gpurun_out
B2="python bench.py --batch 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-extra-configs"
B32="python bench.py --batch 32 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-extra-configs"
# the GPU suite, then the bench line (all legs), both outside any profiler
(timeout 1200 python -m pytest tests -m gpu -x -q 2>&1; echo "rc=$?") > gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
# per-launch DRAM bytes / time / FP64 and issue utilisation of K1-K3 at the benched batch (32)
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum \
    --clock-control none -k regex:"blur|detect_count|detect_emit|refine_kernel" -c 60 --csv $B32 > gpurun_out/r02_k123_b32.csv 2> gpurun_out/r02_k123.err
# launch list of one bench step at batch 8 (every kernel, cold, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --batch 8 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-extra-configs > gpurun_out/r02_launches_b8.csv 2> gpurun_out/r02_launches.err
# full captures with source: the descriptor, the upsampled bridge, the largest level blur, extrema count
ncu --set full --import-source on --clock-control none -k regex:describe_stream -c 1 -o gpurun_out/r02_describe_stream -f $B2 > gpurun_out/ncu_desc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:blur_level2 -c 1 -o gpurun_out/r02_bridge -f $B2 > gpurun_out/ncu_bridge.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:blur_strip --launch-skip 4 -c 1 -o gpurun_out/r02_blur_strip_r13 -f $B2 > gpurun_out/ncu_blur.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:detect_count -c 1 -o gpurun_out/r02_detect_count -f $B2 > gpurun_out/ncu_det.log 2>&1
ls -la gpurun_out
