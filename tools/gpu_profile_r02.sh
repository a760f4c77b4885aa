#!/bin/bash
# Round-2 profiling pass: ncu launch list of the default bench command (C2), one `ncu --set full`
# capture per headline kernel (C2 fused, C4 ipm_step, C3 CTA, split factor/solve/residual).
# Reports land in gpurun_out/ (scratch); summaries are written into profiles/ by tools/*.py here.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-others > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rr_fused_mma -s 1 -c 1 \
    -o gpurun_out/prof_c2_r02 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-others > gpurun_out/ncu_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ipm_step -s 1 -c 1 \
    -o gpurun_out/prof_c4_r02 python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rr_cta -s 1 -c 1 \
    -o gpurun_out/prof_c3_r02 python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-others > gpurun_out/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"rr_fused_mma|rr_solve_kernel|rr_residual" -s 3 -c 3 \
    -o gpurun_out/prof_split_r02 python bench.py --workload split --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_split.log 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches_r02.csv
