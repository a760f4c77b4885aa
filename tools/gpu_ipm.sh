#!/bin/bash
# GPU parity + C4 bench + optional ncu full capture of ipm_step_kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload c4 --steps 10 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python -c "import json;d=json.load(open('gpurun_out/bench_c4.json'));print('c4', round(d['ms_per_step'],3),'ms', round(d['roofline']['frac'],3), d.get('e2e'), d.get('clocks'), d.get('status_nonzero'))"
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ipm_step -s 1 -c 1 \
      -o gpurun_out/prof_ipm python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ipm.log 2>&1
  tail -2 gpurun_out/ncu_ipm.log
fi
