#!/bin/bash
# C3 parity subset + bench + optional ncu full capture of rr_cta_kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "64-32 or 32-16 or 24-8 or c3" > gpurun_out/pytest_c3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c3.log
tail -2 gpurun_out/pytest_c3.log
timeout 600 python bench.py --workload c3 --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python -c "import json;d=json.load(open('gpurun_out/bench_c3.json'));print('c3', round(d['ms_per_step'],3),'ms', round(d['roofline']['frac'],3), d.get('clocks'))"
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:rr_cta -s 1 -c 1 \
      -o gpurun_out/prof_c3 python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3.log 2>&1
  tail -2 gpurun_out/ncu_c3.log
fi
