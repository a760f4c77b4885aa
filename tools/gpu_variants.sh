#!/bin/bash
# parity tests + bench per kernel variant; optional ncu full capture of the default variant
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-0 1 2}; do
  RR_B200_VARIANT=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_v$v.json 2> gpurun_out/bench_v$v.err
  python -c "import json;d=json.load(open('gpurun_out/bench_v$v.json'));print('variant $v', round(d['ms_per_step'],3),'ms', round(d['roofline']['frac'],3), d['clocks'])"
done
if [ -n "$NCU" ]; then
  RR_B200_VARIANT=${NCU_VARIANT:-0} timeout 900 ncu --set full --clock-control none --import-source on -k regex:rr_fused -s 1 -c 1 \
      -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
  tail -2 gpurun_out/ncu_full.log
fi
