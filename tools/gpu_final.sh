#!/bin/bash
# Round-end style GPU session: all GPU tests, smoke, every bench workload, ncu launch list of the
# default bench and full captures of the main kernels.  Output under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for w in c1 c3 c4 split c4solve pit; do
  timeout 900 python bench.py --workload $w --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 900 python bench.py --workload c5 --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launches.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:rr_fused_mma -s 1 -c 1 \
      -o gpurun_out/prof_c2 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2.log 2>&1
  timeout 900 ncu --set full --clock-control none -k regex:"rr_fused_mma|rr_solve_kernel|rr_residual_kernel" -s 3 -c 3 \
      -o gpurun_out/prof_split python bench.py --workload split --steps 1 --warmup 1 > gpurun_out/ncu_split.log 2>&1
  timeout 900 ncu --set full --clock-control none -k regex:ipm_step_kernel -s 1 -c 1 \
      -o gpurun_out/prof_c4 python bench.py --workload c4 --steps 1 --warmup 1 > gpurun_out/ncu_c4.log 2>&1
  timeout 900 ncu --set full --clock-control none -k regex:rr_cta_kernel -s 1 -c 1 \
      -o gpurun_out/prof_c3 python bench.py --workload c3 --steps 1 --warmup 1 --no-e2e > gpurun_out/ncu_c3.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log
tail -1 gpurun_out/smoke.log
for f in gpurun_out/bench_*.json; do echo "== $f"; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(d.get('metric','')[:60], d.get('value'), d.get('unit'), 'ms', round(d.get('ms_per_step') or 0, 3), 'frac', r.get('frac'))
" 2>&1 | tail -1; done
