#!/bin/bash
# One GPU session: parity tests, smoke, bench for C2 (default), C3, C4. Output under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for w in ${EXTRA_WORKLOADS:-c3 c4}; do
  timeout 900 python bench.py --workload $w --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
tail -3 gpurun_out/pytest_gpu.log
tail -2 gpurun_out/smoke.log
cat gpurun_out/bench_*.json; for f in gpurun_out/bench_*.err; do tail -n 3 $f; done
