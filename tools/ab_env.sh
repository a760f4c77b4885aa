#!/bin/bash
# A/B the bench over environment settings: tools/ab_env.sh "NAME1:VAR=x,VAR2=y" "NAME2:" ...
# Runs each setting twice, interleaved.  Output: gpurun_out/abe_<name>_<k>.json
mkdir -p gpurun_out
for k in 1 2; do
  for spec in "$@"; do
    name=${spec%%:*}; envs=${spec#*:}
    env $(echo "$envs" | tr ',' ' ') timeout 300 python bench.py --steps ${STEPS:-10} --no-cpu-baseline --no-e2e --no-others ${BENCH_ARGS:-} \
      > gpurun_out/abe_${name}_$k.json 2> gpurun_out/abe_${name}_$k.err
    python - "$name" "$k" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/abe_%s_%s.json" % (sys.argv[1], sys.argv[2])).read().strip().splitlines()[-1])
    r = d.get("roofline", {})
    print("%-12s run%s  %.3f ms/step  frac %.4f  clocks %s" % (sys.argv[1], sys.argv[2], d["ms_per_step"], r.get("frac", 0), d.get("clocks", {}).get("sm_mhz")))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
  done
done
