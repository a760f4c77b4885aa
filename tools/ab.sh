#!/bin/bash
# A/B the C2 bench over library variants: tools/ab.sh name1 name2 ... (paper_2509_16370_b200/librr_b200_<name>.so,
# "cur" = librr_b200.so).  Runs each variant twice, interleaved.  Output: gpurun_out/ab_<name>_<k>.json
mkdir -p gpurun_out
for k in 1 2; do
  for v in "$@"; do
    if [ "$v" = cur ]; then L=paper_2509_16370_b200/librr_b200.so; else L=paper_2509_16370_b200/librr_b200_$v.so; fi
    RR_B200_LIB=$PWD/$L timeout 300 python bench.py --steps ${STEPS:-10} --no-cpu-baseline --no-e2e --no-others ${BENCH_ARGS:-} \
      > gpurun_out/ab_${v}_$k.json 2> gpurun_out/ab_${v}_$k.err
    python - "$v" "$k" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/ab_%s_%s.json" % (sys.argv[1], sys.argv[2])).read().strip().splitlines()[-1])
    r = d.get("roofline", {})
    print("%-10s run%s  %.3f ms/step  frac %.4f  clocks %s" % (sys.argv[1], sys.argv[2], d["ms_per_step"], r.get("frac", 0), d.get("clocks", {}).get("sm_mhz")))
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
  done
done
