#!/bin/bash
# compute-sanitizer over small launches of every kernel; summaries into gpurun_out/sanitizer_*.txt
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/san_cases.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Error" gpurun_out/sanitizer_$tool.txt | head -5
done
