#!/bin/bash
# compute-sanitizer over the whole kernel set (tools/sanitize_workload.py).  Usage: bash tools/gpu_sanitize.sh TAG
TAG=${1:-san_r02}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_workload.py > $OUT/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize workload done' $OUT/$tool.log | tr '\n' ' ')"
done
