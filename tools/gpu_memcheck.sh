#!/bin/bash
# one compute-sanitizer tool per gpurun call (B200_PROFILING.md).  Usage: bash tools/gpu_memcheck.sh TAG [tool]
TAG=${1:-memcheck}; TOOL=${2:-memcheck}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 600 python tools/sanitize_workload.py > $OUT/plain.log 2>&1 || { echo "plain run failed"; tail $OUT/plain.log; exit 1; }
timeout 1200 compute-sanitizer --tool $TOOL --print-limit 20 python tools/sanitize_workload.py > $OUT/$TOOL.log 2>&1
echo "$TOOL rc=$? $(grep -E 'ERROR SUMMARY|sanitize workload done' $OUT/$TOOL.log | tr '\n' ' ')"
