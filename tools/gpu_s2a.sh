#!/bin/bash
# round-2 session-2 baseline: full GPU suite + default bench + smoke
TAG=s2a; OUT=gpurun_out/$TAG; mkdir -p $OUT
bash tools/gpu_tests.sh $TAG
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -c 1500 $OUT/bench.json; tail -3 $OUT/bench.err; tail -2 $OUT/smoke.log
