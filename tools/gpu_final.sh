#!/bin/bash
TAG=${1:-final}; OUT=gpurun_out/$TAG; mkdir -p $OUT
bash tools/gpu_tests.sh $TAG
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log; tail -2 $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; tail -c 600 $OUT/bench.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.json 2>&1; tail -c 300 $OUT/bench_ref.json
timeout 300 python bench.py --gpus 2 > $OUT/bench_g2.json 2>&1; tail -c 300 $OUT/bench_g2.json
