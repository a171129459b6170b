#!/bin/bash
# final round-2 suite: GPU tests, smoke, every bench line, ncu launch list + captures, sweeps. Usage: bash tools/gpu_suite_r02h.sh TAG
TAG=${1:-r02h}; OUT=gpurun_out/$TAG; mkdir -p $OUT
bash tools/gpu_tests.sh $TAG > /dev/null 2>&1; tail -2 $OUT/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log; tail -2 $OUT/smoke.log
timeout 600 python tools/slab_sweep.py --out $OUT/slab_sweep.jsonl > /dev/null 2>&1
bash tools/run_bench_suite.sh $TAG
