#!/bin/bash
# full GPU suite + default bench + ncu full captures of the elasticity kernels (fused CG, fem_apply)
TAG=${1:-s2b}; OUT=gpurun_out/$TAG; mkdir -p $OUT
bash tools/gpu_tests.sh $TAG
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
tail -c 400 $OUT/bench.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elastic2_kernel -s 8 -c 1 \
  -o $OUT/prof_el_fused python bench.py --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_el.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elastic2_kernel -s 40 -c 1 \
  -o $OUT/prof_el_apply python bench.py --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_ela.log 2>&1
ls -la $OUT
