#!/bin/bash
# ncu captures of the fem_apply kernels on caller vectors (row-pair staging) at C4 and C2.
# Usage: bash tools/gpu_prof_apply.sh TAG
TAG=${1:-profapply}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
# launches 0-5 of elastic2 are the fused CG applies (3 warm-up + 3 timed), then 3 + 10 apply-only
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elastic2_kernel -s 9 -c 1 \
  -o $OUT/prof_apply_c4 python bench.py --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:laplace_kernel -s 9 -c 1 \
  -o $OUT/prof_apply_c2 python bench.py --config 1 --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_c2.log 2>&1
ls $OUT
