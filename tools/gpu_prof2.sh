#!/bin/bash
# ncu captures of the CG-mode (TMA path) apply kernels: skip warm-up launches, capture 1.
TAG=${1:-prof}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elastic2_kernel -s 6 -c 1 \
  -o $OUT/prof_elastic python bench.py --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_el.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:laplace_kernel -s 6 -c 1 \
  -o $OUT/prof_lap1 python bench.py --config 1 --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_l1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:laplace_kernel -s 6 -c 1 \
  -o $OUT/prof_lap3 python bench.py --config 2 --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_l3.log 2>&1
ls $OUT
