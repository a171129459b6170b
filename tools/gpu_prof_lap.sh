#!/bin/bash
# ncu capture of the fused (CG mode 2) Laplace apply.  Usage: bash tools/gpu_prof_lap.sh TAG [config]
TAG=${1:-lapprof}; CFG=${2:-1}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:laplace_kernel -s 6 -c 1 \
  -o $OUT/prof_lap_c$CFG python bench.py --config $CFG --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu.log 2>&1
ls $OUT
