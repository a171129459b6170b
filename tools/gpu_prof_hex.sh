#!/bin/bash
# ncu capture of the general-hex apply kernel (bench config 6 / 7).  Usage: bash tools/gpu_prof_hex.sh TAG [config]
TAG=${1:-hexprof}; CFG=${2:-6}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hex_apply -s 4 -c 1 \
  -o $OUT/prof_hex_c$CFG python bench.py --config $CFG --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu.log 2>&1
ls $OUT
