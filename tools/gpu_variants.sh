#!/bin/bash
# build-flag sweep: for each quoted flag set, rebuild, run the GPU parity tests (-k filter) and
# bench lines for the given configs.  Usage: bash tools/gpu_variants.sh TAG "CONFIGS" "K" "FLAGS1" "FLAGS2" ...
TAG=$1; CONFIGS=$2; K=$3; shift 3; OUT=gpurun_out/$TAG; mkdir -p $OUT
n=0
for flags in "$@"; do
  n=$((n+1))
  FEM_NVCC_FLAGS="$flags" python -m paper_2308_09839_b200.build --force > $OUT/build_$n.log 2>&1 || { echo "[$flags] build failed"; tail -5 $OUT/build_$n.log; continue; }
  timeout 400 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest_$n.log 2>&1; echo "[$flags] pytest rc=$? $(tail -1 $OUT/pytest_$n.log)"
  for c in $CONFIGS; do
    timeout 300 python bench.py --config $c --no-cpu --no-e2e --no-csr > $OUT/bench_${n}_c$c.json 2> $OUT/bench_${n}_c$c.err
    python - $OUT/bench_${n}_c$c.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e=d['extra']
    print('   %-16s CG %.2f GDOF/s iter %.3f ms apply-in-CG %.3f ms (frac %.3f) apply-only %.3f ms'%(d['config']['workload'], d['value'], d['ms_per_step'], e['apply_in_cg_ms'], d['roofline']['frac'], e['apply_only_ms']))
except Exception as ex: print('   parse failed', ex)
PY
  done
done
python -m paper_2308_09839_b200.build --force > /dev/null 2>&1
