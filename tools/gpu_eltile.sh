#!/bin/bash
# elasticity tile-height sweep: rebuild with -DFEM_EL_TY=<ty>, elastic CG parity test + C4 bench line.
# Usage: bash tools/gpu_eltile.sh TAG TY...
TAG=$1; shift; OUT=gpurun_out/$TAG; mkdir -p $OUT
for ty in "$@"; do
  FEM_NVCC_FLAGS="-DFEM_EL_TY=$ty" python -m paper_2308_09839_b200.build --force > $OUT/build_$ty.log 2>&1 || { tail $OUT/build_$ty.log; continue; }
  timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "elastic" > $OUT/pytest_$ty.log 2>&1; echo "ty=$ty pytest rc=$? $(tail -1 $OUT/pytest_$ty.log)"
  timeout 300 python bench.py --config 3 --no-cpu --no-e2e --no-csr > $OUT/bench_$ty.json 2> $OUT/bench_$ty.err
  python - $OUT/bench_$ty.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e=d['extra']
    print('  CG %.2f GDOF/s iter %.3f ms apply-in-CG %.3f ms apply-only %.3f ms (%.1f GDOF/s)'%(d['value'],d['ms_per_step'],e['apply_in_cg_ms'],e['apply_only_ms'],e['apply_only_gdofs']))
except Exception as ex: print('parse failed', ex)
PY
done
