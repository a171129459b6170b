#!/bin/bash
# quick GPU iteration: build, parity tests, bench lines (no ncu). Usage: bash tools/gpu_quick.sh TAG [pytest-args]
TAG=${1:-quick}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 420 python -m pytest tests -m gpu -x -q ${@} > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -15 $OUT/pytest.log
for c in 1 2 3; do
  timeout 300 python bench.py --config $c --no-cpu --no-e2e --no-csr > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
  python - $OUT/bench_c$c.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    e=d['extra']
    print(d['config']['workload'], 'CG %.1f GDOF/s'%d['value'], 'apply-only %.1f GDOF/s %.3f ms'%(e['apply_only_gdofs'],e['apply_only_ms']), 'apply-in-CG frac %.3f'%d['roofline']['frac'], 'iter %.3f ms'%d['ms_per_step'])
except Exception as ex: print('bench parse failed', ex, open(sys.argv[1]).read()[-500:])
PY
done
