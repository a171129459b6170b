#!/bin/bash
# paired x update: tests + C4 / C2 / C3 bench with x_pairs 0 / 1. Usage: bash tools/gpu_xdefer.sh TAG
TAG=${1:-xp}; OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 900 python -m pytest -m gpu -q -x tests/test_gpu_xdefer.py tests/test_loopback.py tests/test_gpu_parity.py > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
for c in 3 1 2; do for xp in 1 4 8; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-csr --no-e2e --x-defer $xp > $OUT/b_c${c}_xp$xp.json 2> $OUT/b_c${c}_xp$xp.err
  python - $OUT/b_c${c}_xp$xp.json <<'P'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e=d.get('extra',{})
print(sys.argv[1], round(d['value'],2), round(d['ms_per_step'],4), 'apply', round(e.get('apply_in_cg_ms',0),4), 'frac', round(d['roofline']['frac'],3), 'B/DOF', round(e.get('cg_bytes_per_dof_alg',0),2), 'gbs', round(e.get('cg_iteration_gbs',0)))
P
done; done
