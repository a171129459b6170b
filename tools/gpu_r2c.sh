#!/bin/bash
TAG=r2c; OUT=gpurun_out/$TAG; mkdir -p $OUT
bash tools/gpu_tests.sh $TAG -x tests
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-csr > $OUT/bench_c4.json 2> $OUT/bench_c4.err
python -c "
import json; d=json.loads(open('$OUT/bench_c4.json').read().strip().splitlines()[-1]); e=d['extra']
print('C4', d['value'], d['roofline']['frac'], e['apply_in_cg_ms'], e['apply_only_ms'], e['apply_only_frac'], d['e2e']['value'])"
bash tools/gpu_dot_ablation.sh $TAG
