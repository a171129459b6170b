#!/bin/bash
TAG=${1:-s2c}; OUT=gpurun_out/$TAG; mkdir -p $OUT
bash tools/gpu_tests.sh $TAG
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], 'CG %.2f GDOF/s' % d['value'], 'step %.4f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'apply_in_cg %.4f ms' % d['extra']['apply_in_cg_ms'], 'apply_only %.4f ms frac %.3f' % (d['extra']['apply_only_ms'], d['extra']['apply_only_frac']))"
done
