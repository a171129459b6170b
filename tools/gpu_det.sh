#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_hex.py 2>&1 | tail -3
for c in 6 7; do for d in "" "--det"; do
timeout 300 python bench.py --config $c $d --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], 'CG %.2f GDOF/s' % d['value'], 'step %.4f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], d['roofline']['unit'], 'apply_only %.4f ms' % d['extra']['apply_only_ms'])"
done; done
