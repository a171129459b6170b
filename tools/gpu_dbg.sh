#!/bin/bash
for f in 1 0; do
FEM_NVCC_FLAGS=-DFEM_RING_FENCE=$f python -c "from paper_2308_09839_b200 import build as B; B.build(force=True)"
echo "=== FEM_RING_FENCE=$f"
python tools/dbg_c3d.py vector 256 1 2>&1 | grep "^rep"
python tools/dbg_c3d.py vector 256 0 2>&1 | grep "^rep"
for c in 2 3; do python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], 'CG %.2f GDOF/s' % d['value'], 'frac %.3f' % d['roofline']['frac'], 'apply_only %.4f ms' % d['extra']['apply_only_ms'], d['extra'].get('apply_only_path'))"; done
done
