#!/bin/bash
for h in 8 4; do
  FEM_NVCC_FLAGS="-DFEM_EL2_HD=$h" python -c "from paper_2308_09839_b200 import build as B; B.build(force=True)" || exit 1
  echo "=== FEM_EL2_HD=$h"
  [ $h = 8 ] && timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py -k "elastic" 2>&1 | tail -1
  for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); x=d['extra']; print(d['config']['workload'], 'CG %.2f GDOF/s' % d['value'], 'step %.4f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'apply_in_cg %.4f ms' % x['apply_in_cg_ms'], 'apply_only %.4f ms' % x['apply_only_ms'])"
  done
done
