#!/bin/bash
for fl in "" "-DFEM_UPD_MINB=3" "-DFEM_UPD_MINB=4"; do
  FEM_NVCC_FLAGS="$fl" python -c "from paper_2308_09839_b200 import build as B; B.build(force=True)" || exit 1
  echo "=== $fl"
  for c in 3 1; do for i in 1 2; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); x=d['extra']; print(d['config']['workload'], 'CG %.2f' % d['value'], 'step %.4f' % d['ms_per_step'], 'apply %.4f' % x['apply_in_cg_ms'], 'upd~ %.4f' % (d['ms_per_step'] - x['apply_in_cg_ms']))"
  done; done
done
