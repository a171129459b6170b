#!/bin/bash
for fl in "-DFEM_LAP_TY1=16 -DFEM_LAP_MINB=1" "-DFEM_LAP_TY1=16 -DFEM_LAP_MINB=1 -DFEM_LAP_S1=8" "-DFEM_LAP_TY1=4" ""; do
  FEM_NVCC_FLAGS="$fl" python -c "from paper_2308_09839_b200 import build as B; B.build(force=True)" 2>&1 | tail -2
  for c in 1; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/tmp/e.txt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); x=d['extra']; print('$fl', d['config']['workload'], 'CG %.2f' % d['value'], 'step %.4f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'apply %.4f' % x['apply_in_cg_ms'], 'aonly %.4f %.3f' % (x['apply_only_ms'], x['apply_only_frac']))" || tail -3 /tmp/e.txt
  done
done
