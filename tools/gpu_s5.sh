#!/bin/bash
for fl in "-DFEM_EL2_S=5" "" "-DFEM_LAP_S1=6" "-DFEM_LAP_S1=5"; do
  FEM_NVCC_FLAGS="$fl" python -c "from paper_2308_09839_b200 import build as B; B.build(force=True)" || exit 1
  echo "=== $fl"
  [ -n "$fl" ] && timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py 2>&1 | tail -1
  for c in 3 5 1; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); x=d['extra']; print(d['config']['workload'], 'CG %.2f' % d['value'], 'step %.4f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'apply %.4f' % x['apply_in_cg_ms'], 'aonly %.4f ms %.3f' % (x['apply_only_ms'], x['apply_only_frac']))"
  done
done
