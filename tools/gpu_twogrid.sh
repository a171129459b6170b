#!/bin/bash
# elasticity fused apply: interior / edge grids (FEM_EL2_TWOGRID) -- parity + C4 bench, both settings
for tg in 1 0; do
  FEM_NVCC_FLAGS="-DFEM_EL2_TWOGRID=$tg" python -c "from paper_2308_09839_b200 import build as B; B.build(force=True)" || exit 1
  echo "=== FEM_EL2_TWOGRID=$tg"
  if [ $tg = 1 ]; then
    timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_loopback.py tests/test_slab.py tests/test_gpu_gll.py -k "elastic" 2>&1 | tail -2
    timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_fullsize.py -k "fused_cg and 3" 2>&1 | tail -2
  fi
  for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], 'CG %.2f GDOF/s' % d['value'], 'step %.4f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'apply_in_cg %.4f ms' % d['extra']['apply_in_cg_ms'], 'apply_only %.4f ms frac %.3f' % (d['extra']['apply_only_ms'], d['extra']['apply_only_frac']))"
  done
done
