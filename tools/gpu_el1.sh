#!/bin/bash
# elastic1 (one cell row per thread, 16 warps) vs elastic2 (two rows, 8 warps): parity + C4 bench
for fl in "-DFEM_EL_CY=1" "-DFEM_EL_CY=1 -DFEM_EL1_SPLIT=0" "-DFEM_EL_CY=2"; do
  FEM_NVCC_FLAGS="$fl" python -c "from paper_2308_09839_b200 import build as B; B.build(force=True)" || exit 1
  echo "=== $fl"
  timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_parity.py -k "elastic" 2>&1 | tail -2
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], 'CG %.2f GDOF/s' % d['value'], 'frac %.3f' % d['roofline']['frac'], 'apply_in_cg %.4f ms' % d['extra']['apply_in_cg_ms'], 'apply_only %.4f ms frac %.3f' % (d['extra']['apply_only_ms'], d['extra']['apply_only_frac']), d['extra'].get('apply_only_path'))"
done
