#!/bin/bash
for fl in "" "-DFEM_EL2_NOEMPTY=0" "-DFEM_EL2_HD=4"; do
  FEM_NVCC_FLAGS="$fl" python -c "from paper_2308_09839_b200 import build as B; B.build(force=True)" || exit 1
  echo "=== $fl"
  [ -z "$fl" ] && timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_loopback.py -k "elastic" 2>&1 | tail -1
  for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); x=d['extra']; print(d['config']['workload'], 'CG %.2f GDOF/s' % d['value'], 'step %.4f' % d['ms_per_step'], 'ev %.4f' % x['cg_iteration_ms_event_graph'], 'frac %.3f' % d['roofline']['frac'], 'apply %.4f' % x['apply_in_cg_ms'])"
  done
done
