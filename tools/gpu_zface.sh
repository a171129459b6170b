#!/bin/bash
for z in 1 0; do
  FEM_NVCC_FLAGS="-DFEM_EL2_ZFACE=$z" python -c "from paper_2308_09839_b200 import build as B; B.build(force=True)" || exit 1
  echo "=== FEM_EL2_ZFACE=$z"
  [ $z = 1 ] && timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_loopback.py tests/test_slab.py tests/test_gpu_gll.py -k "elastic" 2>&1 | tail -1
  [ $z = 1 ] && timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_fullsize.py -k "3 or 5" 2>&1 | tail -1
  for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], 'CG %.2f GDOF/s' % d['value'], 'step %.4f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'apply_in_cg %.4f ms' % d['extra']['apply_in_cg_ms'], 'apply_only %.4f ms frac %.3f' % (d['extra']['apply_only_ms'], d['extra']['apply_only_frac']))"
  done
done
python -c "from paper_2308_09839_b200 import build as B; B.build(force=True)"
timeout 300 python bench.py --config 0 --no-cpu --no-csr 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], 'CG %.4f GDOF/s' % d['value'], 'step %.5f' % d['ms_per_step'], 'e2e %.4f' % d['e2e']['value'])"
timeout 1200 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_loopback.py tests/test_gpu_hex.py 2>&1 | tail -1
