#!/bin/bash
python -c "from paper_2308_09839_b200 import build as B; B.build()" || exit 1
timeout 1200 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_loopback.py tests/test_slab.py tests/test_gpu_gll.py -k "elastic" 2>&1 | tail -2
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_fullsize.py -k "fused_cg" 2>&1 | tail -2
for d in 1 0 1 0; do
  timeout 300 python bench.py --delay-x $d --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/tmp/e.txt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); x=d['extra']; print(d['config']['workload'], 'dx', x['delay_x'], 'CG %.2f GDOF/s' % d['value'], 'step %.4f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'apply_in_cg %.4f ms' % x['apply_in_cg_ms'], 'launches', d['gpu_launches'])" || tail -3 /tmp/e.txt
done
timeout 300 python bench.py --config 5 --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu 2>/tmp/e.txt | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); x=d['extra']; print(d['config']['workload'], 'dx', x['delay_x'], 'CG %.2f GDOF/s' % d['value'], 'step %.4f' % d['ms_per_step'], 'frac %.3f' % d['roofline']['frac'])"
timeout 900 compute-sanitizer --tool synccheck --print-limit 5 python tools/sanitize_workload.py 2>&1 | grep -E "ERROR SUMMARY|done|Barrier error" | head -5
timeout 900 compute-sanitizer --tool initcheck --print-limit 5 python tools/sanitize_workload.py 2>&1 | grep -E "ERROR SUMMARY|done" | head -3
