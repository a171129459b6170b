#!/bin/bash
# A/B: working-tree kernels (CG scalars loaded up front) vs HEAD's
OUT=gpurun_out/ab2; mkdir -p $OUT; C=paper_2308_09839_b200/csrc
bench() { for c in 1 2 3 4 5; do timeout 300 python bench.py --config $c --no-cpu --no-e2e --no-csr 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['extra']; print('  ', d['config']['workload'], 'CG %.2f' % d['value'], 'iter %.4f' % d['ms_per_step'], 'apply %.4f frac %.3f' % (e['apply_in_cg_ms'], d['roofline']['frac']), 'aonly %.4f' % e['apply_only_ms'])"; done; }
python -m paper_2308_09839_b200.build --force > $OUT/b1.log 2>&1 || { tail $OUT/b1.log; exit 1; }
echo "=== new"; timeout 1200 python -m pytest -q -m gpu tests 2>&1 | tail -2; bench
for f in kernels_elastic.cu kernels_laplace.cu; do cp $C/$f /tmp/new_$f; cp gpurun_tmp_old/$f $C/; done
python -m paper_2308_09839_b200.build --force > $OUT/b2.log 2>&1; echo "=== old"; bench
for f in kernels_elastic.cu kernels_laplace.cu; do cp /tmp/new_$f $C/$f; done
python -m paper_2308_09839_b200.build --force > /dev/null 2>&1; echo "=== new again"; bench
