#!/bin/bash
# Dot-implementation ablation: fused CG with dots in the producing kernels' epilogue,
# separate dot kernels, atomic CTA partials, and single-reduction CG-CG, at C2, C4 and 64^3.
# Usage (under gpurun): bash tools/gpu_dot_ablation.sh TAG
TAG=${1:-dot}; OUT=gpurun_out/$TAG; mkdir -p $OUT
for spec in "1" "3" "1 --n 64" "3 --n 64"; do
  set -- $spec; c=$1; shift
  tag="c$c$(echo $@ | tr -d ' -')"
  for d in fused separate atomic cgcg; do
    if [ $d = cgcg ]; then flag="--cgcg"; else flag="--dot $d"; fi
    timeout 300 python bench.py --config $c $@ $flag --steps 48 --warmup 5 --no-cpu --no-e2e --no-csr \
      > $OUT/dot_${tag}_$d.json 2> $OUT/dot_${tag}_$d.err
    python - $OUT/dot_${tag}_$d.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); e=d['extra']
    print('%-28s CG %7.2f GDOF/s  iter %.4f ms  apply %.4f ms'%(d['config']['workload'], d['value'], d['ms_per_step'], e['apply_in_cg_ms']))
except Exception as ex: print(sys.argv[1], 'parse failed', ex)
PY
  done
done
