#!/bin/bash
# GPU iteration: build, full -m gpu suite, bench lines. Usage: bash tools/gpu_check.sh TAG [pytest-args]
TAG=${1:-check}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x ${@} > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -25 $OUT/pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench_c4.json 2> $OUT/bench_c4.err; tail -3 $OUT/bench_c4.err
timeout 120 python bench.py --config 0 --steps 20 --warmup 5 --no-cpu --no-csr > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 120 python bench.py --gpus 2 --steps 5 --warmup 3 > $OUT/bench_gpus2.json 2> $OUT/bench_gpus2.err; echo "gpus2 rc=$?" >> $OUT/bench_gpus2.err
for f in $OUT/bench_*.json; do echo "== $f"; tail -c 1500 $f; echo; done
