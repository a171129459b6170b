#!/bin/bash
OUT=gpurun_out/s2d; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python bench.py --config 0 --no-cpu --no-csr > $OUT/bench_c1.json 2> $OUT/bench_c1.err; tail -c 1500 $OUT/bench_c1.json; echo
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-csr --no-cpu > $OUT/bench_c4.json 2> $OUT/bench_c4.err; tail -c 900 $OUT/bench_c4.json; echo
timeout 900 python tools/size_sweep.py --out $OUT/size_sweep.jsonl > $OUT/size_sweep.log 2>&1; tail -3 $OUT/size_sweep.log
bash tools/gpu_traffic.sh
