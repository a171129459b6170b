#!/bin/bash
TAG=r2g; OUT=gpurun_out/$TAG; mkdir -p $OUT
bash tools/gpu_tests.sh $TAG -x tests/test_gpu_hex.py tests/test_gpu_parity.py tests/test_gpu_gll.py
timeout 600 python bench.py --pa --steps 10 --warmup 3 --no-cpu --no-csr --no-e2e > $OUT/bench_c4_pa.json 2> $OUT/bench_c4_pa.err
tail -c 600 $OUT/bench_c4_pa.json; tail -3 $OUT/bench_c4_pa.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:laplace_kernel -s 6 -c 1 \
  -o $OUT/prof_lap_fused python bench.py --config 1 --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_lap.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elastic2_kernel -s 8 -c 1 \
  -o $OUT/prof_el_fused python bench.py --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_el.log 2>&1
ls -la $OUT
