#!/bin/bash
# GPU-box session: bench lines for every config, ncu launch list + one full capture of the
# dominant kernels.  Usage (from repo root, under gpurun): bash tools/run_bench_suite.sh TAG
TAG=${1:-r02f}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
timeout 900 python bench.py > $OUT/bench_c4.json 2> $OUT/bench_c4.err
timeout 300 python bench.py --config 1 --no-cpu > $OUT/bench_c2.json 2> $OUT/bench_c2.err
timeout 300 python bench.py --config 2 --no-cpu > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 300 python bench.py --config 0 --no-cpu --no-csr > $OUT/bench_c1.json 2> $OUT/bench_c1.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
for c in 4 5 6 7; do timeout 400 python bench.py --config $c --no-cpu > $OUT/bench_x$c.json 2> $OUT/bench_x$c.err; done
timeout 300 python bench.py --config 6 --pa --no-cpu > $OUT/bench_x6pa.json 2> $OUT/bench_x6pa.err
timeout 300 python bench.py --config 7 --pa --no-cpu > $OUT/bench_x7pa.json 2> $OUT/bench_x7pa.err
for c in 1 3; do timeout 300 python bench.py --config $c --cgcg --no-cpu --no-e2e --no-csr > $OUT/bench_cgcg$c.json 2> $OUT/bench_cgcg$c.err; done
for c in 1 2 3; do timeout 300 python bench.py --config $c --gll --no-cpu --no-e2e > $OUT/bench_gll$c.json 2> $OUT/bench_gll$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c4.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elastic2_kernel -s 3 -c 1 \
  -o $OUT/prof_elastic python bench.py --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cg_update -s 3 -c 1 \
  -o $OUT/prof_update python bench.py --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_upd.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:laplace_kernel -s 6 -c 1 \
  -o $OUT/prof_laplace python bench.py --config 1 --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_full_lap.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:csr_spmv -s 2 -c 1 \
  -o $OUT/prof_spmv python bench.py --config 1 --steps 3 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_spmv.log 2>&1
echo suite done
timeout 300 python bench.py --config 6 --det --no-cpu --no-e2e > $OUT/bench_x6det.json 2> $OUT/bench_x6det.err
timeout 300 python bench.py --config 7 --det --no-cpu --no-e2e > $OUT/bench_x7det.json 2> $OUT/bench_x7det.err
timeout 600 python tools/size_sweep.py --out $OUT/size_sweep.jsonl > $OUT/size_sweep.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elastic2_kernel -s 40 -c 1 \
  -o $OUT/prof_elastic_apply python bench.py --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_apply.log 2>&1
echo suite2 done
