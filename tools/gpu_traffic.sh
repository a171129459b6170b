#!/bin/bash
# DRAM bytes of one fused CG apply at C4 = its edge + interior grids (two consecutive launches)
OUT=gpurun_out/traffic; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --kernel-name-base demangled -k "regex:elastic2_kernel<.bool.1, .int.2, .int.8, .int.4" -s 6 -c 4 --clock-control none \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_traffic.csv 2> $OUT/ncu_traffic.err
tail -20 $OUT/ncu_traffic.csv
