#!/bin/bash
OUT=gpurun_out/el2prof; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elastic -s 3 -c 1 \
  -o $OUT/prof_el2 python bench.py --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu_el.log 2>&1
bash tools/gpu_variants.sh el2v "3" "test_gpu_parity and elastic" "-DFEM_EL2_TY=9" "-DFEM_EL2_TY=11 -DFEM_EL2_S=2" "-DFEM_EL2_TY=7 -DFEM_EL2_S=2"
