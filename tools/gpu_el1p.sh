#!/bin/bash
OUT=gpurun_out/el1p; mkdir -p $OUT
FEM_NVCC_FLAGS="-DFEM_EL_CY=1" python -c "from paper_2308_09839_b200 import build as B; B.build(force=True)" || exit 1
timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_parity.py -k "elastic" 2>&1 | grep -E "Error|assert|FAILED|def test" | head -20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:elastic1_kernel -s 8 -c 1 \
  -o $OUT/prof_el1 python bench.py --steps 3 --warmup 3 --no-e2e --no-csr --no-cpu > $OUT/ncu.log 2>&1
python tools/ncu_summary.py $OUT/prof_el1.ncu-rep | head -40
