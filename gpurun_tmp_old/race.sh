#!/bin/bash
OUT=gpurun_out/race; mkdir -p $OUT; C=paper_2308_09839_b200/csrc
python -m paper_2308_09839_b200.build --force > $OUT/b1.log 2>&1
echo "=== new"
for i in 1 2 3 4; do timeout 600 python -m pytest -q -m gpu tests/test_gpu_fullsize.py -k "x_defer" 2>&1 | grep -E "passed|failed|assert .*C|Error" | tail -3; done
for f in kernels_elastic.cu kernels_laplace.cu; do cp $C/$f /tmp/new_$f; cp gpurun_tmp_old/$f $C/; done
python -m paper_2308_09839_b200.build --force > $OUT/b2.log 2>&1
echo "=== old"
for i in 1 2 3 4; do timeout 600 python -m pytest -q -m gpu tests/test_gpu_fullsize.py -k "x_defer" 2>&1 | grep -E "passed|failed|assert .*C|Error" | tail -3; done
for f in kernels_elastic.cu kernels_laplace.cu; do cp /tmp/new_$f $C/$f; done
python -m paper_2308_09839_b200.build --force > /dev/null 2>&1
