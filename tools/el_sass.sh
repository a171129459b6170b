#!/bin/bash
# compile kernels_elastic.cu alone (extra flags in $1) and print the z-march loop mix of the fused CG kernel
NCCL_INC=$(python -c "import nvidia.nccl;print(list(nvidia.nccl.__path__)[0])")/include
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -I$NCCL_INC \
  --expt-relaxed-constexpr -Xptxas -v $1 -c paper_2308_09839_b200/csrc/kernels_elastic.cu -o /tmp/ke.o 2> /tmp/ke.log || { cat /tmp/ke.log; exit 1; }
grep -A2 "elastic2_kernelILb1ELi${2:-2}ELi8ELi${3:-4}ELb0ELb0E" /tmp/ke.log | grep -o "[0-9]* bytes spill stores\|Used [0-9]* registers" | tr '\n' ' '; echo
python tools/sass_loop.py /tmp/ke.o "elastic2_kernelILb1ELi${2:-2}ELi8ELi${3:-4}ELb0ELb0E" | tail -n +3 | head -3
