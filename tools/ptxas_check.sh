#!/bin/bash
# registers / spills of one kernel file under extra flags: tools/ptxas_check.sh file.cu 'regex' [nvcc flags...]
F=$1; RE=$2; shift 2
ND=$(python -c "from paper_2308_09839_b200 import build as B; print(B.nccl_dir())")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Iinclude -I$ND/include --expt-relaxed-constexpr -Xptxas -v "$@" -c paper_2308_09839_b200/csrc/$F -o /tmp/ptxas_check.o 2>&1 \
  | awk -v re="$RE" '/Compiling entry function/ {name=$0; show = (name ~ re)} show && /spill|Used/ {sub(/.*Function properties for /,""); print substr(name, 40, 90) " | " $0}'
