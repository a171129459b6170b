#!/bin/bash
# static SASS opcode mix of one kernel in libfem.so: bash tools/sass_mix.sh <mangled-substring>
cuobjdump -sass -fun "$1" paper_2308_09839_b200/libfem.so 2>/dev/null | grep -E "^\s+/\*[0-9a-f]{4}\*/" | \
  awk '{ op=$2; if (op ~ /^@/) op=$3; sub(/\..*/, "", op); c[op]++; n++ } END { printf "total %d:", n; for (o in c) if (c[o] > n/100) printf " %s=%d", o, c[o]; printf "\n" }'
