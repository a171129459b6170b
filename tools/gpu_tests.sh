#!/bin/bash
# GPU tests only: bash tools/gpu_tests.sh TAG [pytest-args]
TAG=${1:-tests}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
timeout 1500 python -m pytest -m gpu -q ${@} > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -30 $OUT/pytest.log
