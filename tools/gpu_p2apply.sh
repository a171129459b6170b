#!/bin/bash
python -c "from paper_2308_09839_b200 import build as B; B.build()" || exit 1
timeout 1500 python -m pytest -q -x -m gpu tests/test_loopback.py tests/test_slab.py 2>&1 | tail -3
timeout 1500 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_fullsize.py 2>&1 | tail -2
