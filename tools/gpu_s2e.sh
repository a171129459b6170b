#!/bin/bash
bash tools/gpu_tests.sh s2e
bash tools/gpu_sanitize.sh san_r02
