#!/bin/bash
mkdir -p gpurun_out
echo "== pytest tc"; timeout 600 python -m pytest tests/test_gpu_tc.py -m gpu -x -q 2>&1 | tail -40 | tee gpurun_out/pytest_tc.log
