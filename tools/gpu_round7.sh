#!/bin/bash
mkdir -p gpurun_out
echo "== pytest tc"; timeout 600 python -m pytest tests/test_gpu_tc.py -m gpu -q 2>&1 | tail -8 | tee gpurun_out/pytest_tc.log
echo "== train bench"; timeout 600 python tools/train_bench.py 2>&1 | tee gpurun_out/train_bench.log
