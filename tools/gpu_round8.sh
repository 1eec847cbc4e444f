#!/bin/bash
mkdir -p gpurun_out
echo "== pytest tasks+tc"; timeout 900 python -m pytest tests/test_gpu_tasks.py tests/test_gpu_tc.py -m gpu -q 2>&1 | tail -30 | tee gpurun_out/pytest_tasks.log
echo "== train bench"; timeout 600 python tools/train_bench.py 2>&1 | head -4 | tee gpurun_out/train_bench.log
