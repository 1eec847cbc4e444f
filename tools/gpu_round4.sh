#!/bin/bash
mkdir -p gpurun_out
echo "== pytest neural"; timeout 900 python -m pytest tests/test_gpu_neural.py -m gpu -q 2>&1 | tail -40 | tee gpurun_out/pytest_neural.log
echo "== pytest parity"; timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q 2>&1 | tail -15 | tee gpurun_out/pytest_parity.log
