#!/bin/bash
mkdir -p gpurun_out
echo "== pytest tc"; timeout 600 python -m pytest tests/test_gpu_tc.py -m gpu -q 2>&1 | tail -5 | tee gpurun_out/pytest_tc.log
echo "== train bench"; timeout 600 python tools/train_bench.py 2>&1 | tee gpurun_out/train_bench.log
echo "== ncu tc kernel"; timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/prof_mlp_tc -f python tools/train_bench.py --once 2>&1 | tail -3
