#!/bin/bash
mkdir -p gpurun_out
echo "== new tests"; timeout 1200 python -m pytest tests/test_gpu_cpp_trainer.py -x -q 2>&1 | tail -15
echo "== train loop"; timeout 900 python tools/train_loop_bench.py 2>&1 | tee gpurun_out/s3_train_loop2.log
echo "== all gpu tests"; timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
