#!/bin/bash
mkdir -p gpurun_out
echo "== memcheck smoke + tc + neural"; timeout 900 compute-sanitizer --tool memcheck --error-exitcode 7 python -m pytest tests/test_gpu_tc.py tests/test_gpu_neural.py tests/test_gpu_tasks.py -m gpu -q -x -k "not large and not fit_image_matches" 2>&1 | tail -12 | tee gpurun_out/memcheck.log
echo "== memcheck parity subset"; timeout 900 compute-sanitizer --tool memcheck --error-exitcode 7 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "golden or empty or accumulator or sparse_adam or dense_adam or more_than_32" 2>&1 | tail -8 | tee -a gpurun_out/memcheck.log
echo "== racecheck encode/mlp exact"; timeout 600 compute-sanitizer --tool racecheck --error-exitcode 7 python -m pytest tests/test_gpu_neural.py -m gpu -q -x -k "odd_shapes or reference_fixture" 2>&1 | tail -6 | tee gpurun_out/racecheck.log
echo "== sweep dims T=2^22"; for d in 2 3 4 5 6; do timeout 300 python tools/sweep.py --dim $d --reps 4 --quick --log2t 22 2>&1 | grep -E "^#|best" ; done | tee gpurun_out/sweep_dims_t22.log
