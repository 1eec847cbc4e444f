#!/bin/bash
mkdir -p gpurun_out
echo "== pytest"; timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -25 | tee gpurun_out/pytest.log
echo "== per level n=3"; timeout 300 python tools/per_level.py 3 2>&1 | tee gpurun_out/per_level_n3.log
echo "== sweep n=3"; timeout 600 python tools/sweep.py --dim 3 --reps 6 --quick 2>&1 | tee gpurun_out/sweep_n3_b.log | grep -v "^  1 \| 16 "
echo "== bench"; timeout 600 python bench.py --steps 20 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench.log | cut -c1-400
