#!/bin/bash
# One gpurun call: parity tests, smoke, launch-shape sweep, bench, ncu launch list + full capture of the top kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
echo "== pytest"; timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 | tee gpurun_out/pytest.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 | tee gpurun_out/smoke.log
echo "== sweep n=3"; timeout 900 python tools/sweep.py --dim 3 --reps 6 --json gpurun_out/sweep_n3.json 2>&1 | tee gpurun_out/sweep_n3.log | tail -70
echo "== bench"; timeout 600 python bench.py --steps 20 --warmup 3 2>&1 | tail -3 | tee gpurun_out/bench.log
echo "== bench split"; timeout 600 python bench.py --steps 20 --warmup 3 --path split --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench_split.log
