#!/bin/bash
mkdir -p gpurun_out
echo "== pytest"; timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 | tee gpurun_out/pytest.log
echo "== ncu launch list (bench)"; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_under_ncu.log 2>&1; tail -2 gpurun_out/bench_under_ncu.log | cut -c1-300
echo "== ncu full"; timeout 900 ncu --set full --clock-control none --import-source on -k regex:encode_kernel --launch-skip 6 --launch-count 3 -o gpurun_out/prof_n3 -f python tools/prof_run.py --dim 3 2>&1 | tail -5
echo "== sweep n=2"; timeout 600 python tools/sweep.py --dim 2 --reps 6 --quick 2>&1 | tee gpurun_out/sweep_n2.log | tail -40
echo "== sweep n=3 T=2^22"; timeout 600 python tools/sweep.py --dim 3 --reps 6 --quick --log2t 22 2>&1 | tee gpurun_out/sweep_n3_t22.log | tail -40
