#!/bin/bash
mkdir -p gpurun_out
echo "== pytest all gpu"; timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6 | tee gpurun_out/pytest_all.log
echo "== smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo "== bench n=3"; timeout 900 python bench.py --steps 30 --warmup 5 2>&1 | tail -1 | tee gpurun_out/bench_n3.json | cut -c1-600
echo "== bench n=2"; timeout 900 python bench.py --steps 30 --warmup 5 --dim 2 --no-cpu 2>&1 | tail -1 | tee gpurun_out/bench_n2.json | cut -c1-300
echo "== bench n=3 T22"; timeout 900 python bench.py --steps 20 --warmup 5 --log2t 22 --no-cpu --no-train 2>&1 | tail -1 | tee gpurun_out/bench_n3_t22.json | cut -c1-300
echo "== ncu launch list"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-train > gpurun_out/bench_under_ncu.log 2>&1; grep -c encode_kernel gpurun_out/launches_bench.csv
echo "== ncu full fused"; timeout 900 ncu --set full --clock-control none --import-source on -k regex:encode_kernel --launch-skip 6 --launch-count 3 -o gpurun_out/prof_n3_final -f python tools/prof_run.py --dim 3 2>&1 | tail -2
