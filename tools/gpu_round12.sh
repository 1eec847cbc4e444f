#!/bin/bash
# second session of round 1: final measurements of the replicas / policies / grid build
mkdir -p gpurun_out
echo "== ncu launch list (bench, n=3)"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_s2.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_under_ncu.log 2>&1; grep -c encode_kernel gpurun_out/launches_bench_s2.csv
echo "== ncu full n=3"; timeout 900 ncu --set full --clock-control none --import-source on -k regex:encode_kernel --launch-skip 6 --launch-count 3 -o gpurun_out/prof_n3_s2 -f python tools/prof_run.py --dim 3 2>&1 | tail -2
echo "== ncu full n=2"; timeout 900 ncu --set full --clock-control none --import-source on -k regex:encode_kernel --launch-skip 6 --launch-count 3 -o gpurun_out/prof_n2_s2 -f python tools/prof_run.py --dim 2 2>&1 | tail -2
for f in prof_n3_s2 prof_n2_s2; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/$f.raw.csv 2>/dev/null; done
ls -la gpurun_out/*.ncu-rep gpurun_out/*.raw.csv
