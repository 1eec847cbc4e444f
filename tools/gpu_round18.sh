#!/bin/bash
# third session, final: launch list of the current bench command + soak + rehearsal
mkdir -p gpurun_out
echo "== ncu launch list"; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-train > gpurun_out/s3_bench_under_ncu.log 2>&1; grep -c encode_kernel gpurun_out/s3_launches_bench.csv
for i in 1 2; do echo "== pytest -m gpu ($i)"; timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3; done
echo "== smoke"; timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo "== bench reference"; timeout 900 python bench.py --impl reference > gpurun_out/s3_bench_ref.json 2> gpurun_out/s3_bench_ref.err; tail -c 300 gpurun_out/s3_bench_ref.json
echo "== bench"; timeout 900 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; python -c "
import json; d=json.load(open('gpurun_out/s3_bench.json')); print(d['value'], d['roofline']['frac'], d['e2e']['value'], json.dumps(d['train_step']))"
