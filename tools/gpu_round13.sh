#!/bin/bash
# third session of round 1: round-end rehearsal (tests, smoke, both bench arms) on a fresh box
mkdir -p gpurun_out
echo "== pytest -m gpu"; timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
echo "== smoke"; timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo "== bench reference"; timeout 900 python bench.py --impl reference > gpurun_out/s3_bench_ref.json 2> gpurun_out/s3_bench_ref.err; tail -c 600 gpurun_out/s3_bench_ref.json
echo "== bench"; timeout 900 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; tail -c 1500 gpurun_out/s3_bench.json
