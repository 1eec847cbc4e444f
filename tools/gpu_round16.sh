#!/bin/bash
# third session: soak (the GPU suite twice, order of the fp32 atomics differs from launch to launch) + round-end rehearsal
mkdir -p gpurun_out
echo "== fuzz"; timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k random_configurations 2>&1 | tail -5
for i in 1 2; do echo "== pytest -m gpu ($i)"; timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3; done
echo "== smoke"; timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo "== bench reference"; timeout 900 python bench.py --impl reference > gpurun_out/s3_bench_ref.json 2> gpurun_out/s3_bench_ref.err; tail -c 300 gpurun_out/s3_bench_ref.json
echo "== bench"; timeout 900 python bench.py > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err; tail -c 900 gpurun_out/s3_bench.json
