#!/bin/bash
# Round 2, fourth session: rehearsal of the driver's round-end sequence on the rebuilt library (GPU suite, smoke, both bench
# arms, the launch list of the bench command).  Run under gpurun.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/r2s4_gpu.txt
( time timeout 1800 python -m pytest tests -m gpu -x -q ) > gpurun_out/r2s4_pytest_gpu.log 2>&1; tail -3 gpurun_out/r2s4_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" 2>&1 | tail -1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2s4_bench_ref.json 2> gpurun_out/r2s4_bench_ref.err
python bench.py > gpurun_out/r2s4_bench_n3.json 2> gpurun_out/r2s4_bench_n3.err
python bench.py --dim 2 --no-train > gpurun_out/r2s4_bench_n2.json 2> gpurun_out/r2s4_bench_n2.err
python bench.py --gpus 2 --oversubscribe --steps 5 --no-train --no-cpu 2> gpurun_out/r2s4_2ranks.err | tail -n1 > gpurun_out/r2s4_2ranks_oversubscribed.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s4_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-train > /dev/null 2>&1
python tools/train_bench.py --reps 20 > gpurun_out/r2s4_train_bench.txt 2>&1
for f in gpurun_out/r2s4_*.err; do echo "== $f"; tail -c 300 "$f"; done
head -c 1500 gpurun_out/r2s4_bench_n3.json
