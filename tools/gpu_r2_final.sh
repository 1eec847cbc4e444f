#!/bin/bash
# Round 2 final rehearsal (what the driver runs at round end, plus the launch list): GPU suite twice, smoke, the two bench arms,
# one rank under torchrun, the oversubscribed 2-rank functional run.  Run under gpurun.
cd "$(dirname "$0")/.."
for i in 1 2; do timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2; done
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_final_bench_ref.json 2> gpurun_out/r2_final_bench_ref.err
python bench.py > gpurun_out/r2_final_bench_n3.json 2> gpurun_out/r2_final_bench_n3.err
python bench.py --dim 2 --no-train > gpurun_out/r2_final_bench_n2.json 2> gpurun_out/r2_final_bench_n2.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 1 --steps 10 --no-train --no-cpu 2> gpurun_out/r2_final_torchrun1.err | tail -n1 > gpurun_out/r2_final_torchrun1.json
python bench.py --gpus 2 --oversubscribe --steps 5 --no-train --no-cpu 2> gpurun_out/r2_final_2ranks.err | tail -n1 > gpurun_out/r2_final_2ranks_oversubscribed.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_final_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-train --path fused --lpt 2 --level-major 0 > /dev/null 2>&1
python tools/config_runs.py --skip-c1 > gpurun_out/r2_final_config_runs.log 2>&1
python tools/train_bench.py --reps 20 > gpurun_out/r2_final_train_bench.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2_final_launches_train_step.csv \
    python tools/train_bench.py --reps 3 > /dev/null 2>&1
for f in gpurun_out/r2_final_*.err; do echo "== $f"; tail -c 300 "$f"; done
