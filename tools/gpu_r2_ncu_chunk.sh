#!/bin/bash
# Round 2: ncu --set full of the fused encode launch at configs[1], one grid slice (level_chunk = -1) vs the chunked launch
# (library default at dim 3: ranges of 8 levels), plus the launch list of the bench command.  Run under gpurun.
set -x
cd "$(dirname "$0")/.."
for tag in one_slice:-1 chunked:0; do
  name=${tag%%:*}; ch=${tag##*:}
  ncu --set full --clock-control none --import-source on -k regex:encode_kernel --launch-skip 8 --launch-count 1 \
      -o gpurun_out/r2_ncu_n3_$name -f python tools/prof_run.py --dim 3 --level-chunk $ch > gpurun_out/r2_ncu_n3_$name.log 2>&1
  ncu -i gpurun_out/r2_ncu_n3_$name.ncu-rep --page raw --csv > gpurun_out/r2_ncu_n3_${name}_raw.csv
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_bench.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --no-train --path fused --lpt 2 --level-major 0 > gpurun_out/r2_launches_bench.log 2>&1
python bench.py --steps 30 > gpurun_out/r2_bench_n3.json 2> gpurun_out/r2_bench_n3.err
python bench.py --steps 30 --dim 2 --no-train > gpurun_out/r2_bench_n2.json 2> gpurun_out/r2_bench_n2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 10 --no-train --no-cpu > gpurun_out/r2_bench_torchrun1.json 2> gpurun_out/r2_bench_torchrun1.err
tail -c 400 gpurun_out/r2_bench_torchrun1.err
