#!/bin/bash
# Round 2: the stand-alone tcgen05 training kernel with two tiles in flight (csrc/sxen_mlp_tc2.cu) against the one-tile kernel
# (csrc/sxen_mlp_tc.cu): CUDA-event A/B with the kernels' cycle counters, ncu --set full of one launch of each, the per-kernel
# launch list of the training step.  Run under gpurun; everything lands in gpurun_out/.
cd "$(dirname "$0")/.."
python tools/mlp_variant_bench.py --reps 30 > gpurun_out/r2_mlp_variants.txt 2>&1
python tools/mlp_variant_bench.py --reps 30 --width 16 >> gpurun_out/r2_mlp_variants.txt 2>&1
python tools/mlp_variant_bench.py --reps 30 --log2n 24 >> gpurun_out/r2_mlp_variants.txt 2>&1
cat gpurun_out/r2_mlp_variants.txt
for v in 1 2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_tc --launch-skip 3 --launch-count 1 \
      -o gpurun_out/r2_ncu_mlp_v$v -f python tools/mlp_variant_bench.py --variant $v --reps 1 > gpurun_out/r2_ncu_mlp_v$v.log 2>&1
  ncu -i gpurun_out/r2_ncu_mlp_v$v.ncu-rep --page raw --csv > gpurun_out/r2_ncu_mlp_v${v}_raw.csv
done
python tools/train_bench.py --reps 20 > gpurun_out/r2_train_bench_tc2.txt 2>&1
tail -8 gpurun_out/r2_train_bench_tc2.txt
