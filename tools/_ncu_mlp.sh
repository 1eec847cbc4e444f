for v in 1 2; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mlp_tc --launch-skip 3 --launch-count 1 \
      -o gpurun_out/r2_ncu_mlp_v$v -f python tools/mlp_variant_bench.py --variant $v --reps 1 > gpurun_out/r2_ncu_mlp_v$v.log 2>&1
  ncu -i gpurun_out/r2_ncu_mlp_v$v.ncu-rep --page raw --csv > gpurun_out/r2_ncu_mlp_v${v}_raw.csv
done
ls -la gpurun_out/ | tail -5
