#!/bin/bash
# Round 2, fourth session (b): the tcgen05 probes from their own test-only library, the configs[4] sweep (n = 2..6, T = 2^22) and
# configs[2]/[3] on the final code.  Run under gpurun.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_abi_exports.py -x -q 2>&1 | tail -2
python tools/tc_probe.py 2>&1 | tail -3
: > gpurun_out/r2s4_bench_dims_T22.jsonl
for n in 2 3 4 5 6; do
  python bench.py --dim $n --log2t 22 --no-train --no-cpu --steps 20 2> gpurun_out/r2s4_dims_$n.err | tail -n1 >> gpurun_out/r2s4_bench_dims_T22.jsonl
done
python tools/config_runs.py --skip-c1 > gpurun_out/r2s4_config_runs.log 2>&1
tail -5 gpurun_out/r2s4_config_runs.log
python - <<'PY'
import json
for l in open('gpurun_out/r2s4_bench_dims_T22.jsonl'):
    a=json.loads(l); print(a['config']['dim'], round(a['ms_per_step'],4), f"{a['value']:.3e}", round(a['roofline']['frac'],3), a['roofline']['kernel'], a['launch']['path'])
PY
