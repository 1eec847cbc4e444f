#!/bin/bash
# third session: refresh the BASELINE config matrix with the final library
mkdir -p gpurun_out
echo "== config runs (C1, C3, C4)"; timeout 1500 python tools/config_runs.py > gpurun_out/s3_config_runs.log 2>&1; tail -c 1500 gpurun_out/s3_config_runs.log
echo "== C5 sweep"; : > gpurun_out/s3_c5.jsonl; for n in 2 3 4 5 6; do timeout 600 python bench.py --dim $n --log2t 22 --no-cpu --no-train >> gpurun_out/s3_c5.jsonl 2>> gpurun_out/s3_c5.err; done; python - <<'PY'
import json
for line in open("gpurun_out/s3_c5.jsonl"):
    d = json.loads(line)
    print(d["config"]["dim"], round(d["ms_per_step"], 3), "ms", f'{d["value"]:.3e}', "frac", round(d["roofline"]["frac"], 3), d["config"]["path"])
PY
echo "== n=2"; timeout 600 python bench.py --dim 2 --no-cpu --no-train > gpurun_out/s3_bench_n2.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/s3_bench_n2.json')); print(d['value'], d['roofline']['frac'])"
