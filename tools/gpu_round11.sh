#!/bin/bash
mkdir -p gpurun_out
for args in "--dim 3" "--dim 2 --no-cpu" "--dim 3 --log2t 22 --no-cpu --no-train" "--dim 2 --log2t 22 --no-cpu --no-train"; do
  echo "== bench $args"; timeout 900 python bench.py --steps 30 --warmup 5 $args 2>&1 | tail -1 > gpurun_out/b.json; python - <<'PY'
import json
d=json.loads(open('gpurun_out/b.json').read())
print('value %.4e'%d['value'],'ms',round(d['ms_per_step'],4),'path',d['config']['path'],'tuning',d['config']['tuning'],'frac',round(d['roofline']['frac'],4))
print('  autotune',{k:round(v,4) for k,v in (d['config'].get('autotune_ms') or {}).items()})
print('  e2e %.3e'%d['e2e']['value'],'train',d.get('train_step'))
PY
done
