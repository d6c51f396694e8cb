#!/bin/bash
# A/B of an engine setting through the bench (env var + value list): AB_VAR, AB_VALS
mkdir -p gpurun_out
for v in $AB_VALS; do
  env $AB_VAR=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/ab_$v.log 2>&1
  python -c "
import json;l=[json.loads(x) for x in open('gpurun_out/ab_$v.log') if x.startswith('{')][-1]
print('$AB_VAR=$v', 'ms/step',round(l['ms_per_step'],4),'img/s',int(l['value']),'sweep',l['batch_sweep_images_per_s'],'layers',l['layers_ms_per_step'], 'parity', l['parity_vs_oracle'])"
done
