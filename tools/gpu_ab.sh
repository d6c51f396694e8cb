#!/bin/bash
# A/B of an engine setting through the bench (env var + value list): AB_VAR, AB_VALS (values may
# repeat: runs alternate); AB_E2E=1 also times the end-to-end pipeline
mkdir -p gpurun_out
i=0
for v in $AB_VALS; do
  i=$((i+1))
  E2E="--no-e2e"; [ -n "$AB_E2E" ] && E2E=""
  env $AB_VAR=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $E2E --no-configs > gpurun_out/ab_${i}_$v.log 2>&1
  python -c "
import json;l=[json.loads(x) for x in open('gpurun_out/ab_${i}_$v.log') if x.startswith('{')][-1]
print('$AB_VAR=$v', 'ms/step',round(l['ms_per_step'],4),'img/s',int(l['value']),'e2e',l.get('e2e') and int(l['e2e']['value']),'sweep',l['batch_sweep_images_per_s'],'layers',l['layers_ms_per_step'], 'parity', l['parity_vs_oracle'])"
done
