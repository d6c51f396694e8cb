#!/bin/bash
# A/B of two builds of libbnn_b200.so on one box: abtmp/<name>.so for each name in AB_SOS
# (alternating as listed), bench line per run
mkdir -p gpurun_out
cp paper_1911_04477_b200/libbnn_b200.so /tmp/lib_keep.so
i=0
for n in $AB_SOS; do
  i=$((i+1))
  cp abtmp/$n.so paper_1911_04477_b200/libbnn_b200.so
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-configs > gpurun_out/abso_${i}_$n.log 2>&1
  python -c "
import json;l=[json.loads(x) for x in open('gpurun_out/abso_${i}_$n.log') if x.startswith('{')][-1]
print('$n', 'ms/step',round(l['ms_per_step'],4),'img/s',int(l['value']),'sweep',l['batch_sweep_images_per_s'],'parity', l['parity_vs_oracle'])"
done
cp /tmp/lib_keep.so paper_1911_04477_b200/libbnn_b200.so
