#!/bin/bash
# every fused-engine tiling (parity) + a bench line + launch list
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_fused_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/fused_all.log 2>&1; echo "rc=$?" >> gpurun_out/fused_all.log
tail -3 gpurun_out/fused_all.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-configs > gpurun_out/halo_bench.log 2>&1
python -c "
import json;l=[json.loads(x) for x in open('gpurun_out/halo_bench.log') if x.startswith('{')][-1]
print('ms/step',l['ms_per_step'],'img/s',l['value'],'e2e',l['e2e']['value'],'sweep',l['batch_sweep_images_per_s'],'layers',l['layers_ms_per_step'], 'parity', l['parity_vs_oracle'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|pack_pixels|logits|pix_|halo" -c 9 --csv --log-file gpurun_out/halo_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-configs > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/halo_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:10]: print(r[ki][:70], r[vi])
PY
