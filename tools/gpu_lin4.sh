#!/bin/bash
# lin4 bring-up: fused parity (auto = lin4, nolin4 = int8), bench-parity tests, bench line, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_gpu.py -m gpu -q -x -p no:cacheprovider -k "auto or nolin4" > gpurun_out/lin4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/lin4_pytest.log
tail -15 gpurun_out/lin4_pytest.log
timeout 600 python -m pytest tests/test_bench_parity_gpu.py tests/test_harness_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/lin4_pytest2.log 2>&1; grep -E "passed|failed|Error|^E " gpurun_out/lin4_pytest2.log | head -12
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/lin4_bench.log 2>&1
python -c "
import json;l=[json.loads(x) for x in open('gpurun_out/lin4_bench.log') if x.startswith('{')][-1]
print('ms/step',l['ms_per_step'],'img/s',l['value'],'e2e',l['e2e']['value'],'sweep',l['batch_sweep_images_per_s'],'layers',l['layers_ms_per_step'], 'parity', l['parity_vs_oracle'])
c=l['configs']; print({k:(v.get('ms'),v.get('binary_tops'),v.get('parity_vs_reference'),v.get('kernels')) for k,v in c.items() if k.startswith('cfg')})"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|pack_pixels|logits|pix_|halo|lin" -c 11 --csv --log-file gpurun_out/lin4_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-configs > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/lin4_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:12]: print(r[ki][:70], r[vi])
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"lin4" -c 2 -o gpurun_out/lin4_b256 -f python tools/prof_net.py 256 > /dev/null 2>&1
echo "ncu rc=$?"
