#!/bin/bash
# halo4 kernel bring-up: fused parity (auto = halo, nohalo = swap4), benchmarked-batch parity,
# a short bench line, and the launch list of one forward at batch 256
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fused_gpu.py -m gpu -q -x -p no:cacheprovider -k "auto or nohalo" > gpurun_out/halo_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/halo_pytest.log
tail -5 gpurun_out/halo_pytest.log
timeout 600 python -m pytest tests/test_bench_parity_gpu.py -m gpu -q -x -p no:cacheprovider > gpurun_out/halo_pytest2.log 2>&1; echo "rc=$?" >> gpurun_out/halo_pytest2.log
tail -3 gpurun_out/halo_pytest2.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-configs > gpurun_out/halo_bench.log 2>&1
tail -c 3000 gpurun_out/halo_bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|pack_pixels|logits|pix_|halo" -c 40 --csv --log-file gpurun_out/halo_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-configs > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/halo_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:30]: print(r[ki][:70], r[vi])
PY
