#!/bin/bash
# FP4 CTA-pair kernel: parity, per-role waits, bench (pairs on / off).
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_fused_gpu.py -q -x --timeout 120 -p no:cacheprovider -k "auto or nopair or fp4all" > gpurun_out/pair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pair_tests.log
tail -3 gpurun_out/pair_tests.log
timeout 300 python -m pytest tests/test_fused_gpu.py -q --timeout 120 -p no:cacheprovider >> gpurun_out/pair_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pair_tests.log
tail -2 gpurun_out/pair_tests.log
for p in 1 0; do
  BNN_FP4_PAIR=$p timeout 200 python bench.py --no-cpu-baseline --no-configs --steps 50 --warmup 5 > gpurun_out/pair_bench_$p.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/pair_bench_$p.log').readline()); print('pair=$p', round(d['value']), round(d['e2e']['value']), d['batch_sweep_images_per_s'], d['layers_ms_per_step'])"
done
for p in 1 0; do BNN_FP4_PAIR=$p BNN_FUSED_PROFILE=1 timeout 120 python tools/prof_net.py 4096 2>&1 | grep swap4 | head -6; done
