#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_fused_gpu.py -q -x --timeout 120 -p no:cacheprovider -k "auto or nopair or pair224 or fp4all or swapall or nofp4" > gpurun_out/ro_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ro_tests.log; tail -2 gpurun_out/ro_tests.log
BNN_FUSED_PROFILE=1 timeout 120 python tools/prof_net.py 256 2>&1 | grep "per-CTA"
timeout 120 python tools/timeline.py 256 0 2>&1 | grep timeline
timeout 200 python bench.py --no-cpu-baseline --no-configs --steps 50 --warmup 5 > gpurun_out/ro_bench.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/ro_bench.log').readline()); print(round(d['value']), round(d['e2e']['value']), d['batch_sweep_images_per_s'], d['layers_ms_per_step'])"
