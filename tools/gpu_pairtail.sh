#!/bin/bash
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_fused_gpu.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pt_tests.log; tail -2 gpurun_out/pt_tests.log
timeout 120 python tools/timeline.py 256 0 2>&1 | grep timeline
timeout 200 python bench.py --no-cpu-baseline --no-configs --steps 50 --warmup 5 > gpurun_out/pt_bench.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/pt_bench.log').readline()); print(round(d['value']), round(d['e2e']['value']), d['batch_sweep_images_per_s'], d['layers_ms_per_step'])"
