#!/bin/bash
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_fused_gpu.py -q -x --timeout 200 -p no:cacheprovider 2>&1 | tail -2
timeout 200 python bench.py --no-cpu-baseline --no-configs --steps 50 --warmup 5 > gpurun_out/fc_bench.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/fc_bench.log').readline()); print(round(d['value']), round(d['e2e']['value']), d['batch_sweep_images_per_s'], d['layers_ms_per_step'])"
