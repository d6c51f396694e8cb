#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_fused_gpu.py -q -x --timeout 200 -p no:cacheprovider -k "pipeline or graph" 2>&1 | tail -3
for r in 1 2 3; do
timeout 200 python bench.py --no-cpu-baseline --no-configs --no-sweep --steps 50 --warmup 5 > gpurun_out/pipe_bench.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/pipe_bench.log').readline()); print(round(d['value']), d['e2e'])"
done
