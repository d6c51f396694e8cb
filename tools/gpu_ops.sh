#!/bin/bash
# standalone operators: parity (encoders, im2col, GEMM both kernels, conv/linear), the GEMM
# crossover sweep (tools/gemm_bench.py) and the bench's per-config section
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_cpp_api.py -m gpu -q -x -p no:cacheprovider > gpurun_out/ops_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ops_pytest.log
tail -3 gpurun_out/ops_pytest.log
timeout 600 python tools/gemm_bench.py --shapes 64,1024,576 128,1024,1152 256,256,1024 512,512,1024 1024,1024,1024 1000,1024,4096 4096,1024,9216 128,262144,1152 8192,8192,8192 > gpurun_out/gemm_crossover.jsonl 2>&1
cat gpurun_out/gemm_crossover.jsonl
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/ops_bench.log 2>&1
python -c "
import json;l=[json.loads(x) for x in open('gpurun_out/ops_bench.log') if x.startswith('{')][-1]
c=l['configs']
for k,v in c.items(): print(k, {kk:vv for kk,vv in v.items() if kk in ('ms','device_ms','xnor_gemm_device_tops','binary_tops','gbs','frac_hbm','xnor_gemm_ms','xnor_gemm_tops','gemm_kernel','parity_vs_reference','images_per_s','encode_ms','cols_frac_hbm','rows_frac_hbm')})"
