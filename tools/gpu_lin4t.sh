#!/bin/bash
# TMA-fed lin4 + TMA-fed xnor_gemm: parity subsets, then cfg4 / sweep A/B (images TMA-loaded vs
# producer-expanded).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_halo_lin4_gpu.py tests/test_fused_gpu.py -m gpu -q -x --timeout 300 -p no:cacheprovider -k "gemm or conv_large or lin4 or default_network_fused" > gpurun_out/l4t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/l4t_pytest.log
tail -n 3 gpurun_out/l4t_pytest.log
for m in 0 -1 0 -1; do
  BNN_LIN4_TMA=$m timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --sweep 256,1024,4096,16384 > gpurun_out/l4t_bench_$m.log 2>&1
  python - "$m" <<'P'
import json, sys
for line in open(f"gpurun_out/l4t_bench_{sys.argv[1]}.log"):
    if line.startswith("{"):
        l = json.loads(line)
        c = l["configs"]["cfg4_fc_stack_b1024"]
        print("TMA", sys.argv[1], "b256", round(l["value"]), "cfg4", round(c["binary_tops"]), c["ms"], c.get("kernels"),
              [(s.get("batch"), round(s.get("images_per_s", 0))) for s in l.get("batch_sweep", l.get("sweep", []))])
P
done
