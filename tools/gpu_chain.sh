#!/bin/bash
# Chained-engine dev loop: smoke, fused parity tests, bench chained vs per-layer, role clocks.
mkdir -p gpurun_out
timeout 120 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ -z "$QUICK" ]; then
timeout 600 python -m pytest tests/test_fused_gpu.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
fi
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_chain.log 2>&1
BNN_FUSED_CHAIN=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_perlayer.log 2>&1
for B in 256 4096; do
  echo "== B=$B" >> gpurun_out/roles.log
  BNN_FUSED_PROFILE=1 timeout 120 python tools/prof_net.py $B >> gpurun_out/roles.log 2>&1
done
