#!/bin/bash
# Fused-engine pass: fused parity tests, bench at B=256 and B=4096, per-kernel launch list.
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_fused_gpu.py -q -x --timeout 120 -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fused.log
timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_fused.log 2>&1; echo "rc=$?" >> gpurun_out/bench_fused.log
timeout 200 python bench.py --steps 10 --warmup 5 --batch 4096 --no-cpu-baseline --no-e2e > gpurun_out/bench_fused_4k.log 2>&1; echo "rc=$?" >> gpurun_out/bench_fused_4k.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fused -c 40 --csv --log-file gpurun_out/launches_fused.csv python bench.py --steps 2 --warmup 3 --batch 4096 --no-cpu-baseline --no-e2e > /dev/null 2>&1
#!/bin/bash
# Per-role barrier wait cycles of every fused launch (BNN_FUSED_PROFILE=1), B=4096.
mkdir -p gpurun_out
BNN_FUSED_PROFILE=1 timeout 120 python tools/prof_net.py 4096 > gpurun_out/dbg.log 2>&1
echo rc=$? >> gpurun_out/dbg.log
