#!/bin/bash
# quick GPU iteration: halo/lin4/fused parity subset, warm halo4 role counters, bench line
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_halo_lin4_gpu.py tests/test_fused_gpu.py tests/test_parity_gpu.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/q_pytest.log
cat gpurun_out/q_pytest.log
BATCHES="${BATCHES:-256 4096}" MODES="${MODES:-0}" bash tools/gpu_halo_prof.sh > /dev/null
cut -c1-60,100-460 gpurun_out/halo_prof.log
timeout 300 python bench.py --steps 30 --warmup 5 > gpurun_out/q_bench.log 2>&1
python tools/summ.py gpurun_out/q_bench.log 2>/dev/null || tail -c 600 gpurun_out/q_bench.log
