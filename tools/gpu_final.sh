#!/bin/bash
# Round-end evidence on one B200: GPU tests, smoke, bench line, reference arm, launch list, ncu
# --set full of every weighted-layer launch of one forward at the bench batch, into gpurun_out/.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|pack_pixels|logits|pix_tile|pix_popc|halo4|lin4" -c 30 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep --no-configs > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"fused|pix_tile|pix_popc|halo4|lin4|logits" -c 9 -o gpurun_out/prof_b256 -f python tools/prof_net.py 256 > gpurun_out/prof.log 2>&1
echo "ncu rc=$?" >> gpurun_out/prof.log
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/prof.log
timeout 300 python tools/gemm_bench.py --kernels umma,tma --shapes 1024,1024,1024 4096,1024,9216 1000,1024,4096 4096,4096,4096 128,262144,1152 8192,8192,8192 16384,16384,16384 > gpurun_out/gemm_crossover.jsonl 2>&1
timeout 120 python tools/timeline.py 256 > gpurun_out/timeline_b256.log 2>&1
timeout 120 python tools/timeline.py 1024 fc4 > gpurun_out/timeline_fc4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"xnor4t" -c 1 -o gpurun_out/prof_xnor4t -f python tools/gemm_bench.py --kernels tma --iters 1 --shapes 8192,8192,8192 > gpurun_out/prof_xnor4t.log 2>&1; echo "ncu xnor4t rc=$?" >> gpurun_out/prof_xnor4t.log
