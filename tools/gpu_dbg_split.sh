mkdir -p gpurun_out
BNN_FUSED_PROFILE=1 timeout 60 python tools/prof_net.py 1 > gpurun_out/dbg_split.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_split.log
BNN_FUSED_SPLIT=1 BNN_FUSED_PROFILE=1 timeout 60 python tools/prof_net.py 1 >> gpurun_out/dbg_split.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_split.log
