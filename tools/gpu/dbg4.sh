set -u
O=gpurun_out/dbg4
mkdir -p $O
CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_lgt.py 2 > $O/d0.log 2>&1
timeout 120 python tools/dbg_lgt.py 8 > $O/d0b8.log 2>&1
echo done > $O/done
