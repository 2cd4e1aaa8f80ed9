set -u
O=gpurun_out/dbg
mkdir -p $O
FLEXCTC_WARP=1 timeout 120 python tools/dbg_lgt.py 2 > $O/warp.log 2>&1
FLEXCTC_LOGITS_DIRECT=0 timeout 120 python tools/dbg_lgt.py 2 > $O/copy.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/dbg_lgt.py 2 > $O/direct.log 2>&1
echo done > $O/done
