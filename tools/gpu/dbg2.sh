set -u
O=gpurun_out/dbg2
mkdir -p $O
for d in 0 1 2 3; do CUDA_LAUNCH_BLOCKING=1 FLEXCTC_DBG=$d timeout 120 python tools/dbg_lgt.py 2 > $O/d$d.log 2>&1; done
CUDA_LAUNCH_BLOCKING=1 FLEXCTC_FAST=0 timeout 120 python tools/dbg_lgt.py 2 > $O/nofast.log 2>&1
echo done > $O/done
