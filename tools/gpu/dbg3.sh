set -u
O=gpurun_out/dbg3
mkdir -p $O
for d in 4 8; do CUDA_LAUNCH_BLOCKING=1 FLEXCTC_DBG=$d timeout 120 python tools/dbg_lgt.py 2 > $O/d$d.log 2>&1; done
echo done > $O/done
