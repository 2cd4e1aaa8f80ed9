set -u
O=gpurun_out/phase5
mkdir -p $O
FLEXCTC_PHASE_TIMERS=1 python profiles/phase_split.py --workload c5 > $O/phase_c5.jsonl 2>&1
echo done > $O/done
