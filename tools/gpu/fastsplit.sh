set -u
O=gpurun_out
FLEXCTC_PHASE_TIMERS=1 python profiles/phase_split.py --workload c4 > $O/fastsplit_c4.jsonl 2>&1
echo done > $O/fastsplit_done
