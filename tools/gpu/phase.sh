set -u
O=gpurun_out/phase
mkdir -p $O
FLEXCTC_PHASE_TIMERS=1 python profiles/phase_split.py --workload c4 > $O/phase_c4.jsonl 2>&1
FLEXCTC_PHASE_TIMERS=1 FLEXCTC_CMP=0 python profiles/phase_split.py --workload c4 > $O/phase_c4_nocmp.jsonl 2>&1
echo done > $O/done
