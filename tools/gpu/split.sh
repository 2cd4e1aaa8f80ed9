set -u
O=gpurun_out
FLEXCTC_PHASE_TIMERS=1 python tools/warp_split.py --workload c4 > $O/sp_help.jsonl 2>&1
FLEXCTC_WARP=1 FLEXCTC_HELPERS=0 FLEXCTC_PHASE_TIMERS=1 python tools/warp_split.py --workload c4 > $O/sp_nohelp.jsonl 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "warp or c4 or c3 or c1 or c2 or fixture or host" > $O/sp_pytest.log 2>&1
python bench.py --no-cpu-baseline --no-e2e > $O/sp_bench_c4.log 2>&1
echo done > $O/sp_done
ncu --set full --clock-control none --import-source on -k regex:frame_compact -s 3 -c 1 -o $O/ncu_cmp2_c4 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu -i $O/ncu_cmp2_c4.ncu-rep --page raw --csv > $O/ncu_cmp2_raw.csv 2>&1
