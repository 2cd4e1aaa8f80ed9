#!/bin/bash
# GPU evidence for profiles/ (run under gpurun from the repo root): bench lines, launch lists and
# one `ncu --set full` capture per dominant kernel. Output in gpurun_out/ev_*.
set -u
O=gpurun_out
mkdir -p $O
python bench.py > $O/ev_bench_c4.log 2>&1
python bench.py --workload c5 --steps 20 > $O/ev_bench_c5.log 2>&1
python bench.py --workload c2 --beam 1 > $O/ev_bench_c2k1.log 2>&1
python bench.py --workload c2 --beam 1 --batch 512 --steps 30 --no-cpu-baseline > $O/ev_bench_c2k1_b512.log 2>&1
python bench.py --workload c4 --beam 1 > $O/ev_bench_c4k1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/ev_launches_c4.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/ev_launches_c4k1.csv \
    python bench.py --workload c4 --beam 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/ev_launches_c2k1.csv \
    python bench.py --workload c2 --beam 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ctc_beam -s 3 -c 1 -o $O/ev_prof_beam_c4 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:frame_summary -s 3 -c 1 -o $O/ev_prof_sum_c2 \
    python bench.py --workload c2 --beam 1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:greedy_fused -s 3 -c 1 -o $O/ev_prof_fused_c4 \
    python bench.py --workload c4 --beam 1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done > $O/ev_done
