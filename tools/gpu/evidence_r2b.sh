#!/bin/bash
# Round-2 (second half) evidence for profiles/r2b: bench lines, launch lists, ncu --set full of the
# c4 beam kernel and of the compaction pass (serial, so its own roofline is measured alone),
# the L2 rec-warm A/B, compute-sanitizer over every kernel mode.
set -u
O=gpurun_out/ev2b
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1
python bench.py > $O/bench_c4.log 2>&1
python bench.py --input bf16-logits > $O/bench_c4_bf16.log 2>&1
python bench.py --workload c5 --steps 20 > $O/bench_c5.log 2>&1
FLEXCTC_CMP=1 python bench.py --workload c5 --no-cpu-baseline --no-e2e --steps 10 > $O/bench_c5_records.log 2>&1
python bench.py --merge-first --steps 10 > $O/bench_c4_merge_first.log 2>&1
python bench.py --workload c2 --beam 1 > $O/bench_c2k1.log 2>&1
python bench.py --workload c4 --beam 1 > $O/bench_c4k1.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1
for rep in 1 2 3; do
  FLEXCTC_L2_WARM_REC=0 python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/rec0 /" >> $O/ab_warm_rec.txt
  FLEXCTC_L2_WARM_REC=1 python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/rec1 /" >> $O/ab_warm_rec.txt
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c5.csv \
    python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:ctc_beam -s 3 -c 1 -o $O/prof_beam_c4 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:frame_compact -s 3 -c 1 -o $O/prof_compact_c4 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:frame_compact -s 3 -c 1 -o $O/prof_compact_c5 \
    env FLEXCTC_CMP=1 python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
(echo "## memcheck"; compute-sanitizer --tool memcheck python tests/sanitize_run.py 2>&1 | tail -25;
 echo "## racecheck"; compute-sanitizer --tool racecheck python tests/sanitize_run.py 2>&1 | tail -25;
 echo "## synccheck"; compute-sanitizer --tool synccheck python tests/sanitize_run.py 2>&1 | tail -25) > $O/sanitizer.txt 2>&1
echo done > $O/done
