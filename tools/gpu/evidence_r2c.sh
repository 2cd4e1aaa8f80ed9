#!/bin/bash
# Final round-2 evidence (profiles/r2c): GPU suite, smoke, bench lines of the final tree.
set -u
O=gpurun_out/ev2c
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python bench.py > $O/bench_c4.log 2>&1
python bench.py --input bf16-logits > $O/bench_c4_bf16.log 2>&1
python bench.py --workload c5 --steps 20 > $O/bench_c5.log 2>&1
FLEXCTC_CMP=1 python bench.py --workload c5 --no-cpu-baseline --no-e2e --steps 10 > $O/bench_c5_records.log 2>&1
python bench.py --merge-first --steps 10 > $O/bench_c4_merge_first.log 2>&1
python bench.py --workload c2 --beam 1 > $O/bench_c2k1.log 2>&1
python bench.py --workload c4 --beam 1 > $O/bench_c4k1.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c4_bf16.csv \
    python bench.py --input bf16-logits --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done > $O/done
