set -u
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/base_smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/base_pytest.log 2>&1
python bench.py > $O/base_bench_c4.log 2>&1
python bench.py --workload c5 --steps 10 --no-cpu-baseline > $O/base_bench_c5.log 2>&1
FLEXCTC_PHASE_TIMERS=1 python profiles/phase_split.py --workload c4 > $O/base_phase_c4.jsonl 2>&1
echo done > $O/base_done
