# quick iteration: GPU tests, c4/c5 bench lines (run from the repo root under gpurun)
set -u
O=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > $O/it_pytest.log 2>&1
python bench.py --no-cpu-baseline > $O/it_bench_c4.log 2>&1
FLEXCTC_HELPERS=0 python bench.py --no-cpu-baseline --no-e2e > $O/it_bench_c4_nohelp.log 2>&1
FLEXCTC_WARP=0 python bench.py --no-cpu-baseline --no-e2e > $O/it_bench_c4_cta.log 2>&1
python bench.py --workload c5 --steps 10 --no-cpu-baseline --no-e2e > $O/it_bench_c5.log 2>&1
echo done > $O/it_done
