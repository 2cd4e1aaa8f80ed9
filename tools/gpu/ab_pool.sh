set -u
O=gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pool_pytest.log 2>&1
python tools/ab.py time --workload c4 nopool pool > $O/ab_pool_c4.jsonl 2>&1
python tools/ab.py time --workload c3 nopool pool > $O/ab_pool_c3.jsonl 2>&1
FLEXCTC_WARP=1 python bench.py --no-cpu-baseline --no-e2e > $O/pool_bench_c4_warp.log 2>&1
python bench.py --no-cpu-baseline --no-e2e > $O/pool_bench_c4.log 2>&1
echo done > $O/pool_done
