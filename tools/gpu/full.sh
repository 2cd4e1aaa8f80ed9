set -u
O=gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > $O/full_pytest.log 2>&1
python bench.py > $O/full_bench_c4.log 2>&1
python bench.py --workload c5 --steps 10 --no-cpu-baseline > $O/full_bench_c5.log 2>&1
python bench.py --workload c3 --no-cpu-baseline --no-e2e > $O/full_bench_c3.log 2>&1
echo done > $O/full_done
