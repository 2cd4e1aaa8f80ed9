set -u
O=gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > $O/e2e_pytest.log 2>&1
python bench.py --workload c5 --steps 10 --no-cpu-baseline > $O/e2e_bench_c5.log 2>&1
python bench.py --no-cpu-baseline > $O/e2e_bench_c4.log 2>&1
python bench.py --workload c5 --steps 10 --no-cpu-baseline --input bf16-logits > $O/e2e_bench_c5_bf16.log 2>&1
echo done > $O/e2e_done
