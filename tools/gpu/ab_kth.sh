set -u
O=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "c4 or c5 or c3 or c2 or c1 or fixture or variants or stress or strides or padding or beam_sizes or theta" > $O/kth_pytest.log 2>&1
python tools/ab.py time --workload c4 nokth kth > $O/ab_kth_c4.jsonl 2>&1
python tools/ab.py time --workload c5 nokth kth > $O/ab_kth_c5.jsonl 2>&1
FLEXCTC_WARP=1 python bench.py --no-cpu-baseline --no-e2e > $O/kth_bench_c4_warp.log 2>&1
echo done > $O/kth_done
