set -u
O=gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "records or c4_full or fixture" > $O/rec_pytest.log 2>&1
python tools/ab.py time --workload c4 rec rec:FLEXCTC_CMP=1 > $O/ab_rec_c4.jsonl 2>&1
FLEXCTC_CMP=1 python bench.py --no-cpu-baseline --no-e2e > $O/rec_bench_c4.log 2>&1
echo done > $O/rec_done
