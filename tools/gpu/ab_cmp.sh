set -u
O=gpurun_out
mkdir -p ab && cp paper_2508_07315_b200/libflexctc.so ab/libcur.so
timeout 900 python -m pytest tests -x -q -m gpu -k "c4 or c5 or c3 or c2 or c1 or fixture or variants or stress or strides or padding or warp" > $O/ab_pytest.log 2>&1
python tools/ab.py time --workload c4 cur:FLEXCTC_CMP=0 cur:FLEXCTC_CMP=1 > $O/ab_cmp_c4.jsonl 2>&1
python tools/ab.py time --workload c5 cur:FLEXCTC_CMP=0 cur:FLEXCTC_CMP=1 > $O/ab_cmp_c5.jsonl 2>&1
python bench.py --no-cpu-baseline --no-e2e --steps 20 > $O/ab_bench_c4.log 2>&1
python bench.py --workload c5 --no-cpu-baseline --no-e2e --steps 10 > $O/ab_bench_c5.log 2>&1
echo done > $O/ab_done
