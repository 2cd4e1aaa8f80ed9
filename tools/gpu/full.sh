set -u
O=gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > $O/full_pytest.log 2>&1
python bench.py > $O/full_bench_c4.log 2>&1
FLEXCTC_WARP=1 python bench.py --no-cpu-baseline --no-e2e > $O/full_bench_c4_warp.log 2>&1
python bench.py --workload c5 --steps 10 --no-cpu-baseline --no-e2e > $O/full_bench_c5.log 2>&1
FLEXCTC_CMP=1 python bench.py --workload c5 --steps 10 --no-cpu-baseline --no-e2e > $O/full_bench_c5_cmp.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:frame_compact -s 3 -c 1 -o $O/ncu_cmp5_c4 \
    env FLEXCTC_WARP=1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done > $O/full_done
