set -u
O=gpurun_out/san2
mkdir -p $O
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tests/sanitize_run.py > $O/${tool}.txt 2>&1
done
python bench.py --workload c5 --steps 10 --no-cpu-baseline > $O/bench_c5.log 2>&1
FLEXCTC_WARP=1 python bench.py --no-cpu-baseline --no-e2e > $O/bench_c4_warp.log 2>&1
echo done > $O/done
