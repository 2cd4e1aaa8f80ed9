set -u
O=gpurun_out
./tools/micro/zc > $O/misc_zc.json 2>&1
python tools/h2d_bw.py > $O/misc_h2d.json 2>&1
timeout 600 python -m pytest tests -x -q -m gpu -k "greedy" > $O/misc_pytest.log 2>&1
python bench.py --workload c4 --beam 1 --no-cpu-baseline > $O/misc_bench_c4k1.log 2>&1
python bench.py --workload c5 --steps 10 --no-cpu-baseline > $O/misc_bench_c5.log 2>&1
echo done > $O/misc_done
