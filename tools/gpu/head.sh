set -u
O=gpurun_out/head
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1
python bench.py > $O/bench_c4.log 2>&1
python bench.py --workload c5 --steps 10 --no-cpu-baseline > $O/bench_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done > $O/done
