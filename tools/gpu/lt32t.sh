set -u
O=gpurun_out/lt32t
mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python bench.py --workload c5 --steps 20 --no-cpu-baseline > $O/bench_c5.log 2>&1
python bench.py --no-cpu-baseline > $O/bench_c4.log 2>&1
echo done > $O/done
