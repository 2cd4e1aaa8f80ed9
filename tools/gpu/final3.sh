set -u
O=gpurun_out/final3
mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
python bench.py > $O/bench_c4.log 2>&1
python bench.py --input bf16-logits > $O/bench_c4_bf16.log 2>&1
python bench.py --workload c5 --steps 20 > $O/bench_c5.log 2>&1
python bench.py --merge-first --steps 10 --no-cpu-baseline > $O/bench_c4_merge_first.log 2>&1
echo done > $O/done
