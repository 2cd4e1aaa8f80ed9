set -u
O=gpurun_out/mf2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_merge_first.py -x -q > $O/pytest.log 2>&1
python bench.py --merge-first --steps 10 --no-cpu-baseline > $O/bench_c4_mf.log 2>&1
echo done > $O/done
