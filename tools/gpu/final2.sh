set -u
O=gpurun_out/final2
mkdir -p $O
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest.log 2>&1
python bench.py --input bf16-logits > $O/bench_c4_bf16.log 2>&1
python bench.py > $O/bench_c4.log 2>&1
FLEXCTC_WARP=1 python bench.py --input bf16-logits --steps 10 --no-cpu-baseline --no-e2e > $O/bench_c4_bf16_warp.log 2>&1
echo done > $O/done
