set -u
O=gpurun_out/etab2
mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu -k "logits or bf16 or warp or smoke or host" > $O/pytest.log 2>&1
python bench.py --workload c5 --input bf16-logits --steps 10 --no-cpu-baseline > $O/bench_c5_bf16.log 2>&1
FLEXCTC_LOGITS_DIRECT=0 python bench.py --input bf16-logits --steps 20 --no-cpu-baseline --no-e2e > $O/bench_c4_bf16_copy.log 2>&1
python bench.py --workload c2 --beam 1 --input bf16-logits --no-cpu-baseline > $O/bench_c2k1_bf16.log 2>&1
echo done > $O/done
