set -u
O=gpurun_out/etab
mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu -k "logits or bf16 or warp" > $O/pytest.log 2>&1
for rep in 1 2; do
  python bench.py --input bf16-logits --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/etab c4bf16 /" >> $O/ab.txt
  FLEXCTC_WARP=1 python bench.py --input bf16-logits --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/etab c4bf16warp /" >> $O/ab.txt
done
echo done > $O/done
