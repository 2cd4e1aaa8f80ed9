set -u
O=gpurun_out/lgt
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_logits.py -x -q > $O/pytest_logits.log 2>&1
for rep in 1 2; do
  python bench.py --input bf16-logits --steps 20 --no-cpu-baseline 2>/dev/null | grep '^{' | sed "s/^/direct bf16 /" >> $O/ab.txt
  FLEXCTC_LOGITS_DIRECT=0 python bench.py --input bf16-logits --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/copy bf16 /" >> $O/ab.txt
done
python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/f32 c4 /" >> $O/ab.txt
timeout 1800 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1
echo done > $O/done
