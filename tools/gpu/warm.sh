set -u
O=gpurun_out/warm
mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu -k "c4 or warp or logits or compaction or records" > $O/pytest.log 2>&1
for rep in 1 2 3; do
  FLEXCTC_WARM_IN_PASS=0 python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/sep c4 /" >> $O/ab.txt
  python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/fused c4 /" >> $O/ab.txt
done
python bench.py --input bf16-logits --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/fused c4bf16 /" >> $O/ab.txt
FLEXCTC_WARM_IN_PASS=0 python bench.py --batch 1024 --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/sep c4b1024 /" >> $O/ab.txt
python bench.py --batch 1024 --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/fused c4b1024 /" >> $O/ab.txt
echo done > $O/done
