set -u
O=gpurun_out/cmp3
mkdir -p $O
for rep in 1 2 3; do
  python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/new c4 /" >> $O/ab.txt
  FLEXCTC_CMP=1 python bench.py --workload c5 --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/new c5 /" >> $O/ab.txt
done
FLEXCTC_WARP=1 python bench.py --input bf16-logits --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/new c4bf16warp /" >> $O/ab.txt
timeout 900 python -m pytest tests -x -q -m gpu -k "compaction or warp or bf16 or logits or c5_full or c4" > $O/pytest.log 2>&1
echo done > $O/done
