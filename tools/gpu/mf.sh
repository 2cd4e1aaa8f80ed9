set -u
O=gpurun_out/mf
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_merge_first.py -x -q > $O/pytest_mf.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "compaction or warp or bf16 or logits or c5_full" > $O/pytest_cmp.log 2>&1
for rep in 1 2; do
  python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/new c4 /" >> $O/ab.txt
  FLEXCTC_CMP=1 python bench.py --workload c5 --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/new c5 /" >> $O/ab.txt
done
echo done > $O/done
