# A/B of the compaction pass: register-loading kernel vs the TMA-staged ring (2/3/4 stages)
set -u
O=gpurun_out/cmptma
mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu -k "compaction or warp or bf16 or c5_full or logits" > $O/pytest.log 2>&1
for rep in 1 2; do
for v in "FLEXCTC_CMP_TMA=0" "FLEXCTC_CMP_STAGES=2" "FLEXCTC_CMP_STAGES=3" "FLEXCTC_CMP_STAGES=4"; do
  env $v python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/$v c4 /" >> $O/ab.txt
  env $v FLEXCTC_CMP=1 python bench.py --workload c5 --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/$v c5 /" >> $O/ab.txt
  env $v FLEXCTC_WARP=1 python bench.py --input bf16-logits --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/$v c4bf16warp /" >> $O/ab.txt
done
done
echo done > $O/done
